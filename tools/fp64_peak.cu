// FP64 throughput probes on the B200 (sm_100a): the roofline denominator for
// the FP64-bound kernels of the filter path (MEASURED_PEAKS.json carries only
// HBM and bf16 figures).
//   dfma  : independent DFMA chains per thread (FP64 vector pipe)
//   dmma  : mma.sync.aligned.m8n8k4.f64 (FP64 tensor pipe, warp level)
//   dmma16: mma.sync.aligned.m16n8k16.f64 (sm_90+ shape)
// Output: one JSON line with TFLOP/s per probe (best of 5, CUDA events).
#include <cuda_runtime.h>
#include <stdio.h>

#define ITERS 4096

__global__ void dfma_kernel(double* out, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 1234.5) out[0] = s;
}

__global__ void dmma_kernel(double* out) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[0] = s;
}

__global__ void dmma16_kernel(double* out) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + i * 1e-4;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) c[i][j] = 0.0;
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
          "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
          : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
            "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 1234.5) out[0] = s;
}

template <class F>
float best_ms(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int blocks = sms * 8, threads = 256;
  const double nthreads = double(blocks) * threads;
  float ms = best_ms([&] { dfma_kernel<<<blocks, threads>>>(out, 1.0000001, 1e-9); });
  const double dfma_tf = nthreads * ITERS * 16 * 2 / (ms * 1e-3) / 1e12;
  ms = best_ms([&] { dmma_kernel<<<blocks, threads>>>(out); });
  // m8n8k4: 8*8*4 MACs per warp-instruction
  const double warps = nthreads / 32;
  const double dmma_tf = warps * ITERS * 8 * (8 * 8 * 4 * 2) / (ms * 1e-3) / 1e12;
  ms = best_ms([&] { dmma16_kernel<<<blocks, threads>>>(out); });
  const double dmma16_tf = warps * (ITERS / 4) * 4 * (16 * 8 * 16 * 2) / (ms * 1e-3) / 1e12;
  cudaError_t e = cudaGetLastError();
  printf("{\"dfma_tflops\": %.2f, \"dmma_m8n8k4_tflops\": %.2f, \"dmma_m16n8k16_tflops\": %.2f, \"sms\": %d, \"err\": \"%s\"}\n",
         dfma_tf, dmma_tf, dmma16_tf, sms, cudaGetErrorString(e));
  return 0;
}

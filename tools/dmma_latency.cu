// DMMA (mma.sync.m8n8k4.f64) latency / throughput vs independent accumulator
// chains per warp, one CTA of W warps on one SM. Prints cycles per DMMA.
#include <cuda_runtime.h>
#include <stdio.h>

template <int CH>
__global__ void chain_kernel(double* out, long long* cyc, int iters) {
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = threadIdx.x * 1e-9;
  const double a = 1.0 + threadIdx.x * 1e-12, b = 0.999;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int CH>
void run(int warps) {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8);
  const int iters = 2048;
  chain_kernel<CH><<<1, 32 * warps>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  chain_kernel<CH><<<1, 32 * warps>>>(out, cyc, iters);
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("chains/warp %2d warps %2d: %.1f cycles per warp-DMMA-step (per chain-step latency %.1f), "
         "SM throughput %.1f cycles/DMMA\n",
         CH, warps, double(h) / iters, double(h) / iters, double(h) / (double(iters) * CH * warps));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<1>(1);
  run<2>(1);
  run<4>(1);
  run<8>(1);
  run<16>(1);
  run<4>(4);
  run<4>(8);
  run<8>(8);
  run<4>(16);
  run<8>(16);
  return 0;
}

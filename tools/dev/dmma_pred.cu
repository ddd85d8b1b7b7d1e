// development: do predicated-off DMMAs cost tensor-pipe time? 8 chains per warp,
// k-step mask from a runtime argument (predicated), vs an explicit warp-uniform branch.
#include <cuda_runtime.h>
#include <stdio.h>

template <int MODE>  // 0: predicated by mask bit, 1: branch per k-step
__global__ void k(double* out, long long* cyc, int iters, unsigned km) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = threadIdx.x * 1e-9;
  const double a = 1.0 + threadIdx.x * 1e-12, b = 0.999;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int kb = 0; kb < 8; ++kb) {
      if (MODE == 0) {
        if (!((km >> kb) & 1u)) continue;
      } else {
        if (__any_sync(0xffffffffu, ((km >> kb) & 1u) == 0)) continue;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1])
                     : "d"(a), "d"(b));
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8 * 1024);
  const int iters = 2000, warps = 16;
  unsigned masks[] = {0xffu, 0x0fu, 0x55u, 0x01u, 0x00u};
  for (int mode = 0; mode < 2; ++mode)
    for (unsigned km : masks) {
      long long h = 0;
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0)
          k<0><<<148, 32 * warps>>>(out, cyc, iters, km);
        else
          k<1><<<148, 32 * warps>>>(out, cyc, iters, km);
        cudaDeviceSynchronize();
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      }
      const int on = __builtin_popcount(km);
      const double issued = 8.0 * 8 * iters * warps / 4.0;  // DMMAs per SMSP if all on
      printf("mode %s mask %02x (%d/8 on): %lld cycles, %.2f cycles per issued-slot DMMA, %.2f per executed\n",
             mode ? "branch" : "pred  ", km, on, h, h / issued, on ? h / (issued * on / 8.0) : 0.0);
    }
  return 0;
}

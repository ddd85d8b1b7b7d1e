// (development) peak rate of the sweeps' 3M tile product loop (mma.cuh mma_tile3) with the data
// always resident in shared memory: 8 consumer warps per CTA, one CTA per SM, no barriers.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../include tile3_rate.cu -o tile3_rate
#include <cstdio>
#include "../../paper_1701_08935_b200/csrc/mma.cuh"
using namespace zolo;

template <int XC, int NB>
__global__ void __launch_bounds__(256, 1) rate(int iters, unsigned mask, double* out) {
  __shared__ __align__(1024) cd ts[TT];
  __shared__ __align__(1024) cd xs[XC * TILE];
  for (int e = threadIdx.x; e < TT; e += blockDim.x) ts[e] = mk(1e-3 * (e % 7), 1e-3 * (e % 5));
  for (int e = threadIdx.x; e < XC * TILE; e += blockDim.x) xs[e] = mk(1e-3 * (e % 3), 1e-3 * (e % 11));
  __syncthreads();
  const Frag f = frag();
  const TileOff o = tile_off<XC>(f);
  Acc3<NB> acc;
  acc3_zero(acc);
  for (int it = 0; it < iters; ++it)
    mma_tile3<XC, NB>(acc, ts, xs, (it & 1) != 0, (it & 2) != 0, o, (mask >> f.r0) & 0xffu);
  cd r[2 * NB];
  acc3_fold(acc, r);
  double s = 0;
  for (int q = 0; q < 2 * NB; ++q) s += r[q].x + r[q].y;
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  for (int variant = 0; variant < 2; ++variant) {
    for (int pass = 0; pass < 2; ++pass) {
      cudaEventRecord(a);
      if (variant == 0)
        rate<64, 4><<<sms, 256>>>(iters, 0xffffffffu, d);
      else
        rate<32, 2><<<sms * 2, 256>>>(iters, 0xffffffffu, d);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double ctas = variant == 0 ? sms : 2.0 * sms;
      const double dmma = ctas * 8.0 * iters * 8 * 3 * (variant == 0 ? 4 : 2);  // warps x k-steps x 3 x blocks
      const double tf = dmma * 512.0 / (ms * 1e-3) / 1e12;
      if (pass) printf("%s: %.3f ms, %.2f TF/s of DMMA (peak ~37.1)\n", variant == 0 ? "64-col 8x32 warps, 1 CTA/SM" : "32-col 8x16 warps, 2 CTA/SM", ms, tf);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

// (development) peak rate of the sweeps' 3M tile product loop (mma.cuh mma_tile3) with the data
// always resident in shared memory: 8 consumer warps per CTA, one CTA per SM, no barriers.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../include tile3_rate.cu -o tile3_rate
#include <cstdio>
#include "../../paper_1701_08935_b200/csrc/mma.cuh"
using namespace zolo;

// variant of mma.cuh mma_tile3 whose B sums are NOT computed (timing only: wrong P3)
template <int XC, int NB, int MODE>
__device__ __forceinline__ void tile3_probe(Acc3<NB>& acc, const cd* ts, const cd* xs, bool opH, bool neg, const TileOff& o,
                                           unsigned km) {
  if (km == 0) return;
  __syncwarp();
  const int a0 = opH ? o.ah0 : o.an, a1 = opH ? o.ah1 : o.an, ash = opH ? 2 : 7;
  const int mre = neg ? static_cast<int>(0x80000000u) : 0;
  const int mim = (neg != opH) ? static_cast<int>(0x80000000u) : 0;
#pragma unroll
  for (int k0 = 0; k0 < TILE / 4; k0 += 4) {
    cd a[4], b[4][NB];
    double bsum[4][NB];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int kk = k0 + q;
      a[q] = ts[((kk & 1) ? a1 : a0) + (kk << ash)];
      const int xo = ((kk & 1) ? o.xb1 : o.xb0) + 8 * XC * (kk >> 1);
#pragma unroll
      for (int h = 0; h < NB; ++h) b[q][h] = xs[xo + 128 * h];
      if (MODE == 3) {  // sums from a plane of doubles: [col][32 rows], row index XOR-swizzled by the column
        const double* ss = reinterpret_cast<const double*>(ts);  // (timing probe: aliases the tile)
        const int lane = threadIdx.x & 31, col = lane >> 2, k = 4 * kk + (lane & 3);
#pragma unroll
        for (int h = 0; h < NB; ++h) bsum[q][h] = ss[(col + 16 * h) * 32 + (k ^ (4 * (col & 7)))];
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (!((km >> (k0 + q)) & 1u)) continue;
      const double re = flip_sign(a[q].x, mre);
      const double im = flip_sign(a[q].y, mim);
      const double s = MODE == 2 ? re : re + im;
#pragma unroll
      for (int h = 0; h < NB; ++h) dmma_nv(acc.p[h][0], re, b[q][h].x);
#pragma unroll
      for (int h = 0; h < NB; ++h) dmma_nv(acc.p[h][1], im, b[q][h].y);
#pragma unroll
      for (int h = 0; h < NB; ++h) dmma_nv(acc.p[h][2], s, MODE == 3 ? bsum[q][h] : (MODE >= 1 ? b[q][h].x : b[q][h].x + b[q][h].y));
    }
  }
}

template <int XC, int NB, int MODE>
__global__ void __launch_bounds__(256, 1) rate_probe(int iters, unsigned mask, double* out) {
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
    tile3_probe<XC, NB, MODE>(acc, ts, xs, (it & 1) != 0, (it & 2) != 0, o, (mask >> f.r0) & 0xffu);
  cd r[2 * NB];
  acc3_fold(acc, r);
  double s = 0;
  for (int q = 0; q < 2 * NB; ++q) s += r[q].x + r[q].y;
  if (s == 12345.0) out[0] = s;
}

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
  for (int mode = 1; mode <= 3; ++mode)
    for (int pass = 0; pass < 2; ++pass) {
      cudaEventRecord(a);
      if (mode == 1)
        rate_probe<64, 4, 1><<<sms, 256>>>(iters, 0xffffffffu, d);
      else if (mode == 2)
        rate_probe<64, 4, 2><<<sms, 256>>>(iters, 0xffffffffu, d);
      else
        rate_probe<64, 4, 3><<<sms, 256>>>(iters, 0xffffffffu, d);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double dmma = sms * 8.0 * iters * 8 * 3 * 4;
      if (pass)
        printf("probe %s: %.3f ms, %.2f TF/s\n", mode == 1 ? "no B sums" : (mode == 2 ? "no A or B sums" : "B sums loaded from smem"), ms,
               dmma * 512.0 / (ms * 1e-3) / 1e12);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

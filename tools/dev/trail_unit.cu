// Unit check of factor.cu's trailing_level_kernel (one target, 3 contributions).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <complex>
#include "../../paper_1701_08935_b200/csrc/factor.cu"
using namespace zolo;

// V1: single buffer, no lambdas
__global__ void __launch_bounds__(ST, 2) v1(const int* tgt, const int* con, int t0, cd* Dt, cd* Lt, cd* Ut) {
  extern __shared__ __align__(16) unsigned char smx[];
  cd* sm = reinterpret_cast<cd*>(smx);
  const int* T = tgt + 4 * (t0 + blockIdx.x);
  const int kind = T[0], id = T[1], cb = T[2], ce = T[3];
  const unsigned long long pol = l2_evict_normal();
  const Frag f = frag();
  Acc8 acc;
  acc8_zero(acc);
  for (int q = cb; q < ce; ++q) {
    load_tile_sw(sm, Lt + static_cast<size_t>(con[2 * q]) * TT, pol);
    load_x32(sm + TT, Ut + static_cast<size_t>(con[2 * q + 1]) * TT, TILE, 0, TILE, pol);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    mma_tile2(acc, sm, sm + TT, false, false, f, 0xffu);
    __syncthreads();
  }
  cd prod[4];
  acc8_fold(acc, prod);
  cd* c = (kind == 0 ? Dt : (kind == 1 ? Lt : Ut)) + static_cast<size_t>(id) * TT;
  for (int q = 0; q < 4; ++q) {
    const int e = ocol(f, q) * TILE + f.row;
    c[e] = csub(c[e], prod[q]);
  }
}
// V2: like mma_unit (fixed nq from arg), pointers direct
__global__ void __launch_bounds__(ST, 2) v2(const int* tgt, const int* con, int t0, cd* Dt, cd* Lt, cd* Ut) {
  extern __shared__ __align__(16) unsigned char smx[];
  cd* sm = reinterpret_cast<cd*>(smx);
  const unsigned long long pol = l2_evict_normal();
  const Frag f = frag();
  Acc8 acc;
  acc8_zero(acc);
  for (int q = 0; q < 3; ++q) {
    load_tile_sw(sm, Lt + q * TT, pol);
    load_x32(sm + TT, Ut + q * TT, TILE, 0, TILE, pol);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    mma_tile2(acc, sm, sm + TT, false, false, f, 0xffu);
    __syncthreads();
  }
  cd prod[4];
  acc8_fold(acc, prod);
  for (int q = 0; q < 4; ++q) {
    const int e = ocol(f, q) * TILE + f.row;
    Dt[e] = csub(Dt[e], prod[q]);
  }
}

// V3: double buffer, no lambdas
__global__ void __launch_bounds__(ST, 2) v3(const int* tgt, const int* con, int t0, cd* Dt, cd* Lt, cd* Ut) {
  extern __shared__ __align__(16) unsigned char smx[];
  cd* sm = reinterpret_cast<cd*>(smx);
  const int* T = tgt + 4 * (t0 + blockIdx.x);
  const int kind = T[0], id = T[1], cb = T[2], ce = T[3];
  const unsigned long long pol = l2_evict_normal();
  const Frag f = frag();
  Acc8 acc;
  acc8_zero(acc);
  load_tile_sw(sm, Lt + static_cast<size_t>(con[2 * cb]) * TT, pol);
  load_x32(sm + TT, Ut + static_cast<size_t>(con[2 * cb + 1]) * TT, TILE, 0, TILE, pol);
  cp_async_commit();
  for (int q = cb; q < ce; ++q) {
    cd* cur = sm + ((q - cb) & 1) * (TT + XS2);
    if (q + 1 < ce) {
      cd* nxt = sm + ((q + 1 - cb) & 1) * (TT + XS2);
      load_tile_sw(nxt, Lt + static_cast<size_t>(con[2 * q + 2]) * TT, pol);
      load_x32(nxt + TT, Ut + static_cast<size_t>(con[2 * q + 3]) * TT, TILE, 0, TILE, pol);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    mma_tile2(acc, cur, cur + TT, false, false, f, 0xffu);
    __syncthreads();
  }
  cd prod[4];
  acc8_fold(acc, prod);
  cd* c = (kind == 0 ? Dt : (kind == 1 ? Lt : Ut)) + static_cast<size_t>(id) * TT;
  for (int q = 0; q < 4; ++q) {
    const int e = ocol(f, q) * TILE + f.row;
    c[e] = csub(c[e], prod[q]);
  }
}
int main() {
  const int nq = 3;
  std::vector<std::complex<double>> L(nq * TT), U(nq * TT), C(TT), R(TT);
  srand(1);
  auto rnd = [] { return std::complex<double>(rand() / (double)RAND_MAX - 0.5, rand() / (double)RAND_MAX - 0.5); };
  for (auto& x : L) x = rnd();
  for (auto& x : U) x = rnd();
  for (auto& x : C) x = rnd();
  R = C;
  for (int q = 0; q < nq; ++q)
    for (int i = 0; i < 32; ++i)
      for (int j = 0; j < 32; ++j) {
        std::complex<double> s = 0;
        for (int k = 0; k < 32; ++k) s += L[q * TT + k * 32 + i] * U[q * TT + j * 32 + k];
        R[j * 32 + i] -= s;
      }
  std::vector<int> tgt = {0, 0, 0, nq}, con = {0, 0, 1, 1, 2, 2};
  cd *dL, *dU, *dC;
  int *dt, *dc;
  cudaMalloc(&dL, sizeof(cd) * L.size()); cudaMalloc(&dU, sizeof(cd) * U.size()); cudaMalloc(&dC, sizeof(cd) * TT);
  cudaMalloc(&dt, 16); cudaMalloc(&dc, 24);
  cudaMemcpy(dL, L.data(), sizeof(cd) * L.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dU, U.data(), sizeof(cd) * U.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dC, C.data(), sizeof(cd) * TT, cudaMemcpyHostToDevice);
  cudaMemcpy(dt, tgt.data(), 16, cudaMemcpyHostToDevice);
  cudaMemcpy(dc, con.data(), 24, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(trailing_level_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TRAIL_SMEM);
  cudaFuncSetAttribute(v1, cudaFuncAttributeMaxDynamicSharedMemorySize, TRAIL_SMEM);
  cudaFuncSetAttribute(v2, cudaFuncAttributeMaxDynamicSharedMemorySize, TRAIL_SMEM);
  int which = getenv("V") ? atoi(getenv("V")) : 0;
  if (which == 0) trailing_level_kernel<<<1, ST, TRAIL_SMEM>>>(dt, dc, 0, dC, dL, dU);
  if (which == 1) v1<<<1, ST, TRAIL_SMEM>>>(dt, dc, 0, dC, dL, dU);
  if (which == 2) v2<<<1, ST, TRAIL_SMEM>>>(dt, dc, 0, dC, dL, dU);
  cudaFuncSetAttribute(v3, cudaFuncAttributeMaxDynamicSharedMemorySize, TRAIL_SMEM);
  if (which == 3) v3<<<1, ST, TRAIL_SMEM>>>(dt, dc, 0, dC, dL, dU);
  cudaError_t e = cudaDeviceSynchronize();
  printf("V%d kernel: %s\n", which, cudaGetErrorString(e));
  cudaMemcpy(C.data(), dC, sizeof(cd) * TT, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < TT; ++i) err = std::max(err, std::abs(C[i] - R[i]));
  printf("max err %.3e\n", err);
  return 0;
}

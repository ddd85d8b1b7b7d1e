// Unit check of the shared DMMA tile helpers (mma.cuh): C -= sum_q A_q B_q for
// 32x32 complex tiles, one CTA, against a host reference.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <complex>
#include "../../paper_1701_08935_b200/csrc/mma.cuh"
using namespace zolo;
__global__ void __launch_bounds__(ST, 2) kern(const cd* A, const cd* B, int nq, cd* C) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  cd* sm = reinterpret_cast<cd*>(sm_raw);
  const unsigned long long pol = l2_evict_normal();
  const Frag f = frag();
  Acc8 acc;
  acc8_zero(acc);
  for (int q = 0; q < nq; ++q) {
    load_tile_sw(sm, A + q * TT, pol);
    load_x32(sm + TT, B + q * TT, TILE, 0, TILE, pol);
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
    C[e] = csub(C[e], prod[q]);
  }
}
int main() {
  const int nq = 3;
  std::vector<std::complex<double>> A(nq * TT), B(nq * TT), C(TT), R(TT);
  srand(1);
  auto rnd = [] { return std::complex<double>(rand() / (double)RAND_MAX - 0.5, rand() / (double)RAND_MAX - 0.5); };
  for (auto& x : A) x = rnd();
  for (auto& x : B) x = rnd();
  for (auto& x : C) x = rnd();
  R = C;
  for (int q = 0; q < nq; ++q)
    for (int i = 0; i < 32; ++i)
      for (int j = 0; j < 32; ++j) {
        std::complex<double> s = 0;
        for (int k = 0; k < 32; ++k) s += A[q * TT + k * 32 + i] * B[q * TT + j * 32 + k];
        R[j * 32 + i] -= s;
      }
  cd *dA, *dB, *dC;
  cudaMalloc(&dA, sizeof(cd) * A.size()); cudaMalloc(&dB, sizeof(cd) * B.size()); cudaMalloc(&dC, sizeof(cd) * TT);
  cudaMemcpy(dA, A.data(), sizeof(cd) * A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), sizeof(cd) * B.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dC, C.data(), sizeof(cd) * TT, cudaMemcpyHostToDevice);
  const int smem = (TT + XS2) * sizeof(cd);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<<<1, ST, smem>>>(dA, dB, nq, dC);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  cudaMemcpy(C.data(), dC, sizeof(cd) * TT, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < TT; ++i) err = std::max(err, std::abs(C[i] - R[i]));
  printf("max err %.3e\n", err);
  return 0;
}

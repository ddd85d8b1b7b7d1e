// Shared device helpers: complex128 as double2, tile geometry, memory-order
// primitives for the flag-synchronised wavefront kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace zolo {

// Block-band tile edge. A tile is TILE x TILE complex128 = 16 KiB, stored
// column-major; the triangular-solve and factorization kernels move whole
// tiles with cp.async into a padded shared-memory copy.
constexpr int TILE = 32;
constexpr int TT = TILE * TILE;
constexpr int TPAD = TILE + 1;  // padded column stride in shared memory
// Right-hand-side columns per solve chain (one column group).
constexpr int CG = 16;

typedef double2 cd;

__host__ __device__ __forceinline__ cd mk(double re, double im) { return make_double2(re, im); }
__host__ __device__ __forceinline__ cd cadd(cd a, cd b) { return mk(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ cd csub(cd a, cd b) { return mk(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ cd cmul(cd a, cd b) { return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__host__ __device__ __forceinline__ cd cconj(cd a) { return mk(a.x, -a.y); }
__host__ __device__ __forceinline__ cd cscale(cd a, double s) { return mk(a.x * s, a.y * s); }
__host__ __device__ __forceinline__ double cabs2(cd a) { return a.x * a.x + a.y * a.y; }
// acc += a * b
__device__ __forceinline__ void cfma(cd& acc, cd a, cd b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
// Smith-style complex division with scaling (avoids overflow like __divdc3).
__host__ __device__ __forceinline__ cd cdiv(cd a, cd b) {
  if (fabs(b.x) >= fabs(b.y)) {
    const double r = b.y / b.x, d = b.x + b.y * r;
    return mk((a.x + a.y * r) / d, (a.y - a.x * r) / d);
  } else {
    const double r = b.x / b.y, d = b.x * r + b.y;
    return mk((a.x * r + a.y) / d, (a.y * r - a.x) / d);
  }
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// 16-byte async copies global -> shared. .cg bypasses L1 (data written by
// other SMs inside the same launch must be read from L2).
__device__ __forceinline__ void cp_async16_cg(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
// L2 eviction-priority policies (createpolicy) and a 16-byte cp.async carrying one
__device__ __forceinline__ unsigned long long l2_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long l2_evict_normal() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long l2_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void cp_async16_cg_hint(void* smem, const void* gmem, unsigned long long pol) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async8_ca(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <class S>
struct ScalarOps;
template <>
struct ScalarOps<double> {
  __device__ static double conj(double x) { return x; }
  __device__ static double abs2(double x) { return x * x; }
  __device__ static cd to_c(double x) { return mk(x, 0.0); }
};
template <>
struct ScalarOps<cd> {
  __device__ static cd conj(cd x) { return cconj(x); }
  __device__ static double abs2(cd x) { return cabs2(x); }
  __device__ static cd to_c(cd x) { return x; }
};

__device__ __forceinline__ double sconj(double x) { return x; }
__device__ __forceinline__ cd sconj(cd x) { return cconj(x); }
__device__ __forceinline__ double smul(double a, double b) { return a * b; }
__device__ __forceinline__ cd smul(cd a, cd b) { return cmul(a, b); }
__device__ __forceinline__ double sadd(double a, double b) { return a + b; }
__device__ __forceinline__ cd sadd(cd a, cd b) { return cadd(a, b); }
__device__ __forceinline__ double ssub(double a, double b) { return a - b; }
__device__ __forceinline__ cd ssub(cd a, cd b) { return csub(a, b); }
__device__ __forceinline__ double sabs2(double x) { return x * x; }
__device__ __forceinline__ double sabs2(cd x) { return cabs2(x); }
__device__ __forceinline__ double sscale(double a, double s) { return a * s; }
__device__ __forceinline__ cd sscale(cd a, double s) { return cscale(a, s); }
__device__ __forceinline__ double szero(double) { return 0.0; }
__device__ __forceinline__ cd szero(cd) { return mk(0.0, 0.0); }
__device__ __forceinline__ cd to_cd(double x) { return mk(x, 0.0); }
__device__ __forceinline__ cd to_cd(cd x) { return x; }

}  // namespace zolo

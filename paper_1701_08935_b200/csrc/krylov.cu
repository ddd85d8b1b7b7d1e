// Krylov-side kernels of the filter application.
//
// Reference map:
//   apply_b / spmm          sparse.hpp:113-129 (spmv over a dense block), SparsePencil::apply_b :141-144
//   combine                 filter_engine.hpp:60-80 (constant term + pole-weight combine)
//   arnoldi (CGS2)          gmres.hpp:128-141 (MGS with one re-orthogonalisation pass)
//   least_squares           gmres.hpp:58-88 + :142-161 (shifted Hessenberg LS, freeze, happy breakdown)
//   assemble                gmres.hpp:163-171 + filter_engine.hpp:112-126 (solutions folded into
//                           the outer partial-fraction combination)
//   gram / block_gemm       eigensolver.hpp:108-109,190 (Rayleigh-Ritz projections, Q = Y Q~)
//
// All reductions are two-stage with a fixed summation order, so results are
// bitwise reproducible run to run.
#include <cuda_runtime.h>

#include <algorithm>

#include "krylov.cuh"
#include "mma.cuh"

namespace zolo {

namespace {

constexpr int RT = 256;          // threads per reduction block
constexpr int RPT = CHUNK / RT;  // rows per thread in a chunk
constexpr int KMAX = KRYLOV_MAX;  // shared-memory room for the Arnoldi coefficients
constexpr int SPC = 8;           // SpMM columns per thread (4 and 16 measured the same)

template <class S>
__device__ __forceinline__ S warp_sum(S v);
template <>
__device__ __forceinline__ double warp_sum<double>(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <>
__device__ __forceinline__ cd warp_sum<cd>(cd v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// perm: device position (0..ld) -> original row, or -1 for identity padding rows.
template <class S>
__global__ void permute_in_kernel(const S* src, int64_t n, S* dst, int64_t ld, const int* perm) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t c = blockIdx.y;
  if (t >= ld) return;
  const int p = perm[t];
  dst[t + c * ld] = (p >= 0) ? src[p + c * n] : szero(S());
}

template <class S>
__global__ void permute_out_kernel(const S* src, int64_t ld, S* dst, int64_t n, const int* perm) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t c = blockIdx.y;
  if (t >= ld) return;
  const int p = perm[t];
  if (p >= 0) dst[p + c * n] = src[t + c * ld];
}

template <class S>
__global__ void col_norms_kernel(const S* v, int64_t n, int64_t ld, double* out) {
  __shared__ double red[32];
  const int64_t c = blockIdx.x;
  double s = 0.0;
  for (int64_t t = threadIdx.x; t < n; t += blockDim.x) s += sabs2(v[t + c * ld]);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) tot += red[w];
    out[c] = sqrt(tot);
  }
}

template <class S>
__global__ void scale_cols_kernel(const S* v, S* out, int64_t ld, const double* norms) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t c = blockIdx.y;
  if (t >= ld) return;
  const double nr = norms[c];
  out[t + c * ld] = nr != 0.0 ? sscale(v[t + c * ld], 1.0 / nr) : szero(S());
}

template <class S>
__global__ void __launch_bounds__(256, 2) apply_b_kernel(int64_t n, int64_t ld, const int* rp, const int* ci, const S* vals, const S* v,
                               const int* act, int na, cd* out) {
  // one row x SPC columns per thread: the row's indices and values are loaded once
  // and reused across the columns (the SpMM is index-load bound otherwise)
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int a0 = blockIdx.y * SPC;
  if (t >= ld) return;
  int64_t col[SPC];
#pragma unroll
  for (int c = 0; c < SPC; ++c) col[c] = (a0 + c < na) ? act[a0 + c] : act[a0];
  S acc[SPC];
#pragma unroll
  for (int c = 0; c < SPC; ++c) acc[c] = szero(S());
  if (t < n) {
    if (rp) {
      constexpr int U = 4;  // the row's entries 4 at a time: 4 x SPC independent loads in flight (-10%)
      const int q1 = rp[t + 1];
      for (int q = rp[t]; q < q1; q += U) {
        int jj[U];
        S bb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const bool ok = q + u < q1;
          jj[u] = ok ? ci[q + u] : static_cast<int>(t);
          bb[u] = ok ? vals[q + u] : szero(S());
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int c = 0; c < SPC; ++c) acc[c] = sadd(acc[c], smul(bb[u], __ldg(v + jj[u] + col[c] * ld)));
      }
    } else {
#pragma unroll
      for (int c = 0; c < SPC; ++c) acc[c] = v[t + col[c] * ld];
    }
  }
#pragma unroll
  for (int c = 0; c < SPC; ++c)
    if (a0 + c < na) out[t + (a0 + c) * ld] = to_cd(acc[c]);
}

template <class S>
__global__ void spmm_kernel(int64_t n, int64_t ld, const int* rp, const int* ci, const S* vals, const S* v, int64_t k,
                            S* out) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t c0 = static_cast<int64_t>(blockIdx.y) * SPC;
  if (t >= ld) return;
  S acc[SPC];
#pragma unroll
  for (int c = 0; c < SPC; ++c) acc[c] = szero(S());
  if (t < n)
    for (int q = rp[t]; q < rp[t + 1]; ++q) {
      const S b = vals[q];
      const int64_t j = ci[q];
#pragma unroll
      for (int c = 0; c < SPC; ++c)
        if (c0 + c < k) acc[c] = sadd(acc[c], smul(b, v[j + (c0 + c) * ld]));
    }
#pragma unroll
  for (int c = 0; c < SPC; ++c)
    if (c0 + c < k) out[t + (c0 + c) * ld] = acc[c];
}

// BSR SpMM (pencils with dense b x b blocks per atom, BASELINE config 4): atoms I in device
// order, block row I holds blocks (I, bci[q]) with dense row-major values bval[q][r][k]; atom I
// occupies device rows row0[I] .. row0[I] + b - 1. One thread per scalar row x SPC columns:
// each block entry is loaded once for the SPC columns, no per-entry column index.
// act != nullptr: columns act[a] of v, output column a of outc (complex, the sweeps' input);
// otherwise columns 0..k-1 of v into out (S).
template <class S>
__global__ void bsr_spmm_kernel(int64_t na, int b, const int* brp, const int* bci, const S* bval, const int* row0,
                                const S* v, int64_t ld, const int* act, int64_t k, S* out, cd* outc) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= na * b) return;
  const int64_t I = t / b;
  const int r = static_cast<int>(t - I * b);
  const int64_t a0 = static_cast<int64_t>(blockIdx.y) * SPC;
  int64_t col[SPC];
#pragma unroll
  for (int c = 0; c < SPC; ++c) {
    const int64_t a = a0 + c < k ? a0 + c : a0;
    col[c] = act ? act[a] : a;
  }
  S acc[SPC];
#pragma unroll
  for (int c = 0; c < SPC; ++c) acc[c] = szero(S());
  for (int q = brp[I]; q < brp[I + 1]; ++q) {
    const S* bv = bval + (static_cast<int64_t>(q) * b + r) * b;
    const int64_t x0 = row0[bci[q]];
    for (int kk = 0; kk < b; ++kk) {
      const S m = bv[kk];
#pragma unroll
      for (int c = 0; c < SPC; ++c) acc[c] = sadd(acc[c], smul(m, v[x0 + kk + col[c] * ld]));
    }
  }
  const int64_t row = row0[I] + r;
#pragma unroll
  for (int c = 0; c < SPC; ++c)
    if (a0 + c < k) {
      if (outc)
        outc[row + (a0 + c) * ld] = to_cd(acc[c]);
      else
        out[row + (a0 + c) * ld] = acc[c];
    }
}

// r_z = b - (A - sigma_z B) x_z per chain z (blockIdx.z), one row x SPC columns per thread: the
// row's A and B entries are read once for the SPC columns (iterative refinement of the shifted
// solves; K = A - sigma B assembled on the fly, assemble_shifted sparse.hpp:153-186)
struct ChainPtrs {
  cd* p[2 * 16];
};
template <class S>
__global__ void shifted_residual_kernel(int64_t n, int64_t ld, const int* arp, const int* aci, const S* av,
                                        const int* brp, const int* bci, const S* bv, const cd* b, ChainPtrs xs,
                                        ChainPtrs rs, const cd* sigma, int na) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int a0 = blockIdx.y * SPC, z = blockIdx.z;
  if (t >= ld) return;
  const cd* x = xs.p[z];
  cd* r = rs.p[z];
  cd ax[SPC], bx[SPC];
#pragma unroll
  for (int c = 0; c < SPC; ++c) ax[c] = bx[c] = mk(0.0, 0.0);
  const int ncl = min(SPC, na - a0);
  if (t < n) {
    for (int q = arp[t]; q < arp[t + 1]; ++q) {
      const cd m = to_cd(av[q]);
      const int64_t j = aci[q];
#pragma unroll
      for (int c = 0; c < SPC; ++c)
        if (c < ncl) cfma(ax[c], m, x[j + (a0 + c) * ld]);
    }
    if (brp) {
      for (int q = brp[t]; q < brp[t + 1]; ++q) {
        const cd m = to_cd(bv[q]);
        const int64_t j = bci[q];
#pragma unroll
        for (int c = 0; c < SPC; ++c)
          if (c < ncl) cfma(bx[c], m, x[j + (a0 + c) * ld]);
      }
    } else {
#pragma unroll
      for (int c = 0; c < SPC; ++c)
        if (c < ncl) bx[c] = x[t + (a0 + c) * ld];
    }
  }
  const cd sg = sigma[z];
#pragma unroll
  for (int c = 0; c < SPC; ++c)
    if (c < ncl) {
      const int64_t off = t + (a0 + c) * ld;
      // padding rows (t >= n) carry zeros in b and x: their residual is zero
      r[off] = t < n ? cadd(csub(b[off], ax[c]), cmul(sg, bx[c])) : mk(0.0, 0.0);
    }
}

__global__ void add_corrections_kernel(int64_t ld, ChainPtrs xs, ChainPtrs ds) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t a = blockIdx.y;
  const int z = blockIdx.z;
  if (t >= ld) return;
  cd* x = xs.p[z];
  x[t + a * ld] = cadd(x[t + a * ld], ds.p[z][t + a * ld]);
}

__global__ void conj_kernel(cd* x, int64_t count) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t < count) x[t].y = -x[t].y;
}

// rows[0..nrows) of columns 0..k-1 set to zero (the identity padding rows of the BSR SpMM output)
__global__ void zero_rows_kernel(const int* rows, int nrows, cd* out, int64_t ld) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < nrows) out[rows[q] + blockIdx.y * ld] = mk(0.0, 0.0);
}

struct XPtrs {
  cd* p[2 * 16];
};

// filter_engine.hpp:60-80
// rb > 0: the row-blocked reduce-scatter layout over nblk blocks (rows >= ld written as zeros)
template <class S>
__global__ void combine_kernel(int64_t ld, double c0, const S* v, const int* act, XPtrs xs, const cd* weights, int r,
                               S* w, int compact, int64_t rb, int nblk) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int a = blockIdx.y;
  if (rb > 0) {
    if (t >= rb * nblk) return;
    if (t >= ld) {
      w[(t / rb) * rb * gridDim.y + a * rb + t % rb] = szero(S());
      return;
    }
  } else if (t >= ld) {
    return;
  }
  const int64_t col = act[a];
  S acc = sscale(v[t + col * ld], c0);
  const int64_t off = t + a * ld;
  if constexpr (sizeof(S) == sizeof(double)) {
    for (int p = 0; p < r; ++p) {
      const cd x = xs.p[p][off];
      const cd wp = weights[p];
      acc += 2.0 * (wp.x * x.x - wp.y * x.y);
    }
  } else {
    for (int p = 0; p < r; ++p) {
      const cd x = xs.p[2 * p][off], xa = xs.p[2 * p + 1][off];
      const cd wp = weights[p];
      acc = cadd(acc, cadd(cmul(wp, x), cmul(cconj(wp), xa)));
    }
  }
  if (rb > 0)
    w[(t / rb) * rb * gridDim.y + a * rb + t % rb] = acc;
  else
    w[t + (compact ? a : col) * ld] = acc;
}

// w[:, act[a]] = wc[:, a] (pole-sharded G: the all-reduced compacted partial sums)
template <class S>
__global__ void scatter_cols_kernel(int64_t ld, const S* wc, const int* act, S* w) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int a = blockIdx.y;
  if (t < ld) w[t + act[a] * ld] = wc[t + a * ld];
}

// ---- CGS2 Arnoldi -------------------------------------------------------
// K1: partial dots <V_i, w> over a row chunk.
template <class S>
__global__ void __launch_bounds__(RT) dots_kernel(int64_t r0, int64_t n, int64_t ld, S* const* basis, int m,
                                                  const S* w, const int* act, S* partial, int nchunk, int hstride,
                                                  const int* done) {
  __shared__ S red[RT / 32][KMAX];
  const int a = blockIdx.x, chunk = blockIdx.y;
  const int64_t col = act[a];
  if (done[col]) return;  // converged in an earlier iteration (lagged active list)
  const int64_t base = r0 + static_cast<int64_t>(chunk) * CHUNK + threadIdx.x;
  S wr[RPT];
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const int64_t t = base + j * RT;
    wr[j] = (t < n) ? w[t + col * ld] : szero(S());
  }
  for (int i = 0; i <= m; ++i) {
    const S* vi = basis[i] + col * ld;
    S s = szero(S());
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const int64_t t = base + j * RT;
      if (t < n) s = sadd(s, smul(sconj(vi[t]), wr[j]));
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][i] = s;
  }
  __syncthreads();
  if (threadIdx.x <= m) {
    S tot = szero(S());
    for (int wq = 0; wq < RT / 32; ++wq) tot = sadd(tot, red[wq][threadIdx.x]);
    partial[(static_cast<int64_t>(a) * nchunk + chunk) * hstride + threadIdx.x] = tot;
  }
}

// K2/K3: h = sum_chunks partial_in; w -= V h; then either dots with the new w
// (partial_out as S) or the squared norm (norm_out as double).
template <class S, bool DOTS>
__global__ void __launch_bounds__(RT) update_kernel(int64_t r0, int64_t n, int64_t ld, S* const* basis, int m, S* w,
                                                    const int* act, const S* partial_in, int nin, S* partial_out,
                                                    double* norm_out, int nchunk, int hstride, S* hsave,
                                                    void* Hmat, int maxit, const int* done) {
  __shared__ S hs[KMAX];
  __shared__ S red[RT / 32][KMAX];
  const int a = blockIdx.x, chunk = blockIdx.y;
  const int64_t col = act[a];
  if (done[col]) return;
  if (threadIdx.x <= m) {
    S tot = szero(S());
    for (int c = 0; c < nin; ++c) tot = sadd(tot, partial_in[(static_cast<int64_t>(a) * nin + c) * hstride + threadIdx.x]);
    hs[threadIdx.x] = tot;
    if (chunk == 0) {
      if (DOTS) {
        hsave[static_cast<int64_t>(a) * hstride + threadIdx.x] = tot;
      } else {
        // H(i, m) = h1 + h2  (gmres.hpp:138 accumulates both passes)
        S* H = reinterpret_cast<S*>(Hmat) + col * static_cast<int64_t>(maxit + 1) * maxit;
        H[threadIdx.x + static_cast<int64_t>(m) * (maxit + 1)] =
            sadd(hsave[static_cast<int64_t>(a) * hstride + threadIdx.x], tot);
      }
    }
  }
  __syncthreads();
  const int64_t base = r0 + static_cast<int64_t>(chunk) * CHUNK + threadIdx.x;
  S wr[RPT];
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const int64_t t = base + j * RT;
    wr[j] = (t < n) ? w[t + col * ld] : szero(S());
  }
  for (int i = 0; i <= m; ++i) {
    const S* vi = basis[i] + col * ld;
    const S h = hs[i];
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const int64_t t = base + j * RT;
      if (t < n) wr[j] = ssub(wr[j], smul(h, vi[t]));
    }
  }
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const int64_t t = base + j * RT;
    if (t < n) w[t + col * ld] = wr[j];
  }
  if (DOTS) {
    for (int i = 0; i <= m; ++i) {
      const S* vi = basis[i] + col * ld;
      S s = szero(S());
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        const int64_t t = base + j * RT;
        if (t < n) s = sadd(s, smul(sconj(vi[t]), wr[j]));
      }
      s = warp_sum(s);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][i] = s;
    }
    __syncthreads();
    if (threadIdx.x <= m) {
      S tot = szero(S());
      for (int wq = 0; wq < RT / 32; ++wq) tot = sadd(tot, red[wq][threadIdx.x]);
      partial_out[(static_cast<int64_t>(a) * nchunk + chunk) * hstride + threadIdx.x] = tot;
    }
  } else {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < RPT; ++j) s += sabs2(wr[j]);
    s = warp_sum(s);
    __shared__ double nred[RT / 32];
    if ((threadIdx.x & 31) == 0) nred[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = 0.0;
      for (int wq = 0; wq < RT / 32; ++wq) tot += nred[wq];
      norm_out[static_cast<int64_t>(a) * nchunk + chunk] = tot;
    }
  }
}

// row-sharded Arnoldi: sum the per-chunk partials of every active column in fixed chunk order
// (cnt entries each: the m + 1 inner products, or 1 squared norm), one chunk per column out
template <class T>
__global__ void reduce_chunks_kernel(const T* partial, int nchunk, int stride, int cnt, const int* act,
                                     const int* done, T* out) {
  const int a = blockIdx.x;
  if (done[act[a]]) return;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    T s = szero(T());
    for (int c = 0; c < nchunk; ++c) s = sadd(s, partial[(static_cast<int64_t>(a) * nchunk + c) * stride + i]);
    out[static_cast<int64_t>(a) * stride + i] = s;
  }
}

// blk: column stride `stride` (>= rows; the reduce-scatter / all-gather block height)
template <class S>
__global__ void pack_rows_kernel(const S* w, int64_t ld, int64_t r0, int64_t rows, int64_t stride, const int* act,
                                 S* blk) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int a = blockIdx.y;
  if (t < rows) blk[t + a * stride] = w[r0 + t + static_cast<int64_t>(act[a]) * ld];
}

template <class S>
__global__ void unpack_rows_kernel(const S* blk, int64_t r0, int64_t rows, int64_t stride, const int* act, S* w,
                                   int64_t ld) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int a = blockIdx.y;
  if (t < rows) w[r0 + t + static_cast<int64_t>(act[a]) * ld] = blk[t + a * stride];
}

template <class S>
__global__ void unpack_blocks_kernel(const S* blocks, int64_t rb, int na, const int* act, S* w, int64_t ld) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;  // global row
  const int a = blockIdx.y;
  if (t >= ld) return;
  const int64_t p = t / rb;
  w[t + static_cast<int64_t>(act[a]) * ld] = blocks[(p * na + a) * rb + (t - p * rb)];
}

__global__ void gmres_init_kernel(GmresDev g) {
  const int c = blockIdx.x, k = threadIdx.x;
  if (k < g.q) {
    const int64_t ck = static_cast<int64_t>(c) * g.q + k;
    cd* G = g.G + ck * (g.maxit + 1);
    for (int i = 0; i <= g.maxit; ++i) G[i] = mk(i == 0 ? g.beta[c] : 0.0, 0.0);
    g.res[ck] = 0.0;
    g.frozen[ck] = 0;
    g.mlen[ck] = 0;
  }
  if (k == 0) {
    g.mcol[c] = 0;
    g.happy[c] = 0;
    g.done[c] = g.beta[c] == 0.0 ? 1 : 0;
    g.wnorm[c] = 0.0;
    for (int i = 0; i < g.maxit; ++i) g.Z[static_cast<int64_t>(c) * g.maxit + i] = mk(0.0, 0.0);
  }
}

// y = R^{-1} g for the leading mm x mm block (gmres.hpp:81-86)
__device__ void back_substitute(const cd* R, const cd* G, cd* y, int mm, int maxit) {
  for (int i = mm - 1; i >= 0; --i) {
    cd v = G[i];
    for (int k = i + 1; k < mm; ++k) v = csub(v, cmul(R[static_cast<int64_t>(k) * maxit + i], y[k]));
    y[i] = cdiv(v, R[static_cast<int64_t>(i) * maxit + i]);
  }
}

// One block per active column, one thread per shift.
template <class S>
__global__ void least_squares_kernel(const int* act, int m, GmresDev g, const double* norm_partial, int nchunk,
                                     double tol) {
  __shared__ double wn_s;
  __shared__ int done_s, happy_s;
  const int a = blockIdx.x, k = threadIdx.x;
  const int col = act[a];
  if (g.done[col]) return;  // converged in an earlier iteration (lagged active list): state frozen
  const int maxit = g.maxit;
  S* H = reinterpret_cast<S*>(g.H) + static_cast<int64_t>(col) * (maxit + 1) * maxit;
  const double beta = g.beta[col];
  if (k == 0) {
    double tot = 0.0;
    for (int c = 0; c < nchunk; ++c) tot += norm_partial[static_cast<int64_t>(a) * nchunk + c];
    const double wn = sqrt(tot);
    wn_s = wn;
    if constexpr (sizeof(S) == sizeof(double))
      reinterpret_cast<double*>(H)[(m + 1) + static_cast<int64_t>(m) * (maxit + 1)] = wn;
    else
      reinterpret_cast<cd*>(H)[(m + 1) + static_cast<int64_t>(m) * (maxit + 1)] = mk(wn, 0.0);
    happy_s = (wn > 1e-14 * beta) ? 0 : 1;  // gmres.hpp:145-150
  }
  __syncthreads();
  const int mm = m + 1;
  if (k < g.q) {
    const int64_t ck = static_cast<int64_t>(col) * g.q + k;
    if (!g.frozen[ck]) {
      cd* R = g.R + ck * maxit * maxit;
      cd* G = g.G + ck * (maxit + 1);
      cd* ROT = g.ROT + ck * 2 * maxit;
      // new column m of H + s I, rotated by the stored Givens (gmres.hpp:62-79)
      cd* rcol = R + static_cast<int64_t>(m) * maxit;  // rows 0..m
      for (int i = 0; i <= m; ++i) rcol[i] = to_cd(H[i + static_cast<int64_t>(m) * (maxit + 1)]);
      rcol[m] = cadd(rcol[m], g.shifts[k]);
      cd below = to_cd(H[(m + 1) + static_cast<int64_t>(m) * (maxit + 1)]);
      for (int j = 0; j < m; ++j) {
        const cd c = ROT[2 * j], sn = ROT[2 * j + 1];
        const cd t0 = rcol[j], t1 = rcol[j + 1];
        rcol[j] = cadd(cmul(cconj(c), t0), cmul(cconj(sn), t1));
        rcol[j + 1] = cadd(cmul(mk(-sn.x, -sn.y), t0), cmul(c, t1));
      }
      const cd av = rcol[m], bv = below;
      const double nr = sqrt(cabs2(av) + cabs2(bv));
      cd c = mk(1.0, 0.0), sn = mk(0.0, 0.0);
      if (nr != 0.0) {
        c = mk(av.x / nr, av.y / nr);
        sn = mk(bv.x / nr, bv.y / nr);
        rcol[m] = cadd(cmul(cconj(c), av), cmul(cconj(sn), bv));
        const cd g0 = G[m], g1 = G[m + 1];
        G[m] = cadd(cmul(cconj(c), g0), cmul(cconj(sn), g1));
        G[m + 1] = cadd(cmul(mk(-sn.x, -sn.y), g0), cmul(c, g1));
      }
      ROT[2 * m] = c;
      ROT[2 * m + 1] = sn;
      const cd gm = G[m + 1];
      const double res = hypot(gm.x, gm.y) / beta;
      g.res[ck] = res;
      if (res <= tol) {  // freeze this shift (gmres.hpp:155-156)
        g.frozen[ck] = 1;
        back_substitute(R, G, g.Y + ck * maxit, mm, maxit);
        g.mlen[ck] = mm;
      }
    }
  }
  __syncthreads();
  if (k == 0) {
    int all = 1;
    for (int s = 0; s < g.q; ++s) all &= g.frozen[static_cast<int64_t>(col) * g.q + s];
    const int done = all || happy_s || mm >= maxit;
    done_s = done;
    g.wnorm[col] = wn_s;
    g.happy[col] = happy_s;
    if (done) {
      g.done[col] = 1;
      g.mcol[col] = mm;
    }
  }
  __syncthreads();
  if (!done_s) return;
  if (k < g.q) {
    const int64_t ck = static_cast<int64_t>(col) * g.q + k;
    if (!g.frozen[ck]) {
      back_substitute(g.R + ck * maxit * maxit, g.G + ck * (maxit + 1), g.Y + ck * maxit, mm, maxit);
      g.mlen[ck] = mm;
    }
  }
  __syncthreads();
  // Z_i = sum_k coef_k y_k[i]  (filter_engine.hpp:112-118 folded through gmres.hpp:163-171)
  for (int i = threadIdx.x; i < mm; i += blockDim.x) {
    cd z = mk(0.0, 0.0);
    for (int s = 0; s < g.q; ++s) {
      const int64_t ck = static_cast<int64_t>(col) * g.q + s;
      if (i < g.mlen[ck]) z = cadd(z, g.ccoef ? cmul(g.Y[ck * maxit + i], g.ccoef[s]) : cscale(g.Y[ck * maxit + i], g.coef[s]));
    }
    g.Z[static_cast<int64_t>(col) * maxit + i] = z;
  }
}

template <class S>
__global__ void next_basis_kernel(int64_t ld, const S* w, S* vnext, const int* act, GmresDev g) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int col = act[blockIdx.y];
  if (t >= ld || g.done[col]) return;
  const double wn = g.wnorm[col];
  vnext[t + col * ld] = sscale(w[t + col * ld], 1.0 / wn);
}

template <class S>
__global__ void assemble_kernel(int64_t ld, S* const* basis, GmresDev g, const S* vin, S* out) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t c = blockIdx.y;
  if (t >= ld) return;
  const int m = g.mcol[c];
  cd acc = mk(0.0, 0.0);
  for (int i = 0; i < m; ++i) {
    const cd z = g.Z[c * g.maxit + i];
    const cd v = to_cd(basis[i][t + c * ld]);
    cfma(acc, z, v);
  }
  const cd half_v = vin ? cscale(to_cd(vin[t + c * ld]), 0.5) : mk(0.0, 0.0);
  if constexpr (sizeof(S) == sizeof(double))
    reinterpret_cast<double*>(out)[t + c * ld] = acc.x + half_v.x;
  else
    reinterpret_cast<cd*>(out)[t + c * ld] = cadd(acc, half_v);
}

// ---- tall-skinny GEMMs for Rayleigh-Ritz -------------------------------
constexpr int GB = 16;
template <class S>
__global__ void gram_partial_kernel(int64_t n, int64_t ld, const S* y, int64_t k, const S* z, int64_t kk,
                                    S* partial) {
  __shared__ S ys[64][GB + 1];
  __shared__ S zs[64][GB + 1];
  const int ti = blockIdx.y * GB, tj = blockIdx.z * GB;
  const int chunk = blockIdx.x;
  const int tx = threadIdx.x % GB, ty = threadIdx.x / GB;  // 256 threads: output (tx, ty)
  S acc = szero(S());
  const int64_t r0 = static_cast<int64_t>(chunk) * CHUNK;
  const int64_t rend = (r0 + CHUNK < n) ? r0 + CHUNK : n;
  for (int64_t rb = r0; rb < rend; rb += 64) {
    for (int e = threadIdx.x; e < 64 * GB; e += 256) {
      const int rr = e % 64, cc = e / 64;
      const int64_t t = rb + rr;
      ys[rr][cc] = (t < n && ti + cc < k) ? y[t + (ti + cc) * ld] : szero(S());
      zs[rr][cc] = (t < n && tj + cc < kk) ? z[t + (tj + cc) * ld] : szero(S());
    }
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < 64; ++rr) acc = sadd(acc, smul(sconj(ys[rr][tx]), zs[rr][ty]));
    __syncthreads();
  }
  if (ti + tx < k && tj + ty < kk) partial[(static_cast<int64_t>(chunk) * k + ti + tx) * kk + tj + ty] = acc;
}

template <class S>
__global__ void gram_reduce_kernel(const S* partial, int nchunk, int64_t k, int64_t kk, S* out) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (e >= k * kk) return;
  const int64_t i = e % k, j = e / k;
  S s = szero(S());
  for (int c = 0; c < nchunk; ++c) s = sadd(s, partial[(static_cast<int64_t>(c) * k + i) * kk + j]);
  out[i + j * k] = s;
}

template <class S>
__global__ void block_gemm_kernel(int64_t ld, const S* y, int64_t k, const S* q, int64_t kk, S* out) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t j = blockIdx.y;
  if (t >= ld) return;
  S acc = szero(S());
  for (int64_t i = 0; i < k; ++i) acc = sadd(acc, smul(y[t + i * ld], q[i + j * k]));
  out[t + j * ld] = acc;
}

// Per column c: num = sum_t |ax - lambda_c bx|^2, den = sum_t |bx|^2
// (relative_residual, eigensolver.hpp:77-93).
template <class S>
__global__ void residual_kernel(int64_t n, const S* ax, const S* bx, const double* lam, double* num, double* den) {
  __shared__ double r1[32], r2[32];
  const int64_t c = blockIdx.x;
  const double l = lam[c];
  double s1 = 0.0, s2 = 0.0;
  for (int64_t t = threadIdx.x; t < n; t += blockDim.x) {
    const S b = bx[t + c * n];
    s1 += sabs2(ssub(ax[t + c * n], sscale(b, l)));
    s2 += sabs2(b);
  }
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  if ((threadIdx.x & 31) == 0) {
    r1[threadIdx.x >> 5] = s1;
    r2[threadIdx.x >> 5] = s2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
      a += r1[w];
      b += r2[w];
    }
    num[c] = a;
    den[c] = b;
  }
}

inline unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

template <class S>
void Krylov<S>::permute_in(cudaStream_t st, const S* src, int64_t n, S* dst, int64_t ld, int64_t k, const int* perm) {
  if (k > 0) permute_in_kernel<S><<<dim3(blocks_for(ld, 256), k), 256, 0, st>>>(src, n, dst, ld, perm);
}
template <class S>
void Krylov<S>::permute_out(cudaStream_t st, const S* src, int64_t ld, S* dst, int64_t n, int64_t k, const int* perm) {
  if (k > 0) permute_out_kernel<S><<<dim3(blocks_for(ld, 256), k), 256, 0, st>>>(src, ld, dst, n, perm);
}
template <class S>
void Krylov<S>::col_norms(cudaStream_t st, const S* v, int64_t n, int64_t ld, int64_t k, double* out) {
  if (k > 0) col_norms_kernel<S><<<k, 512, 0, st>>>(v, n, ld, out);
}
template <class S>
void Krylov<S>::scale_cols(cudaStream_t st, const S* v, S* out, int64_t n, int64_t ld, int64_t k, const double* norms) {
  if (k > 0) scale_cols_kernel<S><<<dim3(blocks_for(ld, 256), k), 256, 0, st>>>(v, out, ld, norms);
}
template <class S>
void Krylov<S>::apply_b(cudaStream_t st, int64_t n, int64_t ld, const int* rp, const int* ci, const S* vals,
                        const S* v, const int* act, int na, cd* out) {
  if (na > 0)
    apply_b_kernel<S><<<dim3(blocks_for(ld, 256), (na + SPC - 1) / SPC), 256, 0, st>>>(n, ld, rp, ci, vals, v, act, na,
                                                                                      out);
}
template <class S>
void Krylov<S>::combine(cudaStream_t st, int64_t n, int64_t ld, double c0, const S* v, const int* act, int na,
                        cd* const* xs, const cd* weights, int r, S* w, bool compact) {
  XPtrs p;
  const int np = sizeof(S) == sizeof(double) ? r : 2 * r;
  for (int i = 0; i < np; ++i) p.p[i] = xs[i];
  if (na > 0)
    combine_kernel<S><<<dim3(blocks_for(ld, 256), na), 256, 0, st>>>(ld, c0, v, act, p, weights, r, w, compact, 0, 1);
}
template <class S>
void Krylov<S>::combine_blocked(cudaStream_t st, int64_t ld, int64_t rb, int nblk, double c0, const S* v,
                                const int* act, int na, cd* const* xs, const cd* weights, int r, S* out) {
  XPtrs p;
  const int np = sizeof(S) == sizeof(double) ? r : 2 * r;
  for (int i = 0; i < np; ++i) p.p[i] = xs[i];
  if (na > 0)
    combine_kernel<S><<<dim3(blocks_for(rb * nblk, 256), na), 256, 0, st>>>(ld, c0, v, act, p, weights, r, out, 0,
                                                                          rb, nblk);
}
template <class S>
void Krylov<S>::pack_rows(cudaStream_t st, const S* w, int64_t ld, int64_t r0, int64_t rows, int64_t stride,
                          const int* act, int na, S* blk) {
  if (na > 0 && rows > 0)
    pack_rows_kernel<S><<<dim3(blocks_for(rows, 256), na), 256, 0, st>>>(w, ld, r0, rows, stride, act, blk);
}
template <class S>
void Krylov<S>::unpack_rows(cudaStream_t st, const S* blk, int64_t r0, int64_t rows, int64_t stride, const int* act,
                            int na, S* w, int64_t ld) {
  if (na > 0 && rows > 0)
    unpack_rows_kernel<S><<<dim3(blocks_for(rows, 256), na), 256, 0, st>>>(blk, r0, rows, stride, act, w, ld);
}
template <class S>
void Krylov<S>::unpack_blocks(cudaStream_t st, const S* blocks, int64_t rb, int nblk, const int* act, int na, S* w,
                              int64_t ld) {
  if (na > 0) unpack_blocks_kernel<S><<<dim3(blocks_for(ld, 256), na), 256, 0, st>>>(blocks, rb, na, act, w, ld);
}
template <class S>
void Krylov<S>::scatter_cols(cudaStream_t st, int64_t ld, const S* wc, const int* act, int na, S* w) {
  if (na > 0) scatter_cols_kernel<S><<<dim3(blocks_for(ld, 256), na), 256, 0, st>>>(ld, wc, act, w);
}
template <class S>
int Krylov<S>::arnoldi(cudaStream_t st, int64_t r0, int64_t r1, int64_t ld, S* const* d_basis, int m, S* w,
                       const int* act, int na, GmresDev g, double* partial, S* hsave, Collective* coll) {
  const int nchunk = static_cast<int>(std::max<int64_t>(1, (r1 - r0 + CHUNK - 1) / CHUNK));
  if (na <= 0) return coll ? 1 : nchunk;
  const int hstride = g.maxit + 1;
  S* p1 = reinterpret_cast<S*>(partial);
  S* p2 = p1 + static_cast<int64_t>(na) * nchunk * hstride;
  double* pn = reinterpret_cast<double*>(p1);  // norm partials reuse p1 after K2
  const dim3 grid(na, nchunk);
  if (!coll) {
    dots_kernel<S><<<grid, RT, 0, st>>>(r0, r1, ld, d_basis, m, w, act, p1, nchunk, hstride, g.done);
    update_kernel<S, true><<<grid, RT, 0, st>>>(r0, r1, ld, d_basis, m, w, act, p1, nchunk, p2, nullptr, nchunk,
                                                hstride, hsave, g.H, g.maxit, g.done);
    update_kernel<S, false><<<grid, RT, 0, st>>>(r0, r1, ld, d_basis, m, w, act, p2, nchunk, nullptr, pn, nchunk,
                                                 hstride, hsave, g.H, g.maxit, g.done);
    return nchunk;
  }
  // row-sharded: local chunk partials -> one partial per column -> all-reduced over the ranks (the
  // done columns' slots carry stale values on every rank alike and are never read)
  const size_t words = static_cast<size_t>(na) * hstride * (sizeof(S) / sizeof(double));
  S* red = p2 + static_cast<int64_t>(na) * nchunk * hstride;
  dots_kernel<S><<<grid, RT, 0, st>>>(r0, r1, ld, d_basis, m, w, act, p1, nchunk, hstride, g.done);
  reduce_chunks_kernel<S><<<na, 64, 0, st>>>(p1, nchunk, hstride, m + 1, act, g.done, red);
  coll->allreduce(reinterpret_cast<double*>(red), words, st);
  update_kernel<S, true><<<grid, RT, 0, st>>>(r0, r1, ld, d_basis, m, w, act, red, 1, p2, nullptr, nchunk, hstride,
                                              hsave, g.H, g.maxit, g.done);
  reduce_chunks_kernel<S><<<na, 64, 0, st>>>(p2, nchunk, hstride, m + 1, act, g.done, red);
  coll->allreduce(reinterpret_cast<double*>(red), words, st);
  update_kernel<S, false><<<grid, RT, 0, st>>>(r0, r1, ld, d_basis, m, w, act, red, 1, nullptr, pn, nchunk, hstride,
                                               hsave, g.H, g.maxit, g.done);
  double* nred = reinterpret_cast<double*>(red);
  reduce_chunks_kernel<double><<<na, 32, 0, st>>>(pn, nchunk, 1, 1, act, g.done, nred);
  coll->allreduce(nred, static_cast<size_t>(na), st);
  cudaMemcpyAsync(pn, nred, sizeof(double) * na, cudaMemcpyDeviceToDevice, st);
  return 1;
}
template <class S>
void Krylov<S>::least_squares(cudaStream_t st, const int* act, int na, int m, GmresDev g, const double* partial,
                              int nchunk, double tol) {
  if (na > 0) least_squares_kernel<S><<<na, 32, 0, st>>>(act, m, g, partial, nchunk, tol);
}
template <class S>
void Krylov<S>::next_basis(cudaStream_t st, int64_t n, int64_t ld, const S* w, S* vnext, const int* act, int na,
                           GmresDev g) {
  if (na > 0) next_basis_kernel<S><<<dim3(blocks_for(ld, 256), na), 256, 0, st>>>(ld, w, vnext, act, g);
}
template <class S>
void Krylov<S>::assemble(cudaStream_t st, int64_t n, int64_t ld, const S* v0, S* const* d_basis, int nv, GmresDev g,
                         const S* vin, S* out) {
  if (nv > 0) assemble_kernel<S><<<dim3(blocks_for(ld, 256), nv), 256, 0, st>>>(ld, d_basis, g, vin, out);
}
// ---- Rayleigh-Ritz block algebra on the FP64 tensor cores (complex pencils) ----------
// (Y^H A Y, Y^H B Y, the CholQR Gram matrices and Q = Y Q~ are
// tall-skinny GEMMs). A 32 x 32 block of a column-major matrix into the swizzled tile layout
// (rows >= nr or columns >= nc are zero).
__device__ __forceinline__ void load_block_sw(cd* s, const cd* g, int64_t ld, int64_t nr, int64_t nc) {
  for (int e = threadIdx.x; e < TT; e += ST) {
    const int col = e / TILE, row = e % TILE;
    cd* dst = &s[col * TILE + (row ^ swz(col))];
    if (row < nr && col < nc)
      cp_async16_cg(dst, g + row + col * ld);
    else
      *dst = mk(0.0, 0.0);
  }
}
// a 32 x 32 block as the right operand [col * XPAD + row]
__device__ __forceinline__ void load_block_x(cd* xs, const cd* g, int64_t ld, int64_t nr, int64_t nc) {
  for (int e = threadIdx.x; e < TILE * TILE; e += ST) {
    const int col = e / TILE, row = e % TILE;
    cd* dst = &xs[col * XPAD + row];
    if (row < nr && col < nc)
      cp_async16_cg(dst, g + row + col * ld);
    else
      *dst = mk(0.0, 0.0);
  }
}

// partial[chunk] (k x kk, row-major like gram_partial_kernel) = Y[rows of chunk]^H Z[rows of chunk]:
// one 32 x 32 output tile per CTA, 32-row blocks of the chunk as DMMA tile products (op H)
__global__ void __launch_bounds__(ST) gram_dmma_kernel(int64_t n, int64_t ld, const cd* y, int64_t k, const cd* z,
                                                       int64_t kk, cd* partial) {
  __shared__ __align__(16) cd ts[TT];
  __shared__ __align__(16) cd xs[XS2];
  const int64_t ti = static_cast<int64_t>(blockIdx.y) * TILE, tj = static_cast<int64_t>(blockIdx.z) * TILE;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * CHUNK;
  const int64_t rend = r0 + CHUNK < n ? r0 + CHUNK : n;
  const Frag f = frag();
  Acc8 acc;
  acc8_zero(acc);
  for (int64_t rb = r0; rb < rend; rb += TILE) {
    load_block_sw(ts, y + rb + ti * ld, ld, rend - rb, k - ti);
    load_block_x(xs, z + rb + tj * ld, ld, rend - rb, kk - tj);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    mma_tile2(acc, ts, xs, true, false, f, 0xffu);
    __syncthreads();
  }
  cd o[4];
  acc8_fold(acc, o);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t i = ti + f.row, j = tj + ocol(f, q);
    if (i < k && j < kk) partial[(static_cast<int64_t>(blockIdx.x) * k + i) * kk + j] = o[q];
  }
}

// out (ld x kk) = Y (ld x k) Q (k x kk): one 32-row x 32-column output tile per CTA
__global__ void __launch_bounds__(ST) block_gemm_dmma_kernel(int64_t ld, const cd* y, int64_t k, const cd* q,
                                                             int64_t kk, cd* out) {
  __shared__ __align__(16) cd ts[TT];
  __shared__ __align__(16) cd xs[XS2];
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * TILE, tj = static_cast<int64_t>(blockIdx.y) * TILE;
  const Frag f = frag();
  Acc8 acc;
  acc8_zero(acc);
  for (int64_t kb = 0; kb < k; kb += TILE) {
    load_block_sw(ts, y + r0 + kb * ld, ld, ld - r0, k - kb);
    load_block_x(xs, q + kb + tj * k, k, k - kb, kk - tj);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    mma_tile2(acc, ts, xs, false, false, f, 0xffu);
    __syncthreads();
  }
  cd o[4];
  acc8_fold(acc, o);
#pragma unroll
  for (int qq = 0; qq < 4; ++qq) {
    const int64_t r = r0 + f.row, j = tj + ocol(f, qq);
    if (r < ld && j < kk) out[r + j * ld] = o[qq];
  }
}

template <class S>
void Krylov<S>::gram(cudaStream_t st, int64_t n, int64_t ld, const S* y, int64_t k, const S* z, int64_t kk, S* out,
                     double* partial) {
  const int nchunk = static_cast<int>((n + CHUNK - 1) / CHUNK);
  S* p = reinterpret_cast<S*>(partial);
  if constexpr (sizeof(S) == sizeof(cd))  // complex: DMMA tile products
    gram_dmma_kernel<<<dim3(nchunk, blocks_for(k, TILE), blocks_for(kk, TILE)), ST, 0, st>>>(
        n, ld, reinterpret_cast<const cd*>(y), k, reinterpret_cast<const cd*>(z), kk, reinterpret_cast<cd*>(p));
  else
    gram_partial_kernel<S><<<dim3(nchunk, blocks_for(k, GB), blocks_for(kk, GB)), 256, 0, st>>>(n, ld, y, k, z, kk, p);
  gram_reduce_kernel<S><<<blocks_for(k * kk, 256), 256, 0, st>>>(p, nchunk, k, kk, out);
}
template <class S>
void Krylov<S>::block_gemm(cudaStream_t st, int64_t n, int64_t ld, const S* y, int64_t k, const S* q, int64_t kk,
                           S* out) {
  if (kk <= 0) return;
  if constexpr (sizeof(S) == sizeof(cd))
    block_gemm_dmma_kernel<<<dim3(blocks_for(ld, TILE), blocks_for(kk, TILE)), ST, 0, st>>>(
        ld, reinterpret_cast<const cd*>(y), k, reinterpret_cast<const cd*>(q), kk, reinterpret_cast<cd*>(out));
  else
    block_gemm_kernel<S><<<dim3(blocks_for(ld, 256), kk), 256, 0, st>>>(ld, y, k, q, kk, out);
}
template <class S>
void Krylov<S>::spmm(cudaStream_t st, int64_t n, int64_t ld, const int* rp, const int* ci, const S* vals, const S* v,
                     int64_t k, S* out) {
  if (k > 0)
    spmm_kernel<S><<<dim3(blocks_for(ld, 256), static_cast<unsigned>((k + SPC - 1) / SPC)), 256, 0, st>>>(n, ld, rp, ci,
                                                                                                       vals, v, k, out);
}

template <class S>
void Krylov<S>::bsr_spmm(cudaStream_t st, int64_t na, int b, const int* brp, const int* bci, const S* bval,
                         const int* row0, const S* v, int64_t ld, const int* act, int64_t k, S* out, cd* outc) {
  if (k > 0 && na > 0)
    bsr_spmm_kernel<S><<<dim3(blocks_for(na * b, 256), static_cast<unsigned>((k + SPC - 1) / SPC)), 256, 0, st>>>(
        na, b, brp, bci, bval, row0, v, ld, act, k, out, outc);
}

template <class S>
void Krylov<S>::shifted_residual(cudaStream_t st, int64_t n, int64_t ld, const int* arp, const int* aci, const S* av,
                                 const int* brp, const int* bci, const S* bv, const cd* b, cd* const* x, cd* const* r,
                                 const cd* sigma, int nch, int na) {
  if (na <= 0 || nch <= 0) return;
  ChainPtrs xp, rp;
  for (int z = 0; z < nch; ++z) xp.p[z] = x[z], rp.p[z] = r[z];
  shifted_residual_kernel<S><<<dim3(blocks_for(ld, 256), (na + SPC - 1) / SPC, nch), 256, 0, st>>>(
      n, ld, arp, aci, av, brp, bci, bv, b, xp, rp, sigma, na);
}

void add_corrections(cudaStream_t st, int64_t ld, cd* const* x, cd* const* d, int nch, int na) {
  if (na <= 0 || nch <= 0) return;
  ChainPtrs xp, dp;
  for (int z = 0; z < nch; ++z) xp.p[z] = x[z], dp.p[z] = d[z];
  add_corrections_kernel<<<dim3(blocks_for(ld, 256), na, nch), 256, 0, st>>>(ld, xp, dp);
}

void conj_inplace(cudaStream_t st, cd* x, int64_t count) {
  if (count > 0) conj_kernel<<<blocks_for(count, 256), 256, 0, st>>>(x, count);
}

void zero_rows(cudaStream_t st, const int* rows, int nrows, cd* out, int64_t ld, int64_t k) {
  if (nrows > 0 && k > 0)
    zero_rows_kernel<<<dim3(static_cast<unsigned>((nrows + 255) / 256), static_cast<unsigned>(k)), 256, 0, st>>>(
        rows, nrows, out, ld);
}

template <class S>
void Krylov<S>::residuals(cudaStream_t st, int64_t n, const S* ax, const S* bx, const double* lam, int64_t k,
                          double* num, double* den) {
  if (k > 0) residual_kernel<S><<<k, 512, 0, st>>>(n, ax, bx, lam, num, den);
}

void gmres_init(cudaStream_t st, GmresDev g) { gmres_init_kernel<<<g.nv, 32, 0, st>>>(g); }

template struct Krylov<double>;
template struct Krylov<cd>;

}  // namespace zolo

// Numeric unpivoted block-sparse LU of P(A - sigma B)P^T in 32 x 32 complex128 tiles.
//
// Reference: factorize (band_factor.hpp:135-182) eliminates one column at a
// time with a rank-1 update of the trailing band (:158-177) under the pivot
// monitor |pivot| > 1e-14 ||row||_inf (:160-166). Here the same unpivoted
// elimination runs over the tiles of the block symbolic structure (host
// symbolic.cpp; nested dissection by default, or any caller ordering such as
// the reference's RCM), one level of the block elimination tree at a time:
//
//   diag_level     diagonal tile LU + pivot monitor + triangular inverses
//   panel_level    L(a,k) = A(a,k) U_kk^-1, U(k,a) = L_kk^-1 A(k,a)
//   trailing_level A(a,b) -= sum_k L(a,k) U(k,b), one target per CTA on DMMA
//
// and the off-diagonal tiles are finally row-scaled by the diagonal inverses
// (scale_sp), so the triangular sweeps (trsm.cu) need no diagonal solves.
#include <cuda_runtime.h>
#include <stdio.h>

#include <algorithm>

#include "tiles.cuh"
#include "mma.cuh"

namespace zolo {

namespace {

constexpr int FT = 256;  // factorization threads per CTA

__device__ __forceinline__ void load_tile_async(cd* s, const cd* g) {
  // 1024 complex values, 4 per thread, into the padded [col*TPAD + row] copy
#pragma unroll
  for (int q = 0; q < TT / FT; ++q) {
    const int e = threadIdx.x + q * FT;
    cp_async16_cg(&s[(e / TILE) * TPAD + (e % TILE)], g + e);
  }
}

// Diagonal tile: unpivoted LU in shared memory with the reference's pivot
// monitor (|pivot| > 1e-14 ||row||_inf, band_factor.hpp:160-166), then the
// inverses of its unit-lower and upper triangles (threads 0..127: L^{-1},
// 128..255: U^{-1}; 4 threads per column share each dot product).
__device__ __forceinline__ void diag_factor_body(int64_t n, int k, cd* tile, cd* DinvL, cd* DinvU,
                                                 const double* row_norm, int* fail_index,
                                                 unsigned long long* min_ratio_bits) {
  extern __shared__ __align__(16) unsigned char diag_smem[];
  __shared__ double rn_s[TILE];
  cd* D = reinterpret_cast<cd*>(diag_smem);
  cd* XL = D + TILE * TPAD;
  cd* XU = XL + TILE * TPAD;
  cd(*red)[4][TILE] = reinterpret_cast<cd(*)[4][TILE]>(XU + TILE * TPAD);
  load_tile_async(D, tile);
  cp_async_commit();
  const int t = threadIdx.x;
  if (t < TILE) {  // the pivot monitor's 32 row norms, read once instead of one round trip per pivot
    const int64_t gi = static_cast<int64_t>(k) * TILE + t;
    rn_s[t] = gi < n ? row_norm[gi] : 0.0;
  }
  cp_async_wait<0>();
  __syncthreads();
  double min_ratio = INFINITY;  // thread 0: the smallest |pivot| / ||row|| of the tile
  for (int p = 0; p < TILE; ++p) {
    const cd piv = D[p * TPAD + p];
    const cd inv = cdiv(mk(1.0, 0.0), piv);
    if (t == 0) {
      const int64_t gi = static_cast<int64_t>(k) * TILE + p;
      if (gi < n) {
        const double rn = rn_s[p];
        const double ap = hypot(piv.x, piv.y);
        min_ratio = fmin(min_ratio, ap / fmax(rn, 1e-300));
        if (!(ap > 1e-14 * rn) && *fail_index < 0) *fail_index = static_cast<int>(gi);
      }
    }
    if (t > p && t < TILE) D[p * TPAD + t] = cmul(D[p * TPAD + t], inv);
    __syncthreads();
    const int m = TILE - 1 - p;
    for (int idx = t; idx < m * m; idx += FT) {
      const int i = p + 1 + idx % m, j = p + 1 + idx / m;
      D[j * TPAD + i] = csub(D[j * TPAD + i], cmul(D[p * TPAD + i], D[j * TPAD + p]));
    }
    __syncthreads();
  }
  if (t == 0 && min_ratio < INFINITY)
    atomicMin(min_ratio_bits, static_cast<unsigned long long>(__double_as_longlong(min_ratio)));
  for (int q = 0; q < TT / FT; ++q) {
    const int e = t + q * FT;
    tile[e] = D[(e / TILE) * TPAD + (e % TILE)];
  }
  // triangular inverses, one row of X per step
  const bool upper = t >= 128;
  const int tt = t & 127, c = tt & 31, part = tt >> 5;
  cd* X = upper ? XU : XL;
  for (int q = tt; q < TT; q += 128) {
    const int rr = q % TILE, cc = q / TILE;
    X[cc * TPAD + rr] = mk(0.0, 0.0);
  }
  __syncthreads();
  for (int s = 0; s < TILE; ++s) {
    // L: row i = s; U: row i = 31 - s
    const int i = upper ? TILE - 1 - s : s;
    cd acc = mk(0.0, 0.0);
    if (!upper) {
      // X(i,c) = -sum_{k=c}^{i-1} L(i,k) X(k,c), i > c
      for (int kk = c + part; kk < i; kk += 4) cfma(acc, D[kk * TPAD + i], X[c * TPAD + kk]);
    } else {
      // X(i,c) = (delta - sum_{k=i+1}^{c} U(i,k) X(k,c)) / U(i,i), i <= c
      for (int kk = i + 1 + part; kk <= c; kk += 4) cfma(acc, D[kk * TPAD + i], X[c * TPAD + kk]);
    }
    red[upper][part][c] = acc;
    __syncthreads();
    if (part == 0) {
      const cd s4 = cadd(cadd(red[upper][0][c], red[upper][1][c]), cadd(red[upper][2][c], red[upper][3][c]));
      if (!upper) {
        if (i == c) X[c * TPAD + i] = mk(1.0, 0.0);
        else if (i > c) X[c * TPAD + i] = mk(-s4.x, -s4.y);
      } else if (i <= c) {
        const cd num = csub(mk(i == c ? 1.0 : 0.0, 0.0), s4);
        X[c * TPAD + i] = cdiv(num, D[i * TPAD + i]);
      }
    }
    __syncthreads();
  }
  cd* outL = DinvL + static_cast<size_t>(k) * TT;
  cd* outU = DinvU + static_cast<size_t>(k) * TT;
  for (int q = t; q < TT; q += FT) {
    const int rr = q % TILE, cc = q / TILE;
    outL[q] = XL[cc * TPAD + rr];
    outU[q] = XU[cc * TPAD + rr];
  }
}

// ---------------------------------------------------------------------------
// block-sparse factor path (any node ordering, e.g. nested dissection)
// ---------------------------------------------------------------------------
__device__ __forceinline__ int sp_lookup(const SpGeom& s, int i, int k) {  // tile id of (i, k), i > k
  int lo = s.row_ptr[i], hi = s.row_ptr[i + 1] - 1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const int v = s.row_idx[mid];
    if (v == k) return mid;
    if (v < k)
      lo = mid + 1;
    else
      hi = mid - 1;
  }
  return -1;
}

__global__ void scatter_sp_kernel(SpGeom s, cd* Dt, cd* Lt, cd* Ut, int64_t nnz, const int* e_row, const int* e_col,
                                  const double* a_val, const double* b_val, int cx, double sr, double si,
                                  unsigned long long* row_norm_bits, const int* pad_rows, int npad_rows,
                                  int* err) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (e < nnz) {
    const int pi = e_row[e], pj = e_col[e];
    cd a, b;
    if (cx) {
      a = mk(a_val[2 * e], a_val[2 * e + 1]);
      b = mk(b_val[2 * e], b_val[2 * e + 1]);
    } else {
      a = mk(a_val[e], 0.0);
      b = mk(b_val[e], 0.0);
    }
    const cd v = csub(a, cmul(mk(sr, si), b));  // assemble_shifted (sparse.hpp:153-186)
    const int bi = pi / TILE, bj = pj / TILE;
    const int r = pi % TILE, c = pj % TILE;
    cd* t;
    if (bi == bj) {
      t = Dt + static_cast<size_t>(bi) * TT;
    } else {
      const int id = bi > bj ? sp_lookup(s, bi, bj) : sp_lookup(s, bj, bi);
      if (id < 0) {
        atomicExch(err, 1);  // symbolic structure does not cover the pattern
        return;
      }
      t = (bi > bj ? Lt : Ut) + static_cast<size_t>(id) * TT;
    }
    t[c * TILE + r] = v;
    atomicMax(&row_norm_bits[pi], static_cast<unsigned long long>(__double_as_longlong(hypot(v.x, v.y))));
  } else if (e < nnz + npad_rows) {
    const int row = pad_rows[e - nnz];  // identity padding row
    const int bi = row / TILE, r = row % TILE;
    Dt[static_cast<size_t>(bi) * TT + r * TILE + r] = mk(1.0, 0.0);
    row_norm_bits[row] = static_cast<unsigned long long>(__double_as_longlong(1.0));
  }
}

// ---- level-scheduled block LU (host factor_plan) --------------------------
// all block columns of one level of the block elimination tree at once
__global__ void __launch_bounds__(FT) diag_level_kernel(const int* cols, int c0, int64_t n, cd* Dt, cd* DinvL,
                                                        cd* DinvU, const double* row_norm, int* fail_index,
                                                        unsigned long long* min_ratio_bits) {
  const int k = cols[c0 + blockIdx.x];
  diag_factor_body(n, k, Dt + static_cast<size_t>(k) * TT, DinvL, DinvU, row_norm, fail_index, min_ratio_bits);
}

// C = A B of three column-major tiles on DMMA (3M), one CTA of ST threads; C may alias A or B
// (both are staged in shared memory before C is written)
__device__ __forceinline__ void tile_mm_dmma(const cd* Ag, const cd* Bg, cd* Cg, cd prod[4], const Frag& f) {
  __shared__ __align__(16) cd sa[TT];
  __shared__ __align__(16) cd sb[XS2];
  load_tile_sw(sa, Ag, l2_evict_normal());
  load_x32(sb, Bg, TILE, 0, TILE, l2_evict_normal());
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  Acc3<2> acc;
  acc3_zero(acc);
  mma_tile3_nx(acc, sa, sb, f, 0xffu);
  acc3_fold(acc, prod);
#pragma unroll
  for (int q = 0; q < 4; ++q) Cg[ocol(f, q) * TILE + f.row] = prod[q];
}
__device__ __forceinline__ void tile_mm_dmma(const cd* Ag, const cd* Bg, cd* Cg) {
  cd prod[4];
  tile_mm_dmma(Ag, Bg, Cg, prod, frag());
}

// panel items (k, 2 id + upper): L(a,k) = A(a,k) U_kk^{-1} | U(k,a) = L_kk^{-1} A(k,a)
// The finished L tile's occupancy mask (SpFactor::lmask) is taken from the product's registers.
__global__ void __launch_bounds__(ST) panel_level_kernel(const int* pan, int p0, cd* Lt, cd* Ut, const cd* DinvL,
                                                         const cd* DinvU, unsigned* lmask) {
  __shared__ unsigned mask;
  const int k = pan[2 * (p0 + blockIdx.x)], code = pan[2 * (p0 + blockIdx.x) + 1];
  const bool lower = (code & 1) == 0;
  const int id = code >> 1;
  cd* c = (lower ? Lt : Ut) + static_cast<size_t>(id) * TT;
  if (!lower) {
    tile_mm_dmma(DinvL + static_cast<size_t>(k) * TT, c, c);
    return;
  }
  if (threadIdx.x == 0) mask = 0u;
  const Frag f = frag();
  cd prod[4];
  tile_mm_dmma(c, DinvU + static_cast<size_t>(k) * TT, c, prod, f);  // (syncs the CTA after `mask = 0`)
  unsigned bits = 0u;
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (prod[q].x != 0.0 || prod[q].y != 0.0) bits |= 1u << ((f.row >> 3) * 8 + (ocol(f, q) >> 2));
  bits = __reduce_or_sync(0xffffffffu, bits);
  if ((threadIdx.x & 31) == 0 && bits) atomicOr(&mask, bits);
  __syncthreads();
  if (threadIdx.x == 0) lmask[id] = mask;
}

// One trailing-update target per CTA (left-looking: the tile's whole update, written once):
// C -= sum_k L(a,k) U(k,b) over ALL its contributions (fixed ascending-k order) on DMMA, 3M complex
// products (mma.cuh mma_tile3_nx: 3 real DMMAs per complex MAC instead of 4), accumulators in
// registers across the list. Two 34 KiB stages: the next contribution's tiles stream in (plain
// cp.async; with the L2::cache_hint operand this loop raised "illegal instruction" on the B200)
// while the current product runs; 3 targets resident per SM. (Three stages with one barrier per
// product and 2 targets per SM: 459 ms against 426 for config 3's 8 poles; occupancy masks of the
// U tiles' 8-column groups on top of the L tiles' row masks: 489 ms, the per-block predicates
// spill at 3 targets per SM.)
constexpr int TRAIL_STAGE = TT + XS2;
constexpr int TRAIL_SMEM = 2 * TRAIL_STAGE * static_cast<int>(sizeof(cd));
#ifndef ZOLO_TRAIL_MINB
#define ZOLO_TRAIL_MINB 3
#endif
__global__ void __launch_bounds__(ST, ZOLO_TRAIL_MINB) trailing_level_kernel(const int* tgt, const int* con, int t0, cd* Dt,
                                                               cd* Lt, cd* Ut, cd* scratch,
                                                               const unsigned* __restrict__ lmask) {
  extern __shared__ __align__(16) unsigned char trail_smem[];
  cd* sm = reinterpret_cast<cd*>(trail_smem);
  const int* T = tgt + 2 * (t0 + blockIdx.x);  // packed: kind << 30 | tile id, first contribution; end = the next target's first
  const int kind = static_cast<unsigned>(T[0]) >> 30, id = T[0] & 0x3fffffff, cb = T[1], ce = T[3];
  const Frag f = frag();
  Acc3<2> acc;
  acc3_zero(acc);
  unsigned km0 = 0u, km1 = 0u;  // this warp's unmasked k-steps of the L tile in each stage
  auto issue = [&](int q, int stage) {
    cd* s = sm + stage * TRAIL_STAGE;
    const int la = con[2 * q];
    const unsigned k8 = (lmask[la] >> f.r0) & 0xffu;
    if (stage)
      km1 = k8;
    else
      km0 = k8;
    load_tile_sw(s, Lt + static_cast<size_t>(la) * TT);
    load_x32(s + TT, Ut + static_cast<size_t>(con[2 * q + 1]) * TT, TILE, 0);
    cp_async_commit();
  };
  if (cb < ce) issue(cb, 0);
  for (int q = cb; q < ce; ++q) {
    const int stage = (q - cb) & 1;
    if (q + 1 < ce) {
      issue(q + 1, stage ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    mma_tile3_nx(acc, sm + stage * TRAIL_STAGE, sm + stage * TRAIL_STAGE + TT, f, stage ? km1 : km0);
    __syncthreads();  // the stage is refilled two iterations later
  }
  cd prod[4];
  acc3_fold(acc, prod);
  if (kind == 3) {  // one part of a split target: its product goes to the level's scratch slot
    cd* c = scratch + static_cast<size_t>(id) * TT;
#pragma unroll
    for (int q = 0; q < 4; ++q) c[ocol(f, q) * TILE + f.row] = prod[q];
    return;
  }
  cd* c = (kind == 0 ? Dt : (kind == 1 ? Lt : Ut)) + static_cast<size_t>(id) * TT;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int e = ocol(f, q) * TILE + f.row;
    c[e] = csub(c[e], prod[q]);
  }
}

// Split targets: tile -= part 0 + part 1 + ... (part order: the fixed summation order).
__global__ void __launch_bounds__(ST) combine_parts_kernel(const int* cmb, int m0, cd* Dt, cd* Lt, cd* Ut,
                                                           const cd* scratch) {
  const int* M = cmb + 3 * (m0 + blockIdx.x);
  const int kind = static_cast<unsigned>(M[0]) >> 30, id = M[0] & 0x3fffffff, s0 = M[1], np = M[2];
  cd* c = (kind == 0 ? Dt : (kind == 1 ? Lt : Ut)) + static_cast<size_t>(id) * TT;
#pragma unroll
  for (int q = 0; q < TT / ST; ++q) {
    const int e = threadIdx.x + q * ST;
    cd sum = scratch[static_cast<size_t>(s0) * TT + e];
    for (int p = 1; p < np; ++p) {
      const cd v = scratch[static_cast<size_t>(s0 + p) * TT + e];
      sum = mk(sum.x + v.x, sum.y + v.y);
    }
    c[e] = csub(c[e], sum);
  }
}

// Row scaling L~(i,k) = DinvL_i L(i,k), U~(k,i) = DinvU_k U(k,i).
__global__ void __launch_bounds__(ST) scale_sp_kernel(SpGeom s, cd* Lt, cd* Ut, const cd* DinvL, const cd* DinvU) {
  const int id = blockIdx.x;
  const bool lower = blockIdx.y == 0;
  const int row = lower ? s.tile_row[id] : s.row_idx[id];
  cd* t = (lower ? Lt : Ut) + static_cast<size_t>(id) * TT;
  tile_mm_dmma((lower ? DinvL : DinvU) + static_cast<size_t>(row) * TT, t, t);
}

}  // namespace

void sp_factor(cudaStream_t st, const SpGeom& s, const SpFactor& f, int64_t nnz, const int* e_row, const int* e_col,
               const double* a_val, const double* b_val, int cx, double sig_re, double sig_im, double* row_norm,
               const int* pad_rows, int npad_rows, FactorDevState ds, int* err, const FactorPlanDev& plan) {
  cudaMemsetAsync(f.Dt, 0, sizeof(cd) * s.nb * TT, st);
  if (s.ntiles > 0) {
    cudaMemsetAsync(f.Lt, 0, sizeof(cd) * s.ntiles * TT, st);
    cudaMemsetAsync(f.Ut, 0, sizeof(cd) * s.ntiles * TT, st);
  }
  cudaMemsetAsync(row_norm, 0, sizeof(double) * s.npad, st);
  const int64_t total = nnz + npad_rows;
  if (total > 0)
    scatter_sp_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(
        s, f.Dt, f.Lt, f.Ut, nnz, e_row, e_col, a_val, b_val, cx, sig_re, sig_im,
        reinterpret_cast<unsigned long long*>(row_norm), pad_rows, npad_rows, err);
  constexpr int diag_smem = (3 * TILE * TPAD + 2 * 4 * TILE) * sizeof(cd);
  // the attributes are per device (a process may drive several GPUs)
  cudaFuncSetAttribute(diag_level_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, diag_smem);
  cudaFuncSetAttribute(trailing_level_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TRAIL_SMEM);
  // level-scheduled, left-looking: per level of the block elimination tree the updates of its
  // block columns (and block rows of U), their diagonal blocks, their panels -- 3 launches
  const std::vector<int>& lv = *plan.lvl_ptr;
  const std::vector<int>& pp = *plan.pan_ptr;
  const std::vector<int>& tp = *plan.tgt_ptr;
  const std::vector<int>& cp = *plan.cmb_ptr;
  for (size_t l = 0; l + 1 < lv.size(); ++l) {
    if (tp[l + 1] > tp[l])
      trailing_level_kernel<<<tp[l + 1] - tp[l], ST, TRAIL_SMEM, st>>>(plan.tgt, plan.con, tp[l], f.Dt, f.Lt, f.Ut,
                                                                        plan.scratch, f.lmask);
    if (cp[l + 1] > cp[l])
      combine_parts_kernel<<<cp[l + 1] - cp[l], ST, 0, st>>>(plan.cmb, cp[l], f.Dt, f.Lt, f.Ut, plan.scratch);
    if (lv[l + 1] > lv[l])
      diag_level_kernel<<<lv[l + 1] - lv[l], FT, diag_smem, st>>>(plan.cols, lv[l], s.npad, f.Dt, f.DinvL, f.DinvU,
                                                                   row_norm, ds.fail_index, ds.min_ratio_bits);
    if (pp[l + 1] > pp[l])
      panel_level_kernel<<<pp[l + 1] - pp[l], ST, 0, st>>>(plan.pan, pp[l], f.Lt, f.Ut, f.DinvL, f.DinvU, f.lmask);
  }
  if (s.ntiles > 0) scale_sp_kernel<<<dim3(static_cast<unsigned>(s.ntiles), 2), ST, 0, st>>>(s, f.Lt, f.Ut, f.DinvL, f.DinvU);
}

// Per-tile occupancy masks for the sweeps' DMMA loops: bit (8 g + kb) of
// .x is set when rows 8g..8g+7 x columns 4kb..4kb+3 of the tile (op N) hold a
// nonzero, .y the same for the conjugate transpose (rows 4kb.. x columns 8g..).
// Exact zeros inside a tile are the structural zeros of the elimination.
__global__ void __launch_bounds__(256) tile_mask_kernel(const cd* tiles, uint2* masks) {
  __shared__ unsigned mn, mh;
  const size_t t = blockIdx.x;
  if (threadIdx.x == 0) mn = mh = 0u;
  __syncthreads();
  const cd* T = tiles + t * TT;
  unsigned bn = 0, bh = 0;
  for (int e = threadIdx.x; e < TT; e += blockDim.x) {
    const int col = e / TILE, row = e % TILE;
    const cd v = T[e];
    if (v.x != 0.0 || v.y != 0.0) {
      bn |= 1u << ((row / 8) * 8 + col / 4);
      bh |= 1u << ((col / 8) * 8 + row / 4);
    }
  }
  if (bn) atomicOr(&mn, bn);
  if (bh) atomicOr(&mh, bh);
  __syncthreads();
  if (threadIdx.x == 0) masks[t] = make_uint2(mn, mh);
}

// Work accounting of the sweeps (zolo_sweep_profile): out[0] += nonzero entries of the tiles,
// out[1] += entries inside their unmasked 8 x 4 blocks (the DMMA k-steps the sweeps execute, op N).
__global__ void __launch_bounds__(256) tile_work_kernel(const cd* tiles, const uint2* masks, int64_t ntiles,
                                                        unsigned long long* out) {
  const int64_t t = blockIdx.x;
  if (t >= ntiles) return;
  const cd* T = tiles + t * TT;
  int nz = 0;
  for (int e = threadIdx.x; e < TT; e += blockDim.x) nz += (T[e].x != 0.0 || T[e].y != 0.0);
  nz = __reduce_add_sync(0xffffffffu, nz);
  if ((threadIdx.x & 31) == 0 && nz) atomicAdd(out, static_cast<unsigned long long>(nz));
  if (threadIdx.x == 0) atomicAdd(out + 1, static_cast<unsigned long long>(__popc(masks[t].x)) * 32ull);
}

// Sylvester inertia: negative real parts among the pivots (diagonal of the
// packed U_ii of every diagonal tile; identity padding rows have pivot 1).
__global__ void neg_pivots_kernel(const cd* dt, int nb, unsigned long long* out) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  int neg = 0;
  if (t < static_cast<int64_t>(nb) * TILE) {
    const int64_t b = t / TILE, k = t % TILE;
    neg = dt[b * TT + k * TILE + k].x < 0.0;
  }
  neg = __reduce_add_sync(0xffffffffu, neg);
  if ((threadIdx.x & 31) == 0 && neg) atomicAdd(out, static_cast<unsigned long long>(neg));
}

int64_t count_negative_pivots(cudaStream_t st, const cd* dt, int nb) {
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, sizeof(unsigned long long)) != cudaSuccess) return -1;
  cudaMemsetAsync(d, 0, sizeof(unsigned long long), st);
  const int64_t n = static_cast<int64_t>(nb) * TILE;
  neg_pivots_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(dt, nb, d);
  unsigned long long h = 0;
  cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  cudaFree(d);
  return static_cast<int64_t>(h);
}

// In-place permutation of each 32 x 32 tile into the sweeps' shared-memory
// layout, element (row, col) at col*32 + (row ^ swz(col)) (mma.cuh), so that a
// whole tile moves with one bulk copy (cp.async.bulk) and lands conflict-free.
__global__ void __launch_bounds__(256) swizzle_tile_kernel(cd* tiles) {
  __shared__ cd buf[TT];
  cd* T = tiles + static_cast<size_t>(blockIdx.x) * TT;
  for (int e = threadIdx.x; e < TT; e += blockDim.x) buf[e] = T[e];
  __syncthreads();
  for (int e = threadIdx.x; e < TT; e += blockDim.x) {
    const int col = e / TILE, row = e % TILE;
    T[col * TILE + (row ^ swz(col))] = buf[e];
  }
}

void tile_work(cudaStream_t st, const cd* tiles, const uint2* masks, int64_t ntiles, unsigned long long* out) {
  if (ntiles > 0) tile_work_kernel<<<static_cast<unsigned>(ntiles), 256, 0, st>>>(tiles, masks, ntiles, out);
}

void swizzle_tiles(cudaStream_t st, cd* tiles, int64_t ntiles) {
  if (ntiles > 0) swizzle_tile_kernel<<<static_cast<unsigned>(ntiles), 256, 0, st>>>(tiles);
}

void tile_masks(cudaStream_t st, const cd* tiles, int64_t ntiles, uint2* masks) {
  if (ntiles > 0) tile_mask_kernel<<<static_cast<unsigned>(ntiles), 256, 0, st>>>(tiles, masks);
}

}  // namespace zolo

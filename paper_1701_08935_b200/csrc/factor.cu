// Numeric unpivoted block-band LU of P(A - sigma B)P^T and the multi-RHS
// pipelined triangular solves on it.
//
// Reference: factorize (band_factor.hpp:135-182) eliminates one column at a
// time with a rank-1 update of the trailing band; ShiftedFactor::solve /
// adjoint_solve (band_factor.hpp:53-117) sweep the band once per right-hand
// side column. Here both become dense TILE x TILE complex128 tile products
// over the envelope of the band (see band.cuh):
//
//   factor step k:  diagonal tile LU + pivot monitor + triangular inverses
//                   -> panel tiles (x DinvU / DinvL) -> trailing updates,
//                   then one post-pass builds the coupling tiles M.
//   solve sweep:    x_i = c_i - M_i x_{i-+1},
//                   c_i = Dinv_i (b_i - sum_{d>=2} T_(i,i-+d) x_(i-+d)).
//                   HELPER tasks compute every c_i (all the flops, off the
//                   critical path: they need x up to i-+2); one OWNER task per
//                   (chain, column group) walks the chain doing only the
//                   M_i x_{i-+1} product with x_{i-+1} kept on chip. All poles,
//                   the solve and adjoint chains and all column groups share
//                   ONE persistent launch per sweep direction; dependencies are
//                   per-(chain, group, block) epoch flags (release/acquire).
//                   Owners take the first task indices and helpers are claimed
//                   in dependency order from an atomic counter, so the launch
//                   is deadlock free whenever the owners fit on the device.
#include <cuda_runtime.h>
#include <stdio.h>

#include <algorithm>

#include "band.cuh"
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

// out[2x2] = A(rows) * B(cols) over the full tile; thread (tx,ty) owns rows
// tx, tx+16 and columns ty, ty+16. A, B padded shared tiles.
__device__ __forceinline__ void tile_mm(const cd* As, const cd* Bs, cd out[4]) {
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  cd c00 = mk(0, 0), c01 = mk(0, 0), c10 = mk(0, 0), c11 = mk(0, 0);
#pragma unroll 8
  for (int k = 0; k < TILE; ++k) {
    const cd a0 = As[k * TPAD + tx], a1 = As[k * TPAD + tx + 16];
    const cd b0 = Bs[ty * TPAD + k], b1 = Bs[(ty + 16) * TPAD + k];
    cfma(c00, a0, b0);
    cfma(c01, a0, b1);
    cfma(c10, a1, b0);
    cfma(c11, a1, b1);
  }
  out[0] = c00;
  out[1] = c01;
  out[2] = c10;
  out[3] = c11;
}

__device__ __forceinline__ void store_tile(cd* c, const cd out[4]) {
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  c[ty * TILE + tx] = out[0];
  c[(ty + 16) * TILE + tx] = out[1];
  c[ty * TILE + tx + 16] = out[2];
  c[(ty + 16) * TILE + tx + 16] = out[3];
}

__global__ void scatter_kernel(BandGeom g, cd* Lt, cd* Ut, int64_t nnz, const int* e_row, const int* e_col,
                               const double* a_val, const double* b_val, int cx, double sr, double si,
                               unsigned long long* row_norm_bits) {
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
    // assemble_shifted (sparse.hpp:153-186): A - sigma B on the union pattern
    const cd v = csub(a, cmul(mk(sr, si), b));
    const int bi = pi / TILE, bj = pj / TILE;
    const int r = pi % TILE, c = pj % TILE;
    if (bi >= bj)
      Lt[lt_off(bi, bi - bj, g.J) + c * TILE + r] = v;
    else
      Ut[lt_off(bj, bj - bi, g.J) + c * TILE + r] = v;
    const double av = hypot(v.x, v.y);
    atomicMax(&row_norm_bits[pi], static_cast<unsigned long long>(__double_as_longlong(av)));
  } else if (e < nnz + (g.npad - g.n)) {
    // identity padding rows beyond n
    const int64_t row = g.n + (e - nnz);
    const int bi = static_cast<int>(row / TILE), r = static_cast<int>(row % TILE);
    Lt[lt_off(bi, 0, g.J) + r * TILE + r] = mk(1.0, 0.0);
    row_norm_bits[row] = static_cast<unsigned long long>(__double_as_longlong(1.0));
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

__global__ void __launch_bounds__(FT) diag_factor_kernel(int64_t n, int k, cd* tile, cd* DinvL, cd* DinvU,
                                                         const double* row_norm, int* fail_index,
                                                         unsigned long long* min_ratio_bits) {
  diag_factor_body(n, k, tile, DinvL, DinvU, row_norm, fail_index, min_ratio_bits);
}

// Panel: L(k+d,k) = A(k+d,k) U_kk^{-1} (blocks 0..J-1),
//        U(k,k+d) = L_kk^{-1} A(k,k+d) (blocks J..2J-1); envelope tiles only.
__global__ void __launch_bounds__(FT) panel_kernel(BandGeom g, int k, cd* Lt, cd* Ut, const cd* DinvL,
                                                   const cd* DinvU) {
  __shared__ cd As[TILE * TPAD];
  __shared__ cd Bs[TILE * TPAD];
  const int J = g.J;
  const bool lower = blockIdx.x < J;
  const int d = lower ? blockIdx.x + 1 : blockIdx.x - J + 1;
  if (k + d >= g.nbk || d > g.dl[k + d]) return;
  cd* c;
  if (lower) {
    c = Lt + lt_off(k + d, d, J);
    load_tile_async(As, c);
    load_tile_async(Bs, DinvU + static_cast<size_t>(k) * TT);
  } else {
    c = Ut + lt_off(k + d, d, J);
    load_tile_async(As, DinvL + static_cast<size_t>(k) * TT);
    load_tile_async(Bs, c);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  cd out[4];
  tile_mm(As, Bs, out);
  store_tile(c, out);
}

// Trailing update A(k+a, k+b) -= L(k+a, k) U(k, k+b), a, b in 1..J (envelope).
__global__ void __launch_bounds__(FT) trailing_kernel(BandGeom g, int k, cd* Lt, cd* Ut) {
  __shared__ cd As[TILE * TPAD];
  __shared__ cd Bs[TILE * TPAD];
  const int J = g.J;
  const int a = blockIdx.x + 1, b = blockIdx.y + 1;
  if (k + a >= g.nbk || k + b >= g.nbk) return;
  if (a > g.dl[k + a] || b > g.dl[k + b]) return;
  load_tile_async(As, Lt + lt_off(k + a, a, J));
  load_tile_async(Bs, Ut + lt_off(k + b, b, J));
  cp_async_commit();
  cd* c = (a >= b) ? Lt + lt_off(k + a, a - b, J) : Ut + lt_off(k + b, b - a, J);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const cd c0 = c[ty * TILE + tx], c1 = c[(ty + 16) * TILE + tx], c2 = c[ty * TILE + tx + 16],
           c3 = c[(ty + 16) * TILE + tx + 16];
  cp_async_wait<0>();
  __syncthreads();
  cd out[4];
  tile_mm(As, Bs, out);
  out[0] = csub(c0, out[0]);
  out[1] = csub(c1, out[1]);
  out[2] = csub(c2, out[2]);
  out[3] = csub(c3, out[3]);
  store_tile(c, out);
}

// Row scaling of the off-diagonal factor tiles by the diagonal-block inverses:
//   L~(i, i-d) = DinvL[i] L(i, i-d),     U~(j-d, j) = DinvU[j-d] U(j-d, j).
// With these, every triangular sweep (trsm.cu) is a recurrence without any
// diagonal operation on its critical path. blockIdx = (block row, d - 1, L|U).
__global__ void __launch_bounds__(FT) scale_tiles_kernel(BandGeom g, FactorTiles f) {
  __shared__ cd As[TILE * TPAD];
  __shared__ cd Bs[TILE * TPAD];
  const int i = blockIdx.x, d = blockIdx.y + 1;
  const bool lower = blockIdx.z == 0;
  if (d > g.dl[i]) return;  // outside the envelope: exact zeros
  cd* t = (lower ? f.Lt : f.Ut) + lt_off(i, d, g.J);
  const cd* dinv = lower ? f.DinvL + static_cast<size_t>(i) * TT : f.DinvU + static_cast<size_t>(i - d) * TT;
  load_tile_async(As, dinv);
  load_tile_async(Bs, t);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  cd o[4];
  tile_mm(As, Bs, o);
  store_tile(t, o);
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

// L(i,k) = A(i,k) U_kk^{-1}, U(k,i) = L_kk^{-1} A(k,i) for the structural rows i of column k.
__global__ void __launch_bounds__(FT) panel_sp_kernel(SpGeom s, int k, cd* Lt, cd* Ut, const cd* DinvL,
                                                      const cd* DinvU) {
  __shared__ cd As[TILE * TPAD];
  __shared__ cd Bs[TILE * TPAD];
  const int e0 = s.col_ptr[k], cnt = s.col_ptr[k + 1] - e0;
  const bool lower = static_cast<int>(blockIdx.x) < cnt;
  const int id = s.col_tile[e0 + (lower ? blockIdx.x : blockIdx.x - cnt)];
  cd* c = (lower ? Lt : Ut) + static_cast<size_t>(id) * TT;
  if (lower) {
    load_tile_async(As, c);
    load_tile_async(Bs, DinvU + static_cast<size_t>(k) * TT);
  } else {
    load_tile_async(As, DinvL + static_cast<size_t>(k) * TT);
    load_tile_async(Bs, c);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  cd out[4];
  tile_mm(As, Bs, out);
  store_tile(c, out);
}

// A(a,b) -= L(a,k) U(k,b) over all structural pairs (a, b) of column k.
__global__ void __launch_bounds__(FT) trailing_sp_kernel(SpGeom s, int k, cd* Dt, cd* Lt, cd* Ut, int* err) {
  __shared__ cd As[TILE * TPAD];
  __shared__ cd Bs[TILE * TPAD];
  const int e0 = s.col_ptr[k];
  const int a = s.col_idx[e0 + blockIdx.x], b = s.col_idx[e0 + blockIdx.y];
  load_tile_async(As, Lt + static_cast<size_t>(s.col_tile[e0 + blockIdx.x]) * TT);
  load_tile_async(Bs, Ut + static_cast<size_t>(s.col_tile[e0 + blockIdx.y]) * TT);
  cp_async_commit();
  cd* c;
  if (a == b) {
    c = Dt + static_cast<size_t>(a) * TT;
  } else {
    const int id = a > b ? sp_lookup(s, a, b) : sp_lookup(s, b, a);
    if (id < 0) {
      if (threadIdx.x == 0) atomicExch(err, 1);
      return;
    }
    c = (a > b ? Lt : Ut) + static_cast<size_t>(id) * TT;
  }
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const cd c0 = c[ty * TILE + tx], c1 = c[(ty + 16) * TILE + tx], c2 = c[ty * TILE + tx + 16],
           c3 = c[(ty + 16) * TILE + tx + 16];
  cp_async_wait<0>();
  __syncthreads();
  cd out[4];
  tile_mm(As, Bs, out);
  out[0] = csub(c0, out[0]);
  out[1] = csub(c1, out[1]);
  out[2] = csub(c2, out[2]);
  out[3] = csub(c3, out[3]);
  store_tile(c, out);
}

// ---- level-scheduled block LU (host factor_plan) --------------------------
// all block columns of one level of the block elimination tree at once
__global__ void __launch_bounds__(FT) diag_level_kernel(const int* cols, int c0, int64_t n, cd* Dt, cd* DinvL,
                                                        cd* DinvU, const double* row_norm, int* fail_index,
                                                        unsigned long long* min_ratio_bits) {
  const int k = cols[c0 + blockIdx.x];
  diag_factor_body(n, k, Dt + static_cast<size_t>(k) * TT, DinvL, DinvU, row_norm, fail_index, min_ratio_bits);
}

// panel items (k, 2 id + upper): L(a,k) = A(a,k) U_kk^{-1} | U(k,a) = L_kk^{-1} A(k,a)
__global__ void __launch_bounds__(FT) panel_level_kernel(const int* pan, int p0, cd* Lt, cd* Ut, const cd* DinvL,
                                                         const cd* DinvU) {
  __shared__ cd As[TILE * TPAD];
  __shared__ cd Bs[TILE * TPAD];
  const int k = pan[2 * (p0 + blockIdx.x)], code = pan[2 * (p0 + blockIdx.x) + 1];
  const bool lower = (code & 1) == 0;
  const int id = code >> 1;
  cd* c = (lower ? Lt : Ut) + static_cast<size_t>(id) * TT;
  if (lower) {
    load_tile_async(As, c);
    load_tile_async(Bs, DinvU + static_cast<size_t>(k) * TT);
  } else {
    load_tile_async(As, DinvL + static_cast<size_t>(k) * TT);
    load_tile_async(Bs, c);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  cd out[4];
  tile_mm(As, Bs, out);
  store_tile(c, out);
}

// One trailing-update target per CTA: C -= sum_k L(a,k) U(k,b) over its
// contributions (fixed ascending-k order), on DMMA. (A double-buffered variant
// of this loop raised "illegal instruction" on the B200 -- tools/dev/trail_unit.cu
// reproduces it -- so the stages are single-buffered; the factorization is setup.)
constexpr int TRAIL_SMEM = (TT + XS2) * static_cast<int>(sizeof(cd));
#ifndef ZOLO_TRAIL_MINB
#define ZOLO_TRAIL_MINB 4  // 4 resident targets per SM hide the single-buffered tile loads (cfg3 factor -8%)
#endif
__global__ void __launch_bounds__(ST, ZOLO_TRAIL_MINB) trailing_level_kernel(const int* tgt, const int* con, int t0, cd* Dt,
                                                               cd* Lt, cd* Ut) {
  extern __shared__ __align__(16) unsigned char trail_smem[];
  cd* sm = reinterpret_cast<cd*>(trail_smem);
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
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int e = ocol(f, q) * TILE + f.row;
    c[e] = csub(c[e], prod[q]);
  }
}

// (debug) SIMT variant of trailing_level_kernel
__global__ void __launch_bounds__(FT) trailing_level_simt_kernel(const int* tgt, const int* con, int t0, cd* Dt,
                                                                 cd* Lt, cd* Ut) {
  __shared__ cd As[TILE * TPAD];
  __shared__ cd Bs[TILE * TPAD];
  const int* T = tgt + 4 * (t0 + blockIdx.x);
  const int kind = T[0], id = T[1], cb = T[2], ce = T[3];
  cd acc[4] = {mk(0.0, 0.0), mk(0.0, 0.0), mk(0.0, 0.0), mk(0.0, 0.0)};
  for (int q = cb; q < ce; ++q) {
    load_tile_async(As, Lt + static_cast<size_t>(con[2 * q]) * TT);
    load_tile_async(Bs, Ut + static_cast<size_t>(con[2 * q + 1]) * TT);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    cd out[4];
    tile_mm(As, Bs, out);
    for (int u = 0; u < 4; ++u) acc[u] = cadd(acc[u], out[u]);
    __syncthreads();
  }
  cd* c = (kind == 0 ? Dt : (kind == 1 ? Lt : Ut)) + static_cast<size_t>(id) * TT;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  c[ty * TILE + tx] = csub(c[ty * TILE + tx], acc[0]);
  c[(ty + 16) * TILE + tx] = csub(c[(ty + 16) * TILE + tx], acc[1]);
  c[ty * TILE + tx + 16] = csub(c[ty * TILE + tx + 16], acc[2]);
  c[(ty + 16) * TILE + tx + 16] = csub(c[(ty + 16) * TILE + tx + 16], acc[3]);
}

// Row scaling L~(i,k) = DinvL_i L(i,k), U~(k,i) = DinvU_k U(k,i) (see band path).
__global__ void __launch_bounds__(FT) scale_sp_kernel(SpGeom s, cd* Lt, cd* Ut, const cd* DinvL, const cd* DinvU) {
  __shared__ cd As[TILE * TPAD];
  __shared__ cd Bs[TILE * TPAD];
  const int id = blockIdx.x;
  const bool lower = blockIdx.y == 0;
  const int row = lower ? s.tile_row[id] : s.row_idx[id];
  cd* t = (lower ? Lt : Ut) + static_cast<size_t>(id) * TT;
  load_tile_async(As, (lower ? DinvL : DinvU) + static_cast<size_t>(row) * TT);
  load_tile_async(Bs, t);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  cd o[4];
  tile_mm(As, Bs, o);
  store_tile(t, o);
}

}  // namespace

void sp_factor(cudaStream_t st, const SpGeom& s, const std::vector<int>& col_cnt, const SpFactor& f, int64_t nnz,
               const int* e_row, const int* e_col, const double* a_val, const double* b_val, int cx, double sig_re,
               double sig_im, double* row_norm, const int* pad_rows, int npad_rows, FactorDevState ds, int* err,
               const FactorPlanDev* plan) {
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
  static bool diag_attr = false;
  if (!diag_attr) {
    cudaFuncSetAttribute(diag_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, diag_smem);
    diag_attr = true;
  }
  if (plan) {  // level-scheduled: 3 launches per level of the block elimination tree
    static bool trail_attr = false;
    if (!trail_attr) {
      cudaFuncSetAttribute(diag_level_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, diag_smem);
      cudaFuncSetAttribute(trailing_level_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TRAIL_SMEM);
      trail_attr = true;
    }
    const std::vector<int>& lv = *plan->lvl_ptr;
    const std::vector<int>& pp = *plan->pan_ptr;
    const std::vector<int>& tp = *plan->tgt_ptr;
    for (size_t l = 0; l + 1 < lv.size(); ++l) {
      if (lv[l + 1] > lv[l])
        diag_level_kernel<<<lv[l + 1] - lv[l], FT, diag_smem, st>>>(plan->cols, lv[l], s.npad, f.Dt, f.DinvL,
                                                                     f.DinvU, row_norm, ds.fail_index,
                                                                     ds.min_ratio_bits);
      if (pp[l + 1] > pp[l])
        panel_level_kernel<<<pp[l + 1] - pp[l], FT, 0, st>>>(plan->pan, pp[l], f.Lt, f.Ut, f.DinvL, f.DinvU);
      if (tp[l + 1] > tp[l]) {
        if (plan->simt)
          trailing_level_simt_kernel<<<tp[l + 1] - tp[l], FT, 0, st>>>(plan->tgt, plan->con, tp[l], f.Dt, f.Lt,
                                                                        f.Ut);
        else
          trailing_level_kernel<<<tp[l + 1] - tp[l], ST, TRAIL_SMEM, st>>>(plan->tgt, plan->con, tp[l], f.Dt, f.Lt,
                                                                            f.Ut);
      }
    }
  } else {
    for (int k = 0; k < s.nb; ++k) {
      diag_factor_kernel<<<1, FT, diag_smem, st>>>(s.npad, k, f.Dt + static_cast<size_t>(k) * TT, f.DinvL, f.DinvU,
                                                   row_norm, ds.fail_index, ds.min_ratio_bits);
      const int cnt = col_cnt[k];
      if (cnt > 0) {
        panel_sp_kernel<<<2 * cnt, FT, 0, st>>>(s, k, f.Lt, f.Ut, f.DinvL, f.DinvU);
        trailing_sp_kernel<<<dim3(cnt, cnt), FT, 0, st>>>(s, k, f.Dt, f.Lt, f.Ut, err);
      }
    }
  }
  if (s.ntiles > 0) scale_sp_kernel<<<dim3(static_cast<unsigned>(s.ntiles), 2), FT, 0, st>>>(s, f.Lt, f.Ut, f.DinvL, f.DinvU);
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

// ---- selective inversion of the trailing dense block (host.hpp DT_*) ------
// M = (I + N)^{-1} for S = [s0, s0 + K): N = the row-scaled L~_SS (mode 0,
// strictly lower) or U~_SS (mode 1, strictly upper). One CTA per block column
// k walks its rows in dependency order, M(i,k) = -sum_j N(i,j) M(j,k) with
// M(k,k) = I, on DMMA in a fixed order. tab[a*K + b] (a > b) = tile id of
// L(s0+a, s0+b) (= of U(s0+b, s0+a)); out at strict index a(a-1)/2 + b with
// (a, b) = (larger, smaller) block index.
constexpr int SELINV_SMEM = (TT + XS2) * static_cast<int>(sizeof(cd));
__device__ __forceinline__ size_t sel_sidx(int a, int b) { return static_cast<size_t>(a) * (a - 1) / 2 + b; }
__device__ __forceinline__ size_t sel_didx(int a, int b) { return static_cast<size_t>(a) * (a + 1) / 2 + b; }

__device__ __forceinline__ void identity_x32(cd* xs) {
  for (int e = threadIdx.x; e < XS2; e += ST) {
    const int col = e / XPAD, row = e % XPAD;
    xs[e] = mk(col == row ? 1.0 : 0.0, 0.0);
  }
}

__device__ __forceinline__ void store_tile_acc(const Acc8& acc, const Frag& f, cd* dst, double sign) {
  cd o[4];
  acc8_fold(acc, o);
#pragma unroll
  for (int q = 0; q < 4; ++q) dst[ocol(f, q) * TILE + f.row] = cscale(o[q], sign);
}

__global__ void __launch_bounds__(ST) selinv_kernel(int mode, int K, const int* tab, const cd* N, cd* out) {
  extern __shared__ __align__(16) unsigned char sel_smem[];
  cd* ts = reinterpret_cast<cd*>(sel_smem);
  cd* xs = ts + TT;
  const int k = blockIdx.x;
  const Frag f = frag();
  const unsigned long long pol = l2_evict_normal();
  const int nsteps = mode == 0 ? K - 1 - k : k;
  for (int s = 0; s < nsteps; ++s) {
    const int i = mode == 0 ? k + 1 + s : k - 1 - s;
    Acc8 acc;
    acc8_zero(acc);
    const int nj = mode == 0 ? i - k : k - i;
    for (int q = 0; q < nj; ++q) {
      const int j = mode == 0 ? k + q : k - q;
      const int tid = mode == 0 ? tab[i * K + j] : tab[j * K + i];
      load_tile_sw(ts, N + static_cast<size_t>(tid) * TT, pol);
      if (j == k)
        identity_x32(xs);
      else
        load_x32(xs, out + (mode == 0 ? sel_sidx(j, k) : sel_sidx(k, j)) * TT, TILE, 0, TILE, pol);
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
      mma_tile2(acc, ts, xs, false, false, f, 0xffu);
      __syncthreads();
    }
    store_tile_acc(acc, f, out + (mode == 0 ? sel_sidx(i, k) : sel_sidx(k, i)) * TT, -1.0);
    __threadfence();  // this column's later steps read the tile back through L2
    __syncthreads();
  }
}

// Backward-sweep tiles of S, index a(a+1)/2 + b (a >= b), from the strict inverses:
// mode 0: W(b, a) = MU(b, a) DinvU_a (MU(a, a) = I), MU(b, a) stored at sel_sidx(a, b);
// mode 1: X(a, b) = DinvU_a ML(a, b) (ML(a, a) = I), ML(a, b) stored at sel_sidx(a, b).
__global__ void __launch_bounds__(ST) selinv_post_kernel(int mode, int s0, const cd* DinvU, const cd* M, cd* out) {
  extern __shared__ __align__(16) unsigned char sel_smem[];
  cd* ts = reinterpret_cast<cd*>(sel_smem);
  cd* xs = ts + TT;
  const int p = blockIdx.x;
  int a = static_cast<int>((sqrt(8.0 * p + 1.0) - 1.0) * 0.5);
  while (static_cast<int64_t>(a + 1) * (a + 2) / 2 <= p) ++a;
  while (static_cast<int64_t>(a) * (a + 1) / 2 > p) --a;
  const int b = p - a * (a + 1) / 2;
  const cd* D = DinvU + static_cast<size_t>(s0 + a) * TT;
  cd* dst = out + static_cast<size_t>(p) * TT;
  if (a == b) {
    for (int e = threadIdx.x; e < TT; e += ST) dst[e] = D[e];
    return;
  }
  const cd* Mt = M + sel_sidx(a, b) * TT;
  const unsigned long long pol = l2_evict_normal();
  const Frag f = frag();
  load_tile_sw(ts, mode == 0 ? Mt : D, pol);
  load_x32(xs, mode == 0 ? D : Mt, TILE, 0, TILE, pol);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  Acc8 acc;
  acc8_zero(acc);
  mma_tile2(acc, ts, xs, false, false, f, 0xffu);
  store_tile_acc(acc, f, dst, 1.0);
}

void selinv(cudaStream_t st, int K, int s0, const int* tab, const SpFactor& f, cd* ML, cd* MU, cd* WU, cd* WX) {
  if (K < 2) return;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(selinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SELINV_SMEM);
    cudaFuncSetAttribute(selinv_post_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SELINV_SMEM);
    attr = true;
  }
  selinv_kernel<<<K, ST, SELINV_SMEM, st>>>(0, K, tab, f.Lt, ML);
  selinv_kernel<<<K, ST, SELINV_SMEM, st>>>(1, K, tab, f.Ut, MU);
  const unsigned npair = static_cast<unsigned>(K) * (K + 1) / 2;
  selinv_post_kernel<<<npair, ST, SELINV_SMEM, st>>>(0, s0, f.DinvU, MU, WU);
  if (WX) selinv_post_kernel<<<npair, ST, SELINV_SMEM, st>>>(1, s0, f.DinvU, ML, WX);
}

void swizzle_tiles(cudaStream_t st, cd* tiles, int64_t ntiles) {
  if (ntiles > 0) swizzle_tile_kernel<<<static_cast<unsigned>(ntiles), 256, 0, st>>>(tiles);
}

void tile_masks(cudaStream_t st, const cd* tiles, int64_t ntiles, uint2* masks) {
  if (ntiles > 0) tile_mask_kernel<<<static_cast<unsigned>(ntiles), 256, 0, st>>>(tiles, masks);
}

void factor_scatter(cudaStream_t st, const BandGeom& g, const FactorTiles& f, int64_t nnz, const int* e_row,
                    const int* e_col, const double* a_val, const double* b_val, int cx, double sig_re,
                    double sig_im, double* row_norm) {
  const size_t bytes = g.tiles_per_array() * TT * sizeof(cd);
  cudaMemsetAsync(f.Lt, 0, bytes, st);
  cudaMemsetAsync(f.Ut, 0, bytes, st);
  cudaMemsetAsync(row_norm, 0, sizeof(double) * g.npad, st);
  const int64_t total = nnz + (g.npad - g.n);
  const int threads = 256;
  const int64_t blocks = (total + threads - 1) / threads;
  if (blocks > 0)
    scatter_kernel<<<static_cast<unsigned>(blocks), threads, 0, st>>>(
        g, f.Lt, f.Ut, nnz, e_row, e_col, a_val, b_val, cx, sig_re, sig_im,
        reinterpret_cast<unsigned long long*>(row_norm));
}

void factor_run(cudaStream_t st, const BandGeom& g, const FactorTiles& f, const double* row_norm,
                FactorDevState ds, int cx) {
  constexpr int diag_smem = (3 * TILE * TPAD + 2 * 4 * TILE) * sizeof(cd);
  static bool diag_attr = false;
  if (!diag_attr) {
    cudaFuncSetAttribute(diag_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, diag_smem);
    diag_attr = true;
  }
  for (int k = 0; k < g.nbk; ++k) {
    diag_factor_kernel<<<1, FT, diag_smem, st>>>(g.n, k, f.Lt + lt_off(k, 0, g.J), f.DinvL, f.DinvU, row_norm, ds.fail_index,
                                                 ds.min_ratio_bits);
    if (k + 1 < g.nbk && g.J > 0) {
      panel_kernel<<<2 * g.J, FT, 0, st>>>(g, k, f.Lt, f.Ut, f.DinvL, f.DinvU);
      trailing_kernel<<<dim3(g.J, g.J), FT, 0, st>>>(g, k, f.Lt, f.Ut);
    }
  }
  if (g.J > 0) scale_tiles_kernel<<<dim3(g.nbk, g.J, 2), FT, 0, st>>>(g, f);
}

}  // namespace zolo

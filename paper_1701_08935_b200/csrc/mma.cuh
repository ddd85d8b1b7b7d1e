// Shared FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) tile helpers for the
// sweeps (trsm.cu) and the level-scheduled factorization (factor.cu).
//
// A CTA of ST = 256 threads (8 warps) computes a 32 x 32 complex output
// block; tiles are staged in shared memory XOR-swizzled (load_tile_sw), the
// right operand column-padded [col*XPAD + k] (load_x32).
#pragma once

#include "common.cuh"

namespace zolo {
namespace {

constexpr int ST = 256;         // threads per CTA (8 warps)
constexpr int XPAD = TILE + 4;  // x column stride: B fragment loads conflict free
constexpr int DCG = 32;         // columns per DAG task / output block
constexpr int XS2 = DCG * XPAD; // padded 32 x 32 x block

// Per-thread ownership of the 32 x 16 complex output block: warp w holds rows
// 8 ((w%4) ^ 2 (w/4)) + lane/4 and columns 8 (w/4) + 2 (lane%4) + {0,1}.
struct Frag {
  int row, col;  // first of the two owned (row, col), (row, col+1)
  int r0, c0;    // warp block origin
  int lane;
};
__device__ __forceinline__ Frag frag() {
  Frag f;
  const int w = threadIdx.x >> 5;
  f.lane = threadIdx.x & 31;
  // warps w and w + 4 share an SM sub-partition (DMMA pipe): give them row groups g and g ^ 2, so
  // a tile whose nonzeros sit in some row groups (occupancy masks) still spreads over all pipes
  f.r0 = 8 * ((w & 3) ^ ((w >> 1) & 2));
  f.c0 = 8 * ((w >> 2) & 1);
  f.row = f.r0 + (f.lane >> 2);
  f.col = f.c0 + 2 * (f.lane & 3);
  return f;
}

// Swizzled tile layout: element (row, col) of a 32 x 32 tile at
// col*32 + (row ^ swz(col)), swz(c) = 4 (c&1) + 2 ((c>>1)&1). Both fragment
// patterns -- op N reads T(ar, k), op H reads T(k, ar), with ar = lane/4 and
// k = lane%4 (+ block offsets) -- hit 8 distinct 16-byte bank groups per
// quarter warp, so the conjugate-transposed chains are conflict free too, and
// the tile needs no padding.
__device__ __forceinline__ int swz(int c) { return ((c & 1) << 2) | (c & 2); }

__device__ __forceinline__ void load_tile_sw(cd* s, const cd* g, unsigned long long pol) {
#pragma unroll
  for (int q = 0; q < TT / ST; ++q) {
    const int e = threadIdx.x + q * ST;
    const int col = e / TILE, row = e % TILE;
    cp_async16_cg_hint(&s[col * TILE + (row ^ swz(col))], g + e, pol);
  }
}

// the same without an L2 policy (plain cp.async)
__device__ __forceinline__ void load_tile_sw(cd* s, const cd* g) {
#pragma unroll
  for (int q = 0; q < TT / ST; ++q) {
    const int e = threadIdx.x + q * ST;
    const int col = e / TILE, row = e % TILE;
    cp_async16_cg(&s[col * TILE + (row ^ swz(col))], g + e);
  }
}

// non-volatile DMMA: lets the scheduler interleave independent accumulators
__device__ __forceinline__ void dmma_nv(double c[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// Per-thread ownership of a 32 x 32 complex output block: warp w holds rows
// 8 (w%4) + lane/4 and columns 8 (w/4) + 2 (lane%4) + {0,1} (+16 for the
// second block), i.e. two 8x8 DMMA blocks that share their A fragments.
// DMMA accumulators live across tiles: acc8[h][p][ri][e] (half h, product part
// p: a.x or a.y products, re/im, element e) = 8 independent chains, folded once per task.
struct Acc8 {
  double v[2][2][2][2];
};
__device__ __forceinline__ void acc8_zero(Acc8& a) {
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
      for (int ri = 0; ri < 2; ++ri) a.v[h][p][ri][0] = a.v[h][p][ri][1] = 0.0;
}
// out[2h + e] = the complex output (row, ocol(2h + e))
__device__ __forceinline__ void acc8_fold(const Acc8& a, cd out[4]) {
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int e = 0; e < 2; ++e)
      out[2 * h + e] = mk(a.v[h][0][0][e] + a.v[h][1][0][e], a.v[h][0][1][e] + a.v[h][1][1][e]);
}

// km: the k-steps (4-column groups of op(T)) holding nonzeros in this warp's
// 8 rows (tile_mask_kernel); zero k-steps and all-zero row groups are skipped.
template <bool OPH, bool NEG>
__device__ __forceinline__ void mma_tile2_t(Acc8& acc, const cd* ts, const cd* xs, const Frag& f, unsigned km) {
  if (km == 0) return;
  // mma.sync.aligned needs a converged warp: callers branch on loop bounds the
  // compiler cannot prove warp-uniform, so reconverge explicitly
  __syncwarp();
  const int ar = f.r0 + (f.lane >> 2), am = f.lane & 3;
  const int bc = f.c0 + (f.lane >> 2);
  const int sa = swz(ar);
  cd a[TILE / 4], b0[TILE / 4], b1[TILE / 4];
#pragma unroll
  for (int kb = 0; kb < TILE / 4; ++kb) {
    const int k = 4 * kb + am;
    a[kb] = OPH ? ts[ar * TILE + (k ^ sa)] : ts[k * TILE + (ar ^ swz(k))];
    if (NEG) a[kb] = mk(-a[kb].x, -a[kb].y);
    b0[kb] = xs[bc * XPAD + k];
    b1[kb] = xs[(bc + 16) * XPAD + k];
  }
#pragma unroll
  for (int kb = 0; kb < TILE / 4; ++kb) {
    if (!((km >> kb) & 1u)) continue;
    // op N: re += ax bx - ay by, im += ax by + ay bx; op H (conj a): re += ax bx + ay by, im += ax by - ay bx.
    // The a.x products and the a.y products accumulate in separate chains (second index), so the
    // eight DMMAs of a k-step are independent: no DMMA waits on the one before it.
    const double ny = OPH ? a[kb].y : -a[kb].y;
    const double py = OPH ? -a[kb].y : a[kb].y;
    dmma_nv(acc.v[0][0][0], a[kb].x, b0[kb].x);
    dmma_nv(acc.v[1][0][0], a[kb].x, b1[kb].x);
    dmma_nv(acc.v[0][0][1], a[kb].x, b0[kb].y);
    dmma_nv(acc.v[1][0][1], a[kb].x, b1[kb].y);
    dmma_nv(acc.v[0][1][0], ny, b0[kb].y);
    dmma_nv(acc.v[1][1][0], ny, b1[kb].y);
    dmma_nv(acc.v[0][1][1], py, b0[kb].x);
    dmma_nv(acc.v[1][1][1], py, b1[kb].x);
  }
}

// acc += op(T) X, or -= with neg (the pre-transform entry)
__device__ __forceinline__ void mma_tile2(Acc8& acc, const cd* ts, const cd* xs, bool opH, bool neg, const Frag& f,
                                          unsigned km) {
  if (opH) {
    if (neg)
      mma_tile2_t<true, true>(acc, ts, xs, f, km);
    else
      mma_tile2_t<true, false>(acc, ts, xs, f, km);
  } else {
    if (neg)
      mma_tile2_t<false, true>(acc, ts, xs, f, km);
    else
      mma_tile2_t<false, false>(acc, ts, xs, f, km);
  }
}

// ---- 3M complex tile products (the sweeps) ---------------------------------
// A complex 8x8x4 product in three real DMMAs instead of four: with a = ar + i ai and
// b = br + i bi,  P1 = ar br,  P2 = ai bi,  P3 = (ar + ai)(br + bi),  a b = (P1 - P2) + i (P3 - P1 - P2).
// The conjugate transpose (op H) is the same with ai -> -ai. P1, P2, P3 accumulate over every
// tile of a task (fixed order) and are combined once per task (acc3_fold), so the extra
// additions are one per A and B fragment element per k-step -- 6 DMMAs + 3 adds per k-step for
// the two 8x8 output blocks instead of 8 DMMAs. The result is normwise as accurate as the
// 4-product form (each output is a sum of products bounded by |a||b|); only its rounding differs.
template <int NB>  // 8-column output blocks per warp (16 columns apart)
struct Acc3 {
  double p[NB][3][2];  // [block][P1 P2 P3][element]
};
template <int NB>
__device__ __forceinline__ void acc3_zero(Acc3<NB>& a) {
#pragma unroll
  for (int h = 0; h < NB; ++h)
#pragma unroll
    for (int k = 0; k < 3; ++k) a.p[h][k][0] = a.p[h][k][1] = 0.0;
}
// out[2h + e] = the complex output (row, ocol_sw(2h + e))
template <int NB>
__device__ __forceinline__ void acc3_fold(const Acc3<NB>& a, cd out[2 * NB]) {
#pragma unroll
  for (int h = 0; h < NB; ++h)
#pragma unroll
    for (int e = 0; e < 2; ++e)
      out[2 * h + e] = mk(a.p[h][0][e] - a.p[h][1][e], a.p[h][2][e] - a.p[h][0][e] - a.p[h][1][e]);
}
// acc += sg * block value (the add entries: b_i, partial sums), at output (row, ocol_sw(2h + e))
template <int NB>
__device__ __forceinline__ void acc3_add(Acc3<NB>& a, int h, int e, cd v, double sg) {
  a.p[h][0][e] += sg * v.x;          // Re = P1 - P2
  a.p[h][2][e] += sg * (v.x + v.y);  // Im = P3 - P1 - P2
}

// The sweeps' x block (32 columns x 32 rows) as the tensor copy lands it (trsm.cu tma_xblock,
// CU_TENSOR_MAP_SWIZZLE_128B): 128-byte lines of 8 complex rows, line = 32 (k / 8) + c, the
// 16-byte chunk index XORed with line % 8 = c % 8. The sweeps' warps map their DMMA column
// index n to column pcol(n) = n / 2 + 4 (n % 2) of their 8-column block, so the 8 lanes of a
// B-fragment quarter warp (n = 2j, 2j + 1 at 4 consecutive rows) read columns j and j + 4:
// 8 distinct chunks, conflict free without padding, and the address of a fragment is a per-lane
// base plus a compile-time offset (per k-step parity).
template <int XC>  // columns of the x block
__device__ __forceinline__ int xsw(int c, int k) { return 8 * (XC * (k >> 3) + c) + ((k & 7) ^ (c & 7)); }
__device__ __forceinline__ int pcol(int n) { return (n >> 1) + 4 * (n & 1); }
// output column of acc3 entry q (= 2h + e) within the 32-column group, sweeps' column map
__device__ __forceinline__ int ocol_sw(const Frag& f, int q) { return f.c0 + (f.lane & 3) + 4 * (q & 1) + 16 * (q >> 1); }

// Per-lane fragment offsets of the sweeps' tile products, computed once per kernel, so one code
// path serves all four (op N / op H) x (+ / -) products: tiles are XOR-swizzled (swz), x blocks
// 128-byte swizzled (xsw). A fragment (row ar, k = 4 kk + am): op N at an + 128 kk; op H
// (conjugate transpose) at ah[kk & 1] + 4 kk. B fragment (column bc, row k): xb[kk & 1] + 8 XC (kk / 2).
struct TileOff {
  int an, ah0, ah1, xb0, xb1;
};
template <int XC>
__device__ __forceinline__ TileOff tile_off(const Frag& f) {
  const int ar = f.r0 + (f.lane >> 2), am = f.lane & 3, sa = swz(ar);
  const int bc = f.c0 + pcol(f.lane >> 2);
  TileOff o;
  o.an = 32 * am + (ar ^ swz(am));
  const int t = 4 * (sa >> 2), h = 32 * ar + (am ^ (sa & 2));
  o.ah0 = h + t;
  o.ah1 = h - t;
  o.xb0 = 8 * bc + (am ^ (bc & 3)) + (bc & 4);
  o.xb1 = 8 * bc + (am ^ (bc & 3)) + (4 - (bc & 4));
  return o;
}
__device__ __forceinline__ double flip_sign(double v, int hi_mask) {
  return __hiloint2double(__double2hiint(v) ^ hi_mask, __double2loint(v));
}

// acc += op(T) X (3M), or -= with neg (the pre-transform entry); km: the unmasked k-steps of
// this warp's rows. op and sign are warp-uniform run-time values: the conjugation and the
// negation are sign flips of the A fragment (integer pipe), the transpose an offset pattern.
template <int XC, int NB>
__device__ __forceinline__ void mma_tile3(Acc3<NB>& acc, const cd* ts, const cd* xs, bool opH, bool neg,
                                          const TileOff& o, unsigned km) {
  if (km == 0) return;
  __syncwarp();  // mma.sync.aligned needs a converged warp
  const int a0 = opH ? o.ah0 : o.an, a1 = opH ? o.ah1 : o.an, ash = opH ? 2 : 7;
  const int mre = neg ? static_cast<int>(0x80000000u) : 0;
  const int mim = (neg != opH) ? static_cast<int>(0x80000000u) : 0;  // conj for op H, negated for the pre-transform
  constexpr int KG = 4;  // k-steps whose fragments are loaded together (the shared-memory latency overlaps)
#pragma unroll
  for (int k0 = 0; k0 < TILE / 4; k0 += KG) {  // fragments of KG k-steps first: the shared-memory latency overlaps
    cd a[KG], b[KG][NB];
#pragma unroll
    for (int q = 0; q < KG; ++q) {
      const int kk = k0 + q;
      a[q] = ts[((kk & 1) ? a1 : a0) + (kk << ash)];
      const int xo = ((kk & 1) ? o.xb1 : o.xb0) + 8 * XC * (kk >> 1);
#pragma unroll
      for (int h = 0; h < NB; ++h) b[q][h] = xs[xo + 128 * h];  // column bc + 16 h
    }
#pragma unroll
    for (int q = 0; q < KG; ++q) {
      if (!((km >> (k0 + q)) & 1u)) continue;  // predicated off: ~1 issue cycle instead of a DMMA
      const double re = flip_sign(a[q].x, mre);
      const double im = flip_sign(a[q].y, mim);
      const double s = re + im;
#pragma unroll
      for (int h = 0; h < NB; ++h) dmma_nv(acc.p[h][0], re, b[q][h].x);
#pragma unroll
      for (int h = 0; h < NB; ++h) dmma_nv(acc.p[h][1], im, b[q][h].y);
#pragma unroll
      for (int h = 0; h < NB; ++h) dmma_nv(acc.p[h][2], s, b[q][h].x + b[q][h].y);
    }
  }
}

// acc (3M) += T X for the factorization's trailing updates: T a swizzled tile (load_tile_sw),
// X a padded 32 x 32 block [col*XPAD + k] (load_x32), op N, all k-steps; outputs as mma_tile2
// (out[2h + e] at row f.row, column ocol(f, 2h + e)).
// km: the k-steps holding nonzeros in this warp's 8 rows of T (the others are predicated off)
__device__ __forceinline__ void mma_tile3_nx(Acc3<2>& acc, const cd* ts, const cd* xs, const Frag& f, unsigned km) {
  if (km == 0) return;
  __syncwarp();
  const int ar = f.r0 + (f.lane >> 2), am = f.lane & 3;
  const int bc = f.c0 + (f.lane >> 2);
  const int an = 32 * am + (ar ^ swz(am));
#pragma unroll
  for (int k0 = 0; k0 < TILE / 4; k0 += 4) {
    cd a[4], b0[4], b1[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int kk = k0 + q, k = 4 * kk + am;
      a[q] = ts[an + 128 * kk];
      b0[q] = xs[bc * XPAD + k];
      b1[q] = xs[(bc + 16) * XPAD + k];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (!((km >> (k0 + q)) & 1u)) continue;
      const double s = a[q].x + a[q].y;
      dmma_nv(acc.p[0][0], a[q].x, b0[q].x);
      dmma_nv(acc.p[1][0], a[q].x, b1[q].x);
      dmma_nv(acc.p[0][1], a[q].y, b0[q].y);
      dmma_nv(acc.p[1][1], a[q].y, b1[q].y);
      dmma_nv(acc.p[0][2], s, b0[q].x + b0[q].y);
      dmma_nv(acc.p[1][2], s, b1[q].x + b1[q].y);
    }
  }
}

// 32 rows x 32 columns of a column-major block into [col*XPAD + row].
__device__ __forceinline__ void load_x32(cd* xs, const cd* base, int64_t ld, int c0, int nc, unsigned long long pol) {
  const int row = threadIdx.x & 31, cc = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < DCG / 8; ++q) {
    const int c = cc + 8 * q;
    if (c < nc)
      cp_async16_cg_hint(&xs[c * XPAD + row], base + row + (c0 + c) * ld, pol);
    else
      xs[c * XPAD + row] = mk(0.0, 0.0);
  }
}

// all 32 columns, without an L2 policy (plain cp.async)
__device__ __forceinline__ void load_x32(cd* xs, const cd* base, int64_t ld, int c0) {
  const int row = threadIdx.x & 31, cc = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < DCG / 8; ++q) {
    const int c = cc + 8 * q;
    cp_async16_cg(&xs[c * XPAD + row], base + row + (c0 + c) * ld);
  }
}

// output column of acc[q] within the 32-column group
__device__ __forceinline__ int ocol(const Frag& f, int q) { return f.col + (q & 1) + 16 * (q >> 1); }


}  // namespace
}  // namespace zolo

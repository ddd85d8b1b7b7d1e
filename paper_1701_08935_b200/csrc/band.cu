// Numeric unpivoted block-band LU of P(A - sigma B)P^T and the multi-RHS
// wavefront triangular solves on it.
//
// Reference: factorize (band_factor.hpp:135-182) eliminates one column at a
// time with a rank-1 update of the trailing band; ShiftedFactor::solve /
// adjoint_solve (band_factor.hpp:53-117) sweep the band once per right-hand
// side column. Here both become sequences of dense TILE x TILE complex128
// tile products (see band.cuh for the layout):
//
//   factor step k:  diagonal tile LU + pivot monitor + triangular inverses
//                   -> panel tiles (x DinvU / DinvL) -> J x J trailing updates
//   solve sweep:    block row i: x_i = Dinv_i (b_i - sum_d T_(i,i-+d) x_(i-+d))
//                   for all r poles, both solve and adjoint chains and all
//                   column groups of the block in ONE persistent launch; the
//                   cross-block dependency is a per-(chain, group, block)
//                   epoch flag (release/acquire), tasks are claimed in
//                   dependency order from an atomic counter so any grid size
//                   is deadlock free.
#include <cuda_runtime.h>
#include <stdio.h>

#include <algorithm>

#include "band.cuh"

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
// inverses of its unit-lower and upper triangles.
__global__ void __launch_bounds__(FT) diag_factor_kernel(BandGeom g, int k, cd* Lt, cd* DinvL, cd* DinvU,
                                                         const double* row_norm, int* fail_index,
                                                         unsigned long long* min_ratio_bits) {
  __shared__ cd D[TILE * TPAD];
  cd* tile = Lt + lt_off(k, 0, g.J);
  load_tile_async(D, tile);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  const int t = threadIdx.x;
  for (int p = 0; p < TILE; ++p) {
    const cd piv = D[p * TPAD + p];
    const cd inv = cdiv(mk(1.0, 0.0), piv);
    if (t == 0) {
      const int64_t gi = static_cast<int64_t>(k) * TILE + p;
      if (gi < g.n) {
        const double rn = row_norm[gi];
        const double ap = hypot(piv.x, piv.y);
        const double ratio = ap / fmax(rn, 1e-300);
        atomicMin(min_ratio_bits, static_cast<unsigned long long>(__double_as_longlong(ratio)));
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
  for (int q = 0; q < TT / FT; ++q) {
    const int e = t + q * FT;
    tile[e] = D[(e / TILE) * TPAD + (e % TILE)];
  }
  // inverses: thread c < 32 -> column c of L^{-1}; 32 <= t < 64 -> column of U^{-1}
  if (t < TILE) {
    const int c = t;
    cd x[TILE];
#pragma unroll
    for (int i = 0; i < TILE; ++i) x[i] = mk(i == c ? 1.0 : 0.0, 0.0);
#pragma unroll
    for (int i = 0; i < TILE; ++i) {
      if (i > c) {
        cd s = x[i];
        for (int kk = c; kk < i; ++kk) s = csub(s, cmul(D[kk * TPAD + i], x[kk]));
        x[i] = s;
      }
    }
    cd* out = DinvL + static_cast<size_t>(k) * TT;
#pragma unroll
    for (int i = 0; i < TILE; ++i) out[c * TILE + i] = x[i];
  } else if (t < 2 * TILE) {
    const int c = t - TILE;
    cd x[TILE];
#pragma unroll
    for (int i = 0; i < TILE; ++i) x[i] = mk(0.0, 0.0);
#pragma unroll
    for (int ii = TILE - 1; ii >= 0; --ii) {
      if (ii <= c) {
        cd s = mk(ii == c ? 1.0 : 0.0, 0.0);
        for (int kk = ii + 1; kk <= c; ++kk) s = csub(s, cmul(D[kk * TPAD + ii], x[kk]));
        x[ii] = cdiv(s, D[ii * TPAD + ii]);
      }
    }
    cd* out = DinvU + static_cast<size_t>(k) * TT;
#pragma unroll
    for (int i = 0; i < TILE; ++i) out[c * TILE + i] = x[i];
  }
}

// Panel: L(k+d,k) = A(k+d,k) U_kk^{-1} (blocks 0..J-1),
//        U(k,k+d) = L_kk^{-1} A(k,k+d) (blocks J..2J-1).
__global__ void __launch_bounds__(FT) panel_kernel(BandGeom g, int k, cd* Lt, cd* Ut, const cd* DinvL,
                                                   const cd* DinvU) {
  __shared__ cd As[TILE * TPAD];
  __shared__ cd Bs[TILE * TPAD];
  const int J = g.J;
  const bool lower = blockIdx.x < J;
  const int d = lower ? blockIdx.x + 1 : blockIdx.x - J + 1;
  if (k + d >= g.nbk) return;
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
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  c[ty * TILE + tx] = out[0];
  c[(ty + 16) * TILE + tx] = out[1];
  c[ty * TILE + tx + 16] = out[2];
  c[(ty + 16) * TILE + tx + 16] = out[3];
}

// Trailing update A(k+a, k+b) -= L(k+a, k) U(k, k+b), a, b in 1..J.
__global__ void __launch_bounds__(FT) trailing_kernel(BandGeom g, int k, cd* Lt, cd* Ut) {
  __shared__ cd As[TILE * TPAD];
  __shared__ cd Bs[TILE * TPAD];
  const int J = g.J;
  const int a = blockIdx.x + 1, b = blockIdx.y + 1;
  if (k + a >= g.nbk || k + b >= g.nbk) return;
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
  c[ty * TILE + tx] = csub(c0, out[0]);
  c[(ty + 16) * TILE + tx] = csub(c1, out[1]);
  c[ty * TILE + tx + 16] = csub(c2, out[2]);
  c[(ty + 16) * TILE + tx + 16] = csub(c3, out[3]);
}

// ---------------------------------------------------------------------------
// wavefront multi-RHS triangular solve
// ---------------------------------------------------------------------------
constexpr int ST = 256;                      // solve threads per CTA (8 warps)
constexpr int TILE_S = TILE * TPAD;          // padded tile (complex)
constexpr int XS = CG * TPAD;                // padded x block [c*TPAD + k]
constexpr int SOLVE_SMEM = (2 * TILE_S + 2 * XS + TILE_S + XS) * sizeof(cd);

struct SolveArgs {
  const Chain* chains;
  int nchains, ngroups, ncols, nbk, J, epoch, fwd;
  int64_t ld;
  int* flags;
  int* counter;
};

// Thread (r = 4 w + lane/8, kq = lane%8) holds op(T)(r, kq + 8 kk), kk < 4.
__device__ __forceinline__ void solve_accumulate(cd part[CG], const cd* ts, const cd* xs, bool opH, int r, int kq) {
  cd a[4];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const int k = kq + 8 * kk;
    a[kk] = opH ? cconj(ts[r * TPAD + k]) : ts[k * TPAD + r];
  }
#pragma unroll
  for (int c = 0; c < CG; ++c) {
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) cfma(part[c], a[kk], xs[c * TPAD + kq + 8 * kk]);
  }
}

// Reduce-scatter part[16] over the 8 kq lanes: lane kq ends with the full
// sums of columns 2kq, 2kq+1 in out[0..1].
__device__ __forceinline__ void reduce_scatter8(const cd part[CG], cd out[2], int kq) {
  cd k8[8], k4[4];
  const bool b2 = kq & 4, b1 = kq & 2, b0 = kq & 1;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const cd send = b2 ? part[q] : part[8 + q];
    const cd keep = b2 ? part[8 + q] : part[q];
    cd rv;
    rv.x = __shfl_xor_sync(0xffffffffu, send.x, 4);
    rv.y = __shfl_xor_sync(0xffffffffu, send.y, 4);
    k8[q] = cadd(keep, rv);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const cd send = b1 ? k8[q] : k8[4 + q];
    const cd keep = b1 ? k8[4 + q] : k8[q];
    cd rv;
    rv.x = __shfl_xor_sync(0xffffffffu, send.x, 2);
    rv.y = __shfl_xor_sync(0xffffffffu, send.y, 2);
    k4[q] = cadd(keep, rv);
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const cd send = b0 ? k4[q] : k4[2 + q];
    const cd keep = b0 ? k4[2 + q] : k4[q];
    cd rv;
    rv.x = __shfl_xor_sync(0xffffffffu, send.x, 1);
    rv.y = __shfl_xor_sync(0xffffffffu, send.y, 1);
    out[q] = cadd(keep, rv);
  }
}

__device__ __forceinline__ void load_x_async(cd* xs, const cd* base, int64_t ld, int c0, int nc) {
  // 32 rows x CG columns; thread t -> row t%32, columns t/32 + 8 q
  const int row = threadIdx.x & 31, cc = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < CG / 8; ++q) {
    const int c = cc + 8 * q;
    if (c < nc)
      cp_async16_cg(&xs[c * TPAD + row], base + row + (c0 + c) * ld);
    else
      xs[c * TPAD + row] = mk(0.0, 0.0);
  }
}

__device__ __forceinline__ void load_tile_solve(cd* s, const cd* gtile) {
#pragma unroll
  for (int q = 0; q < TT / ST; ++q) {
    const int e = threadIdx.x + q * ST;
    cp_async16_cg(&s[(e / TILE) * TPAD + (e % TILE)], gtile + e);
  }
}

__global__ void __launch_bounds__(ST, 2) trsm_kernel(SolveArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cd* tile_s[2] = {reinterpret_cast<cd*>(smem_raw), reinterpret_cast<cd*>(smem_raw) + TILE_S};
  cd* x_s[2] = {reinterpret_cast<cd*>(smem_raw) + 2 * TILE_S, reinterpret_cast<cd*>(smem_raw) + 2 * TILE_S + XS};
  cd* dinv_s = reinterpret_cast<cd*>(smem_raw) + 2 * TILE_S + 2 * XS;
  cd* acc_s = dinv_s + TILE_S;
  __shared__ int task_s;

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r = 4 * w + (lane >> 3), kq = lane & 7;
  const int per_step = A.nchains * A.ngroups;
  const int ntasks = A.nbk * per_step;
  const int J = A.J;

  for (;;) {
    if (threadIdx.x == 0) task_s = atomicAdd(A.counter, 1);
    __syncthreads();
    const int t = task_s;
    __syncthreads();
    if (t >= ntasks) break;
    const int s = t / per_step, rem = t % per_step;
    const int ci = rem / A.ngroups, gi = rem % A.ngroups;
    const Chain ch = A.chains[ci];
    const bool fwd = A.fwd != 0;
    const bool opH = ch.mode == FWD_UH || ch.mode == BWD_LH;
    const int i = fwd ? s : A.nbk - 1 - s;
    const int c0 = gi * CG;
    const int nc = min(CG, A.ncols - c0);
    int* flags = A.flags + (static_cast<size_t>(ci) * A.ngroups + gi) * A.nbk;
    const int dmax = fwd ? min(J, i) : min(J, A.nbk - 1 - i);
    const int64_t ld = A.ld;

    // diagonal inverse (no dependency) + right-hand side of this block row
    load_tile_solve(dinv_s, ch.dinv + static_cast<size_t>(i) * TT);
    cd bval[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int c = 2 * kq + q;
      bval[q] = (c < nc) ? ch.src[static_cast<int64_t>(i) * TILE + r + (c0 + c) * ld] : mk(0.0, 0.0);
    }
    cd part[CG];
#pragma unroll
    for (int c = 0; c < CG; ++c) part[c] = mk(0.0, 0.0);

    auto dep = [&](int d) { return fwd ? i - d : i + d; };
    auto tile_ptr = [&](int d) -> const cd* {
      // FWD_*: T(i, i-d) from row i's slot d; BWD_*: T(i, i+d) from row i+d's slot d
      const int base = fwd ? i : i + d;
      return ch.off + lt_off(base, d, J);
    };
    auto wait_flag = [&](int j) {
      if (threadIdx.x == 0) {
        const int* f = flags + j;
        int spins = 0;
        while (ld_acquire(f) < A.epoch) {
          // bounded wait: a missing producer is reported, never a hung GPU
          if (++spins > 256) __nanosleep(64);
          if (spins > (1 << 25)) {
            atomicExch(A.counter + 2, 1);
            break;
          }
        }
      }
      __syncthreads();
    };

    if (dmax >= 1) {
      load_tile_solve(tile_s[0], tile_ptr(dmax));
      wait_flag(dep(dmax));
      load_x_async(x_s[0], ch.dst + static_cast<int64_t>(dep(dmax)) * TILE, ld, c0, nc);
    }
    cp_async_commit();
    int cur = 0;
    for (int d = dmax; d >= 1; --d) {
      const int nd = d - 1;
      const int nxt = cur ^ 1;
      if (nd >= 2) {  // far dependency: almost always complete, prefetch fully
        load_tile_solve(tile_s[nxt], tile_ptr(nd));
        wait_flag(dep(nd));
        load_x_async(x_s[nxt], ch.dst + static_cast<int64_t>(dep(nd)) * TILE, ld, c0, nc);
      } else if (nd == 1) {
        load_tile_solve(tile_s[nxt], tile_ptr(nd));
      }
      cp_async_commit();
      cp_async_wait<1>();
      __syncthreads();
      solve_accumulate(part, tile_s[cur], x_s[cur], opH, r, kq);
      __syncthreads();
      if (nd == 1) {  // the critical dependency (block i -+ 1): wait as late as possible
        wait_flag(dep(1));
        load_x_async(x_s[nxt], ch.dst + static_cast<int64_t>(dep(1)) * TILE, ld, c0, nc);
        cp_async_commit();
      }
      cur = nxt;
    }
    cp_async_wait<0>();
    __syncthreads();
    // acc = b - sum_d T x_d
    cd red[2];
    reduce_scatter8(part, red, kq);
#pragma unroll
    for (int q = 0; q < 2; ++q) acc_s[(2 * kq + q) * TPAD + r] = csub(bval[q], red[q]);
    __syncthreads();
    // x_i = op(Dinv_i) acc
#pragma unroll
    for (int c = 0; c < CG; ++c) part[c] = mk(0.0, 0.0);
    solve_accumulate(part, dinv_s, acc_s, opH, r, kq);
    reduce_scatter8(part, red, kq);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 2; ++q) acc_s[(2 * kq + q) * TPAD + r] = red[q];
    __syncthreads();
    {
      const int row = threadIdx.x & 31, cc = threadIdx.x >> 5;
#pragma unroll
      for (int q = 0; q < CG / 8; ++q) {
        const int c = cc + 8 * q;
        if (c < nc) ch.dst[static_cast<int64_t>(i) * TILE + row + (c0 + c) * ld] = acc_s[c * TPAD + row];
      }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) st_release(flags + i, A.epoch);
  }
}

}  // namespace

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
                FactorDevState ds) {
  for (int k = 0; k < g.nbk; ++k) {
    diag_factor_kernel<<<1, FT, 0, st>>>(g, k, f.Lt, f.DinvL, f.DinvU, row_norm, ds.fail_index,
                                         ds.min_ratio_bits);
    if (k + 1 < g.nbk && g.J > 0) {
      panel_kernel<<<2 * g.J, FT, 0, st>>>(g, k, f.Lt, f.Ut, f.DinvL, f.DinvU);
      trailing_kernel<<<dim3(g.J, g.J), FT, 0, st>>>(g, k, f.Lt, f.Ut);
    }
  }
}

void trsm_launch(cudaStream_t st, const BandGeom& g, const Chain* d_chains, int nchains, int ncols, int64_t ld,
                 int* flags, int epoch, int* task_counter, int fwd, int num_sms) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SOLVE_SMEM);
    attr_set = true;
  }
  SolveArgs a;
  a.chains = d_chains;
  a.nchains = nchains;
  a.ngroups = (ncols + CG - 1) / CG;
  a.ncols = ncols;
  a.nbk = g.nbk;
  a.J = g.J;
  a.epoch = epoch;
  a.fwd = fwd;
  a.ld = ld;
  a.flags = flags;
  a.counter = task_counter;
  cudaMemsetAsync(task_counter, 0, sizeof(int), st);
  const int ntasks = g.nbk * nchains * a.ngroups;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, trsm_kernel, ST, SOLVE_SMEM);
  if (per_sm < 1) per_sm = 1;
  const int grid = std::min(ntasks, num_sms * per_sm);
  if (grid > 0) trsm_kernel<<<grid, ST, SOLVE_SMEM, st>>>(a);
}

}  // namespace zolo

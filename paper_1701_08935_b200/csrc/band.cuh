// Block-band storage of the unpivoted LU of P (A - sigma B) P^T.
//
// The reference stores the band column-contiguously as
// band[j(2bw+1) + bw + i - j] (band_factor.hpp:37-43) and eliminates one
// column at a time (band_factor.hpp:158-177). Here the same band is cut into
// TILE x TILE complex128 tiles so that every elimination step and every
// triangular-solve step is a dense tile product:
//
//   Lt[i][d]  = block (i, i-d) of L,  d = 0..J   (d = 0 holds the packed
//               unit-L / U diagonal block, LAPACK style)
//   Ut[j][d]  = block (j-d, j) of U,  d = 1..J   (slot d = 0 unused)
//   DinvL[i]  = inverse of the unit lower triangle of the diagonal block
//   DinvU[i]  = inverse of its upper triangle
//   MF/MB/MFH/MBH[i] = the next-neighbour couplings premultiplied by the
//               diagonal inverse (see trsm below), so that the critical chain
//               of a sweep is one tile product per block row
//
// J = ceil(bw / TILE) is the block half-bandwidth; rows beyond n are padded
// with identity rows so every tile is full. Elimination without pivoting
// never fills outside the envelope of the (symmetric) pattern, so block row i
// only holds dl[i] = i - (first nonzero block column of row i) off-diagonal
// L tiles, and block column i of U the same count: all other tiles are exact
// zeros and are skipped by the factorization and the solves.
#pragma once

#include <vector>

#include "common.cuh"
#include "host.hpp"

namespace zolo {

struct BandGeom {
  int64_t n = 0;           // matrix order
  int64_t npad = 0;        // nbk * TILE
  int nbk = 0;             // block rows
  int J = 0;               // block half-bandwidth (max over rows of dl)
  int64_t bw = 0;          // scalar half-bandwidth
  const int* dl = nullptr; // device: off-diagonal tiles per block row (envelope)
  size_t tiles_per_array() const { return static_cast<size_t>(nbk) * (J + 1); }
};

// After factor_run the off-diagonal tiles are ROW-SCALED by the diagonal-block
// inverses: Lt[i][d] = DinvL[i] L(i,i-d), Ut[j][d] = DinvU[j-d] U(j-d,j).
struct FactorTiles {
  cd* Lt = nullptr;
  cd* Ut = nullptr;
  cd* DinvL = nullptr;
  cd* DinvU = nullptr;
  // block-sparse path: occupancy masks of each array (tile_masks); nullptr for the band
  uint2* mLt = nullptr;
  uint2* mUt = nullptr;
  uint2* mDL = nullptr;
  uint2* mDU = nullptr;
  bool swz = false;  // Lt, Ut, DinvL, DinvU stored in the swizzled sweep layout (swizzle_tiles)
  // selectively inverted trailing block (selinv; host.hpp DT_*), swizzled like the rest
  cd* ML = nullptr;
  cd* MU = nullptr;
  cd* WU = nullptr;
  cd* WX = nullptr;
};

__host__ __device__ inline size_t lt_off(int i, int d, int J) {
  return (static_cast<size_t>(i) * (J + 1) + d) * TT;
}

// Triangular-solve traversal kinds (see band.cu).
enum SweepMode : int {
  FWD_L = 0,   // L y = b           (solve, band_factor.hpp:62-69)
  BWD_U = 1,   // U x = y           (solve, band_factor.hpp:71-80)
  FWD_UH = 2,  // U^H y = b         (adjoint_solve, band_factor.hpp:98-105)
  BWD_LH = 3   // L^H x = y         (adjoint_solve, band_factor.hpp:107-112)
};

// One triangular sweep over row-scaled tiles T~ (op N, or op H for the
// adjoint sweeps): u_i = pre(b_i) - sum_d op(T~_(i,i-+d)) u_(i-+d), where
// pre = op(Dinv_i) or the identity. For the adjoint sweeps u is the
// diagonally transformed unknown (z = U_ii^H y, w = L_ii^H x, see trsm.cu).
struct Chain {
  const cd* off;   // row-scaled Lt or Ut array of the pole
  const cd* pre;   // DinvL / DinvU applied to b_i first, or nullptr (identity)
  const uint2* offm;  // occupancy masks of off (block-sparse path; nullptr = dense)
  const uint2* prem;  // occupancy masks of pre
  const cd* src;   // right-hand side (ld x ncols), read once per block row
  cd* dst;         // solution (ld x ncols), written in place
  cd* cbuf;        // helper -> owner partial solutions c_i (ld x ncols)
  int mode;
  int pad;
  const cd* minv;  // selectively inverted trailing block (forward: M tiles, backward: W tiles), or nullptr
};

struct FactorDevState {
  int* fail_index;                    // first rejected pivot (device, -1 = none)
  unsigned long long* min_ratio_bits; // min |pivot|/||row|| as double bits
};

void factor_scatter(cudaStream_t st, const BandGeom& g, const FactorTiles& f, int64_t nnz, const int* e_row,
                    const int* e_col, const double* a_val, const double* b_val, int cx, double sig_re,
                    double sig_im, double* row_norm);
void factor_run(cudaStream_t st, const BandGeom& g, const FactorTiles& f, const double* row_norm,
                FactorDevState ds, int cx);

// ---- block-sparse factors (any node ordering; host symbolic.cpp) ----------
// Off-diagonal tile ids are row-major slots: row i's tiles (i, row_idx[e]),
// e in [row_ptr[i], row_ptr[i+1]) ascending; column k's structural rows
// col_idx[e] (ascending) carry their tile id in col_tile[e]; tile_row[e] = i.
// L(i,k) lives in Lt[id], U(k,i) in Ut[id]; diagonal blocks in Dt.
struct SpGeom {
  int64_t n = 0, npad = 0;
  int nb = 0;
  int64_t ntiles = 0;
  int max_deps = 0;
  const int* row_ptr = nullptr;
  const int* row_idx = nullptr;
  const int* col_ptr = nullptr;
  const int* col_idx = nullptr;
  const int* col_tile = nullptr;
  const int* tile_row = nullptr;
};

struct SpFactor {
  cd* Dt = nullptr;
  cd* Lt = nullptr;
  cd* Ut = nullptr;
  cd* DinvL = nullptr;
  cd* DinvU = nullptr;
};

// device copy of a FactorPlan (host.hpp): level ranges stay on the host
struct FactorPlanDev {
  const std::vector<int>* lvl_ptr = nullptr;
  const std::vector<int>* pan_ptr = nullptr;
  const std::vector<int>* tgt_ptr = nullptr;
  const int* cols = nullptr;
  const int* pan = nullptr;
  const int* tgt = nullptr;
  const int* con = nullptr;
  int simt = 0;  // (debug) SIMT trailing updates
};
// plan == nullptr: the column-serial right-looking loop (3 launches per block column)
void sp_factor(cudaStream_t st, const SpGeom& s, const std::vector<int>& col_cnt, const SpFactor& f, int64_t nnz,
               const int* e_row, const int* e_col, const double* a_val, const double* b_val, int cx, double sig_re,
               double sig_im, double* row_norm, const int* pad_rows, int npad_rows, FactorDevState ds, int* err,
               const FactorPlanDev* plan = nullptr);

// masks[t] = occupancy of tile t: bit (8 g + kb) of .x for rows 8g.. x cols 4kb..
// (op N), of .y for the conjugate transpose (factor.cu tile_mask_kernel).
void tile_masks(cudaStream_t st, const cd* tiles, int64_t ntiles, uint2* masks);
// tiles permuted in place into the sweep layout: element (row, col) at col*32 + (row ^ swz(col))
void swizzle_tiles(cudaStream_t st, cd* tiles, int64_t ntiles);
// selective inversion of the trailing dense block [s0, s0 + K) of the row-scaled factors (before
// swizzling): ML = (I + L~_SS)^-1, MU = (I + U~_SS)^-1 (strict parts, index a(a-1)/2 + b, a > b);
// WU(b,a) = MU(b,a) DinvU_a and (WX != nullptr) WX(a,b) = DinvU_a ML(a,b), index a(a+1)/2 + b, a >= b.
// tab[a*K + b] (a > b): tile id of L(s0+a, s0+b).
void selinv(cudaStream_t st, int K, int s0, const int* tab, const SpFactor& f, cd* ML, cd* MU, cd* WU, cd* WX);
// number of pivots (diagonal of the packed diagonal-tile LUs) with negative real part
int64_t count_negative_pivots(cudaStream_t st, const cd* dt, int nb);

// DAG-scheduled sweeps over block-sparse row-scaled tiles: the claim-ordered
// schedule (host.hpp dag_schedule, nsched entries) expanded over (chain,
// column group). Chunk tasks write partial sums into the chains' cbuf
// (leading dimension ldp = 32 * nslots) and release cflags[(chain, group, slot)].
// Task record (ints): [i, nd, pa, pc, out, 0, 0, 0, (j, tile id) x nd];
// nd <= DAG_REC_DEPS (the schedule keeps near + chunk within it).
constexpr int DAG_REC = 64, DAG_REC_HDR = 8, DAG_REC_DEPS = (DAG_REC - DAG_REC_HDR) / 2;
struct DagSched {
  const int* recs = nullptr;  // device, ntask x DAG_REC
  int ntask = 0;
  int nslots = 0;
  // ready-queue scheduling (ZOLO_DAG_QUEUE): per record its dependency count, its dependents
  // (CSR) and the records ready at the start (claim order)
  const int* q_cnt0 = nullptr;
  const int* q_dptr = nullptr;
  const int* q_didx = nullptr;
  const int* q_init = nullptr;
  int q_ninit = 0;
};
// device scratch of a ready-queue launch: cnt (ntask x chains x groups), q (same), ctr[2]
struct DagQueueWork {
  int* cnt = nullptr;
  int* q = nullptr;
  int* ctr = nullptr;
};
// presw: the chains' tiles are stored swizzled (swizzle_tiles); required by the v2 kernel
int dag_trsm_launch(cudaStream_t st, const SpGeom& s, const DagSched& sched, const Chain* d_chains, int nchains,
                    int ncols, int64_t ld, int* flags, int* cflags, int epoch, int* counter, int fwd, int num_sms,
                    unsigned long long* trace = nullptr, const int* tmap = nullptr, bool presw = false,
                    bool need_v2 = false, const DagQueueWork* qw = nullptr, const int* gact = nullptr,
                    const int* gdone = nullptr);
int dag_groups(int ncols);
// forward + backward sweeps in one launch (v2 kernel); tmap: fused claim map (bit 30 = backward), or
// nullptr for forward-then-backward order. Returns the grid, or -1 when the v2 kernel cannot run it.
int dag_fused_launch(cudaStream_t st, const SpGeom& s, const DagSched& sf, const DagSched& sb, const Chain* d_fwd,
                     const Chain* d_bwd, int nchains, int ncols, int64_t ld, int* flags, int* cflags, int epoch,
                     int* counter, int num_sms, const int* tmap);
// chains' cbuf rows [dst_row0, dst_row0 + rows) <- their src rows [row0, row0 + rows), all ncols columns
void dag_stage_inputs(cudaStream_t st, const Chain* d_chains, int nchains, int64_t row0, int64_t rows, int ncols,
                      int64_t ld, int64_t ldp, int64_t dst_row0);

// x[:, 0:ncols] <- op(D_i) x for every block row (the adjoint post-pass
// x_i = DinvL_i^H w_i); x is ld x ncols, D is nbk tiles.
void blockdiag_apply(cudaStream_t st, int nb, const cd* D, bool opH, cd* x, int ncols, int64_t ld,
                     bool swizzled = false);

// One launch covers nchains x ngroups independent pipelines (owner + helpers).
// Returns the number of resident CTAs needed (error if owners do not fit).
int trsm_launch(cudaStream_t st, const BandGeom& g, const Chain* d_chains, int nchains, int ncols, int64_t ld,
                unsigned long long* prog, int* flags_c, int epoch, int* counter, int fwd, int num_sms,
                unsigned long long* trace = nullptr);

}  // namespace zolo

// Block-sparse storage of the unpivoted LU of P (A - sigma B) P^T and the
// interfaces of the factorization (factor.cu) and the triangular sweeps (trsm.cu).
//
// The reference stores a band column-contiguously (band_factor.hpp:37-43) and
// eliminates / sweeps one column at a time (band_factor.hpp:53-182). Here the
// factor is cut into TILE x TILE complex128 tiles over the block symbolic
// structure of the chosen ordering (symbolic.cpp): every elimination and sweep
// step is a dense tile product on the FP64 tensor cores.
#pragma once

#include <vector>

#include "common.cuh"
#include "host.hpp"

namespace zolo {

// device row space: n rows padded to nbk whole tiles (padding rows are identity rows)
struct DevGeom {
  int64_t n = 0;     // matrix order
  int64_t npad = 0;  // nbk * TILE
  int nbk = 0;       // block rows
};

// After factor_run the off-diagonal tiles are ROW-SCALED by the diagonal-block
// inverses: Lt[i][d] = DinvL[i] L(i,i-d), Ut[j][d] = DinvU[j-d] U(j-d,j).
struct FactorTiles {
  cd* Lt = nullptr;
  cd* Ut = nullptr;
  cd* DinvL = nullptr;
  cd* DinvU = nullptr;
  // occupancy masks of each array (tile_masks)
  uint2* mLt = nullptr;
  uint2* mUt = nullptr;
  uint2* mDL = nullptr;
  uint2* mDU = nullptr;
  bool swz = false;  // Lt, Ut, DinvL, DinvU stored in the swizzled sweep layout (swizzle_tiles)
};

// Triangular-solve traversal kinds (trsm.cu).
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
  const uint2* offm;  // occupancy masks of off
  const uint2* prem;  // occupancy masks of pre
  const cd* src;   // right-hand side (ld x ncols), read once per block row
  cd* dst;         // solution (ld x ncols), written in place
  cd* cbuf;        // chunk tasks' partial sums (32 * nslots rows x ncols)
  int mode;
  int pad;
  // three TMA tensor maps in device memory (encode_xblock_map): src, dst, cbuf. The sweeps load a
  // 32-row x 32-column block of them with one cp.async.bulk.tensor into the 128-byte swizzled
  // shared-memory layout the DMMA fragments read conflict free (mma.cuh xsw)
  const unsigned char* tmaps;
};
constexpr int XMAP_BYTES = 128;  // sizeof(CUtensorMap)
// x-block tensor map of a column-major complex block (ld rows, ncols columns; ld a multiple of 32)
// into `map` (XMAP_BYTES, 64-byte aligned). False when the driver cannot encode it.
// x blocks of swc (32 or 64) columns
bool encode_xblock_map(void* map, const cd* base, int64_t ld, int64_t ncols, int swc);

struct FactorDevState {
  int* fail_index;                    // first rejected pivot (device, -1 = none)
  unsigned long long* min_ratio_bits; // min |pivot|/||row|| as double bits
};

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
  // per L tile, written by its panel step: bit (8 g + kb) set when rows 8g..8g+7 x columns
  // 4kb..4kb+3 of L(a,k) hold a nonzero -- the trailing updates skip the empty k-steps
  unsigned* lmask = nullptr;
};

// device copy of a FactorPlan (host.hpp): level ranges stay on the host
struct FactorPlanDev {
  const std::vector<int>* lvl_ptr = nullptr;
  const std::vector<int>* pan_ptr = nullptr;
  const std::vector<int>* tgt_ptr = nullptr;
  const std::vector<int>* cmb_ptr = nullptr;
  const int* cols = nullptr;
  const int* pan = nullptr;
  const int* tgt = nullptr;
  const int* con = nullptr;
  const int* cmb = nullptr;
  cd* scratch = nullptr;  // this pole's partial products of split targets (plan.scratch_slots tiles)
};
// scatter of A - sigma B (assemble_shifted, sparse.hpp:153-186) into the tiles, then the
// level-scheduled LU (3 launches per level of the block elimination tree) and the row scaling
void sp_factor(cudaStream_t st, const SpGeom& s, const SpFactor& f, int64_t nnz, const int* e_row, const int* e_col,
               const double* a_val, const double* b_val, int cx, double sig_re, double sig_im, double* row_norm,
               const int* pad_rows, int npad_rows, FactorDevState ds, int* err, const FactorPlanDev& plan);

// masks[t] = occupancy of tile t: bit (8 g + kb) of .x for rows 8g.. x cols 4kb..
// (op N), of .y for the conjugate transpose (factor.cu tile_mask_kernel).
void tile_masks(cudaStream_t st, const cd* tiles, int64_t ntiles, uint2* masks);
// tiles permuted in place into the sweep layout: element (row, col) at col*32 + (row ^ swz(col))
void swizzle_tiles(cudaStream_t st, cd* tiles, int64_t ntiles);
// out[0] += nonzero entries of the tiles, out[1] += entries in their unmasked 8 x 4 blocks (op N)
void tile_work(cudaStream_t st, const cd* tiles, const uint2* masks, int64_t ntiles, unsigned long long* out);
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
};
// One persistent launch of the warp-specialised sweep kernel over all chains x 32-column groups.
// gact / gdone (optional): the lagged GMRES control's active list and per-column done flags --
// tasks of a fully converged column group are skipped. trace (optional): per-task timestamps.
// Returns the grid size, or -1 when the chains exceed the kernel's limit.
int dag_trsm_launch(cudaStream_t st, const SpGeom& s, const DagSched& sched, const Chain* d_chains, int nchains,
                    int ncols, int swc, int64_t ld, int64_t ldp, int* flags, int* cflags, int epoch, int* counter,
                    int num_sms, unsigned long long* trace = nullptr, const int* gact = nullptr,
                    const int* gdone = nullptr);
// column groups of swc (32 or 64) columns: the sweep tasks' width
int dag_groups(int ncols, int swc);

// x[:, 0:ncols] <- op(D_i) x for every block row (the adjoint post-pass
// x_i = DinvL_i^H w_i); x is ld x ncols, D is nbk tiles.
void blockdiag_apply(cudaStream_t st, int nb, const cd* const* D, cd* const* x, int nchains, bool opH, int ncols,
                     int64_t ld);

}  // namespace zolo

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
//
// J = ceil(bw / TILE) is the block half-bandwidth; rows beyond n are padded
// with identity rows so every tile is full. Each tile is TILE*TILE
// contiguous complex values, column-major.
#pragma once

#include "common.cuh"

namespace zolo {

struct BandGeom {
  int64_t n = 0;     // matrix order
  int64_t npad = 0;  // nbk * TILE
  int nbk = 0;       // block rows
  int J = 0;         // block half-bandwidth
  int64_t bw = 0;    // scalar half-bandwidth
  size_t tiles_per_array() const { return static_cast<size_t>(nbk) * (J + 1); }
};

struct FactorTiles {
  cd* Lt = nullptr;
  cd* Ut = nullptr;
  cd* DinvL = nullptr;
  cd* DinvU = nullptr;
};

__host__ __device__ inline size_t lt_off(int i, int d, int J) {
  return (static_cast<size_t>(i) * (J + 1) + d) * TT;
}

// Triangular-solve traversal kinds (see trsm.cu).
enum SweepMode : int {
  FWD_L = 0,   // L y = b           (solve, band_factor.hpp:62-69)
  BWD_U = 1,   // U x = y           (solve, band_factor.hpp:71-80)
  FWD_UH = 2,  // U^H y = b         (adjoint_solve, band_factor.hpp:98-105)
  BWD_LH = 3   // L^H x = y         (adjoint_solve, band_factor.hpp:107-112)
};

struct Chain {
  const cd* off;    // Lt or Ut array of the pole
  const cd* dinv;   // DinvL or DinvU of the pole
  const cd* src;    // right-hand side (ld x ncols), read once per block row
  cd* dst;          // solution (ld x ncols), written in place
  int mode;
  int pad;
};

// Host launchers (band.cu)
struct FactorDevState {
  int* fail_index;                    // first rejected pivot (device, -1 = none)
  unsigned long long* min_ratio_bits; // min |pivot|/||row|| as double bits
};

void factor_scatter(cudaStream_t st, const BandGeom& g, const FactorTiles& f, int64_t nnz, const int* e_row,
                    const int* e_col, const double* a_val, const double* b_val, int cx, double sig_re,
                    double sig_im, double* row_norm);
void factor_run(cudaStream_t st, const BandGeom& g, const FactorTiles& f, const double* row_norm,
                FactorDevState ds);

// One launch covers nchains x ngroups independent wavefront pipelines.
void trsm_launch(cudaStream_t st, const BandGeom& g, const Chain* d_chains, int nchains, int ncols, int64_t ld,
                 int* flags, int epoch, int* task_counter, int fwd, int num_sms);

}  // namespace zolo

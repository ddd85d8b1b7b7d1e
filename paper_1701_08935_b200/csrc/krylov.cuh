// Host launchers for the Krylov-side kernels (krylov.cu). Every block of
// vectors lives on the device in the factor ordering (P v), column-major with
// leading dimension ld = npad; rows n..npad-1 are kept at zero.
#pragma once

#include "common.cuh"
#include "shard.hpp"

namespace zolo {

constexpr int CHUNK = 2048;  // rows per block in the column reductions
constexpr int KRYLOV_MAX = 256;  // largest Krylov dimension per column (outer GMRES and the hybrid inner solve)

struct GmresDev {
  // per column c (n_v) and shift k (q): see krylov.cu
  int maxit, q, nv;
  void* H;        // [nv][(maxit+1) * maxit] S, column-major per column
  cd* R;          // [nv][q][maxit*maxit]
  cd* G;          // [nv][q][maxit+1]
  cd* ROT;        // [nv][q][2*maxit]
  cd* Y;          // [nv][q][maxit]
  cd* Z;          // [nv][maxit]  folded outer combination coefficients
  double* res;    // [nv][q]
  int* frozen;    // [nv][q]
  int* mlen;      // [nv][q]  length of y_k
  double* beta;   // [nv]
  int* mcol;      // [nv]  Krylov dimension of the column
  int* happy;     // [nv]
  int* done;      // [nv]
  double* wnorm;  // [nv]
  cd* shifts;     // [q]
  double* coef;   // [q]  1/2 M_outer * 1/2 a_(k/2)
  cd* ccoef = nullptr;  // [q] complex combination coefficients (hybrid inner solve), overrides coef
};

template <class S>
struct Krylov {
  static void permute_in(cudaStream_t st, const S* src, int64_t n, S* dst, int64_t ld, int64_t k, const int* perm);
  static void permute_out(cudaStream_t st, const S* src, int64_t ld, S* dst, int64_t n, int64_t k, const int* perm);
  static void col_norms(cudaStream_t st, const S* v, int64_t n, int64_t ld, int64_t k, double* out);
  static void scale_cols(cudaStream_t st, const S* v, S* out, int64_t n, int64_t ld, int64_t k, const double* norms);
  // out (complex, ld x na) = B * V[:, act] (or V[:, act] when B = I)
  static void apply_b(cudaStream_t st, int64_t n, int64_t ld, const int* rp, const int* ci, const S* vals,
                      const S* v, const int* act, int na, cd* out);
  // w[:, act[a]] = c0 v[:, act[a]] + sum_p (real: 2 Re(w_p X_p) | complex: w_p X_p + conj(w_p) Xa_p);
  // compact: written to w[:, a] instead
  static void combine(cudaStream_t st, int64_t n, int64_t ld, double c0, const S* v, const int* act, int na,
                      cd* const* xs, const cd* weights, int r, S* w, bool compact = false);
  // the same combine into the row-blocked layout of a reduce-scatter over nblk ranks: row t of
  // column a at out[(t / rb) rb na + a rb + t % rb]; rows ld .. nblk rb - 1 are zero
  static void combine_blocked(cudaStream_t st, int64_t ld, int64_t rb, int nblk, double c0, const S* v,
                              const int* act, int na, cd* const* xs, const cd* weights, int r, S* out);
  // blk (rows x na, column stride `stride` >= rows) <-> rows [r0, r0 + rows) of the columns act of w
  static void pack_rows(cudaStream_t st, const S* w, int64_t ld, int64_t r0, int64_t rows, int64_t stride,
                        const int* act, int na, S* blk);
  static void unpack_rows(cudaStream_t st, const S* blk, int64_t r0, int64_t rows, int64_t stride, const int* act,
                          int na, S* w, int64_t ld);
  // allgathered blocks (nblk x (rb x na)) -> rows [p rb, min(ld, (p + 1) rb)) of the columns act of w
  static void unpack_blocks(cudaStream_t st, const S* blocks, int64_t rb, int nblk, const int* act, int na, S* w,
                            int64_t ld);
  // w[:, act[a]] = wc[:, a]
  static void scatter_cols(cudaStream_t st, int64_t ld, const S* wc, const int* act, int na, S* w);
  // CGS2 Arnoldi step against basis V_0..V_m (device pointer array) over the rows [r0, r1) of w
  // (nchunk = ceil((r1 - r0) / CHUNK) row chunks). coll == nullptr: the rows are all of them, the
  // chunk partial sums are reduced in fixed order inside the kernels. coll != nullptr (row-sharded
  // pole groups): [r0, r1) is this rank's row block; every inner product is reduced over the local
  // chunks and all-reduced over the ranks (n_active x (m + 1) scalars per pass), so all ranks hold
  // the same H; afterwards partial holds the all-reduced squared norms as ONE chunk per column.
  // Returns the chunk count least_squares reads.
  static int arnoldi(cudaStream_t st, int64_t r0, int64_t r1, int64_t ld, S* const* d_basis, int m, S* w,
                     const int* act, int na, GmresDev g, double* partial, S* hsave, Collective* coll = nullptr);
  // incremental shifted Givens LS + freeze / completion bookkeeping
  static void least_squares(cudaStream_t st, const int* act, int na, int m, GmresDev g, const double* partial,
                            int nchunk, double tol);
  static void next_basis(cudaStream_t st, int64_t n, int64_t ld, const S* w, S* vnext, const int* act, int na,
                         GmresDev g);
  // out[:, c] = sum_i Z_i V_i (+ vin / 2 when vin != nullptr: the outer filter's 1/2 v)
  static void assemble(cudaStream_t st, int64_t n, int64_t ld, const S* v0, S* const* d_basis, int nv, GmresDev g,
                       const S* vin, S* out);
  // C (k x kk) = Y^H Z (column-major, ld rows) -- RR projections
  static void gram(cudaStream_t st, int64_t n, int64_t ld, const S* y, int64_t k, const S* z, int64_t kk, S* out,
                   double* partial);
  // out (ld x kk) = Y (ld x k) * Q (k x kk)
  static void block_gemm(cudaStream_t st, int64_t n, int64_t ld, const S* y, int64_t k, const S* q, int64_t kk,
                         S* out);
  // per column: num = ||ax - lam bx||^2, den = ||bx||^2 (n x k, ld = n)
  static void residuals(cudaStream_t st, int64_t n, const S* ax, const S* bx, const double* lam, int64_t k,
                        double* num, double* den);
  // BSR (atoms of b rows, device rows row0[I]..): act != nullptr: outc[:, a] = M V[:, act[a]] (complex),
  // else out[:, 0:k] = M V[:, 0:k]; padding rows are not written
  static void bsr_spmm(cudaStream_t st, int64_t na, int b, const int* brp, const int* bci, const S* bval,
                       const int* row0, const S* v, int64_t ld, const int* act, int64_t k, S* out, cd* outc);
  // out (ld x k) = M * V (M permuted CSR with S values)
  // Refinement residuals of the shifted solves (zolo_set_refinement): for every chain z,
  // r_z[:, a] = b[:, a] - (A - sigma_z B) x_z[:, a], a < na (B = I when brp == nullptr).
  static void shifted_residual(cudaStream_t st, int64_t n, int64_t ld, const int* arp, const int* aci, const S* av,
                               const int* brp, const int* bci, const S* bv, const cd* b, cd* const* x, cd* const* r,
                               const cd* sigma, int nch, int na);
  static void spmm(cudaStream_t st, int64_t n, int64_t ld, const int* rp, const int* ci, const S* vals, const S* v,
                   int64_t k, S* out);
};

// out[rows[q], c] = 0 for q < nrows, c < k (ld rows per column)
// x <- conj(x) (count complex entries)
void conj_inplace(cudaStream_t st, cd* x, int64_t count);
// x_z[:, 0:na] += d_z[:, 0:na] for the chains z < nch (the refinement corrections)
void add_corrections(cudaStream_t st, int64_t ld, cd* const* x, cd* const* d, int nch, int na);
void zero_rows(cudaStream_t st, const int* rows, int nrows, cd* out, int64_t ld, int64_t k);

}  // namespace zolo

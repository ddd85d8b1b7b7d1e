/*
 * zolo_b200.h -- C ABI of the B200-native Zolotarev filter path.
 *
 * Drop-in boundary for the reference's FilterOperator<S> (ZoloEig,
 * proj/include/zoloeig/filter_engine.hpp:37-165). The reference has no
 * runtime plugin seam: its hot path is the concrete class FilterOperator<S>,
 * constructed by value in subspace_iteration (eigensolver.hpp:172) and
 * called at eigensolver.hpp:184. Each entry point below replaces one member
 * or setup step of that class; the header-only C++ adapter
 * cpp/zolo/gpu_filter_operator.hpp rebuilds the reference's surface
 * (same names, same exceptions) on top of it.
 *
 * Conventions (identical to the reference, dense.hpp:53-115, sparse.hpp:31-36):
 *   - dense blocks are column-major, leading dimension n;
 *   - complex scalars are interleaved (re, im) doubles, i.e. std::complex<double>;
 *   - CSR matrices carry the full (not triangular) pattern with sorted
 *     column indices; offsets/indices are int64 (the reference's size_t);
 *   - scalar tag: ZOLO_F64 for real symmetric pencils, ZOLO_C128 for
 *     complex Hermitian pencils; B == NULL means B = I (SparsePencil::b_mat
 *     empty, sparse.hpp:133-150).
 * Every function returns a status (ZOLO_OK, ...). Host pointers are never
 * retained after a call returns. One context drives one GPU from one host
 * thread; calls on a context are stream-ordered on its private stream.
 */
#ifndef ZOLO_B200_H
#define ZOLO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; the C++ adapter maps them back onto the reference's
 * exception types (error.hpp:25-43, gmres.hpp:45-52). */
enum {
  ZOLO_OK = 0,
  ZOLO_ERR_DOMAIN = 1,        /* DomainError: bad sizes / arguments */
  ZOLO_ERR_NUMERICAL = 2,     /* NumericalError */
  ZOLO_ERR_FACTORIZATION = 3, /* FactorizationError{pivot_index} */
  ZOLO_ERR_GMRES = 4,         /* GmresError{report} (report is filled) */
  ZOLO_ERR_CUDA = 5           /* CUDA / device failure (incl. no device) */
};

enum { ZOLO_F64 = 0, ZOLO_C128 = 1 };

/* Packed FilterDesign (filter_design.hpp:53-69), the boundary input that
 * build_filter_design (filter_design.hpp:133-169) produces on the host:
 *   [0..5]   window a, b, a_minus, a_plus, b_minus, b_plus
 *   [6..9]   mobius gamma, alpha, beta, ell1
 *   [10..14] m_hat, ell2, zmax, constant_term, delta0
 *   [15..18] inner.big_m, inner.delta, outer.big_m, outer.delta
 *   then inner_poles (2r doubles), inner_weights (2r), inner_pf (r),
 *   outer_pf (r), inner.c (2r-1), outer.c (2r-1).          length 17 + 10 r */
enum {
  ZOLO_DESIGN_M_HAT = 10,
  ZOLO_DESIGN_CONSTANT = 13,
  ZOLO_DESIGN_DELTA0 = 14,
  ZOLO_DESIGN_OUTER_M = 17,
  ZOLO_DESIGN_HEAD = 19
};
#define ZOLO_DESIGN_LEN(r) (17 + 10 * (r))
#define ZOLO_MAX_ORDER 16

/* ShiftedSolveReport (gmres.hpp:31-43) merged over columns exactly as
 * filter_engine.hpp:127-133 does. column_iterations is caller-owned
 * (ncols entries) and may be NULL. */
typedef struct {
  int64_t iterations;            /* max Krylov dimension over columns */
  int64_t operator_applications; /* sum over columns */
  int32_t n_shifts;              /* 2 r */
  int32_t all_converged;
  double residuals[2 * ZOLO_MAX_ORDER]; /* per shift, worst column */
  int32_t converged[2 * ZOLO_MAX_ORDER];
  int64_t* column_iterations;
} zolo_report;

/* FactorProfile (band_factor.hpp:31-35) plus the failing pivot. */
typedef struct {
  int64_t bandwidth;      /* half bandwidth under the ordering */
  int64_t stored_entries; /* complex entries stored on the device */
  double min_pivot_ratio; /* min |pivot| / ||row||_inf */
  int64_t pivot_index;    /* -1, or first rejected pivot (FactorizationError) */
} zolo_factor_stats;

typedef struct zolo_ctx zolo_ctx;

/* --- context ---------------------------------------------------------- */
int zolo_ctx_create(int device, zolo_ctx** out);
int zolo_ctx_destroy(zolo_ctx* ctx);
/* Last error message of this context (or of the last failed create when ctx is NULL). */
const char* zolo_last_error(const zolo_ctx* ctx);

/* --- setup (FilterOperator ctor, filter_engine.hpp:40-45) -------------- */
/* Upload the Hermitian(-definite) pencil. Replaces SparsePencil<S>. */
int zolo_pencil_upload(zolo_ctx* ctx, int64_t n, int scalar, const int64_t* a_rp, const int64_t* a_ci,
                       const double* a_v, const int64_t* b_rp, const int64_t* b_ci, const double* b_v);

/* Install the filter design (packed, see above); r = design order. The
 * effective weights are m_hat * inner_weights (filter_engine.hpp:43-44). */
int zolo_set_design(zolo_ctx* ctx, const double* design, int r);

/* build_shifted_factors (band_factor.hpp:199-220): one ordering shared by
 * all shifts -- perm (new -> old, n entries) or NULL for the reference's
 * RCM ordering of the pattern of A - iB (rcm.hpp:69-115) -- then r numeric
 * unpivoted factorizations of A - sigma_j B on the device at
 * sigma = design.inner_poles. stats: r entries or NULL. On a rejected pivot
 * returns ZOLO_ERR_FACTORIZATION with stats[j].pivot_index set. */
int zolo_factorize(zolo_ctx* ctx, const int64_t* perm, zolo_factor_stats* stats);

/* Block (BSR) structure of the pencil (BASELINE config 4: dense b x b blocks
 * per atom; no reference equivalent -- the reference reads CSR only): rows
 * [k b, (k + 1) b) form atom k. The nested dissection then runs on the atom
 * graph and keeps every atom's rows contiguous, and the B products of the
 * filter and the A / B products of the Rayleigh-Ritz projection use a BSR
 * SpMM (dense blocks, one column index per block). Call before
 * zolo_factorize; block = 1 (default) is plain CSR. n must be a multiple of
 * block. */
int zolo_set_block_size(zolo_ctx* ctx, int64_t block);
/* out[0] = the block size, out[1] = atoms of the device BSR copies (0 when the
 * SpMMs run on CSR: block 1, or an ordering that splits atoms). */
int zolo_bsr_info(const zolo_ctx* ctx, int64_t* out);

/* Ordering used by zolo_factorize (both factor into 32 x 32-tile block-sparse
 * LU factors with DAG-scheduled sweeps):
 *   ZOLO_ORDER_ND   (default) nested dissection (recursive BFS-level bisection,
 *                   leaves of <= nd_leaf rows ordered by RCM; default 192,
 *                   nd_leaf <= 0 keeps the current value) -- short dependency
 *                   chains;
 *   ZOLO_ORDER_RCM  the reference's RCM ordering of the pattern of A - iB
 *                   (band_factor.hpp:203-204, rcm.hpp:69-115): the factor is the
 *                   reference's band envelope, and FactorizationError pivot
 *                   indices are the reference's (positions in RCM order).
 * With an explicit perm in zolo_factorize, that ordering is factored as is.
 * Pivot indices refer to positions in the chosen order. */
enum { ZOLO_ORDER_ND = 0, ZOLO_ORDER_RCM = 1 };
int zolo_set_ordering(zolo_ctx* ctx, int mode, int64_t nd_leaf);

/* Solve mode of the shifted systems (BASELINE config 2 "hybrid solve";
 * the reference factors every pole):
 *   ZOLO_SOLVE_DIRECT  (default) every pole factored, as the reference;
 *   ZOLO_SOLVE_HYBRID  only `pole` is factored; for the others
 *     (A - s_j B)^{-1} B v = (I - (s_j - s_p) K_p^{-1} B)^{-1} K_p^{-1} B v
 *     by one shift-invariant multi-shift GMRES on K_p^{-1} B per G application
 *     (one Krylov basis serving every other pole), to relative residual
 *     inner_tol within inner_max iterations (else ZOLO_ERR_NUMERICAL).
 * ND ordering, no pole sharding; call after zolo_set_design, before
 * zolo_factorize. The inner-solve counter then counts K_p applications. */
enum { ZOLO_SOLVE_DIRECT = 0, ZOLO_SOLVE_HYBRID = 1 };
int zolo_set_solve_mode(zolo_ctx* ctx, int mode, int pole, double inner_tol, int inner_max);

/* Sylvester inertia (the reference takes eigenvalue
 * counts as inputs): *count = the number of eigenvalues of the
 * pencil (A, B), B Hermitian positive definite, below the real shift sigma,
 * from the signs of the pivots of the unpivoted block LU = L D L^H of
 * A - sigma B under the ND ordering (Sylvester's law of inertia). The count in
 * (a, b) is count(b) - count(a). A pivot under the monitor threshold
 * (|piv| <= 1e-14 ||row||, sigma within rounding of an eigenvalue, or an
 * unpivoted breakdown) returns ZOLO_ERR_FACTORIZATION: retry at a nudged shift.
 * Uses temporary factor storage; the filter factors are untouched.
 * min_pivot_ratio may be NULL. */
int zolo_count_below(zolo_ctx* ctx, double sigma, int64_t* count, double* min_pivot_ratio);

/* Pole sharding over NCCL (no reference equivalent -- the
 * reference sums all poles in one process, filter_engine.hpp:63-69,73-78).
 * Rank g of nranks factors the poles j = g, g + nranks, ... (< r; needs
 * r >= nranks) and every G application ends with one in-place
 * ncclAllReduce(sum) of the ranks' partial sums, so all ranks hold identical
 * G v and run an identical (replicated) Krylov iteration; rank 0 adds the
 * constant term. unique_id: ZOLO_NCCL_ID_BYTES bytes from zolo_nccl_unique_id
 * on rank 0, broadcast by the caller; all ranks call collectively, before
 * zolo_factorize. By default the Arnoldi step is row-sharded: rank g keeps rows
 * [g rb, (g + 1) rb) of the Krylov vectors (rb = npad / nranks rounded up to
 * 32), a G application ends with an ncclReduceScatter of the partial sums over
 * those row blocks, the CGS2 inner products are all-reduced and the next basis
 * vector all-gathered -- the bytes of one all-reduce per iteration, the
 * Arnoldi work divided by the ranks (ZOLO_ROW_SHARD=0: the replicated variant,
 * one ncclAllReduce of G and every rank orthogonalising all rows).
 * unique_id = NULL with nranks > 1 gives an unreduced context:
 * zolo_apply_g returns the rank's partial sum, zolo_apply_filter refuses.
 * NCCL is loaded with dlopen (libnccl.so.2) only when a communicator is built. */
#define ZOLO_NCCL_ID_BYTES 128
int zolo_nccl_unique_id(void* out);
int zolo_set_pole_shard(zolo_ctx* ctx, int rank, int nranks, const void* unique_id);

/* The same pole shard with the group's collectives staged through the host:
 * fn(op, buf, count, user) must complete the collective over the nranks
 * callers (returning 0) on doubles in host memory:
 *   ZOLO_COLL_ALLREDUCE       buf[0..count) in place, summed over the ranks;
 *   ZOLO_COLL_REDUCE_SCATTER  in: buf[0 .. nranks count) (rank-major blocks);
 *                             out: buf[0 .. count) = this rank's block summed;
 *   ZOLO_COLL_ALLGATHER       in: this rank's block at buf[rank count ..);
 *                             out: buf[0 .. nranks count) all blocks.
 * Any transport works (torch.distributed gloo, threads of one process sharing
 * a GPU -- no kernel of one rank ever waits on another's). */
enum { ZOLO_COLL_ALLREDUCE = 0, ZOLO_COLL_REDUCE_SCATTER = 1, ZOLO_COLL_ALLGATHER = 2 };
typedef int (*zolo_collective_fn)(int op, double* buf, int64_t count, void* user);
int zolo_set_pole_shard_host(zolo_ctx* ctx, int rank, int nranks, zolo_collective_fn fn, void* user);

/* FilterOperator(pencil, design): upload + set_design + factorize. */
int zolo_filter_create(zolo_ctx* ctx, int64_t n, int scalar, const int64_t* a_rp, const int64_t* a_ci,
                       const double* a_v, const int64_t* b_rp, const int64_t* b_ci, const double* b_v,
                       const double* design, int r, zolo_factor_stats* stats);

/* --- hot path ----------------------------------------------------------- */
/* FilterOperator::apply_g (filter_engine.hpp:56-82) on an n x ncols host
 * block (one G application, counted once as the reference does). */
int zolo_apply_g(zolo_ctx* ctx, const double* v, double* gv, int64_t ncols);

/* FilterOperator::apply_filter (filter_engine.hpp:86-155) on an n x ncols
 * host block: all 2r outer shifts +-i sqrt(outer.c[2j]) in one multi-shift
 * GMRES per column (lock-step batched on the device), combined as
 * 1/2 M_outer sum_j 1/2 a_j (x_2j + x_2j+1) + 1/2 v. Returns ZOLO_ERR_GMRES
 * with rep filled (y still written) when some shift misses gmres_tol.
 * gmres_max <= ZOLO_KRYLOV_MAX (the reference has no cap, gmres.hpp:98-101;
 * the device keeps at most that many basis vectors per column). */
#define ZOLO_KRYLOV_MAX 256
int zolo_apply_filter(zolo_ctx* ctx, const double* v, double* y, int64_t ncols, double gmres_tol,
                      int64_t gmres_max, zolo_report* rep);

/* Same with device-resident blocks (original ordering, leading dimension n,
 * same element layout); no host<->device copies. */
int zolo_apply_filter_device(zolo_ctx* ctx, const void* d_v, void* d_y, int64_t ncols, double gmres_tol,
                             int64_t gmres_max, zolo_report* rep);

/* ShiftedFactor::solve / adjoint_solve (band_factor.hpp:53-117) of one factored
 * pole: x = (A - sigma_j B)^-1 b (adjoint = 0) or (A - sigma_j B)^-H b
 * (adjoint = 1) for an n x ncols complex block b (original ordering,
 * interleaved complex, column-major), through the same device factors and
 * sweeps as the filter (refined when zolo_set_refinement is on). pole: index
 * of the design's inner pole, factored by this context. */
int zolo_shifted_solve(zolo_ctx* ctx, int pole, int adjoint, const double* b, double* x, int64_t ncols);

/* inner_solve_count / g_application_count (filter_engine.hpp:50-51). */
int zolo_counters(const zolo_ctx* ctx, int64_t* inner_solves, int64_t* g_applications);

/* Rayleigh-Ritz projections (eigensolver.hpp:108-109): Atilde = Y^H A Y,
 * Btilde = Y^H B Y, k x k column-major, Y an n x k host block. */
int zolo_rr_project(zolo_ctx* ctx, const double* y, int64_t k, double* a_tilde, double* b_tilde);

/* Device-side GEMM for the subspace update Q = Y * Qsmall (eigensolver.hpp:190):
 * y n x k, q_small k x kk (host), out n x kk (host). */
int zolo_block_update(zolo_ctx* ctx, const double* y, int64_t k, const double* q_small, int64_t kk, double* out);

/* --- device-resident block helpers (original ordering, leading dimension n) */
/* out = A x (which = 0) or B x (which = 1; a copy when B = I), k columns. */
int zolo_spmm_device(zolo_ctx* ctx, int which, const void* d_x, void* d_out, int64_t k);
/* out (host, k x kk column-major) = Y^H Z. */
int zolo_gram_device(zolo_ctx* ctx, const void* d_y, const void* d_z, int64_t k, int64_t kk, double* out);
/* d_out (n x kk) = Y (n x k) * q (host, k x kk). */
int zolo_block_gemm_device(zolo_ctx* ctx, const void* d_y, int64_t k, const double* q, int64_t kk, void* d_out);
/* per column: num = ||ax - lambda bx||^2, den = ||bx||^2 (relative_residual, eigensolver.hpp:77-93). */
int zolo_residual_norms_device(zolo_ctx* ctx, const void* d_ax, const void* d_bx, int64_t k, const double* lambdas,
                               double* num, double* den);

/* --- driver: subspace_iteration (eigensolver.hpp:154-217) ---------------- */
/* Filtered subspace iteration with Rayleigh-Ritz on this context's GPU for the
 * packed filter design `design` of order r (built on the host, e.g. by the
 * reference's build_filter_design; the window (a, b) is design[0..1]):
 * factorizes, iterates. lambdas has room for n_lambda + oversample values;
 * vectors (optional) for n x (n_lambda + oversample) entries. stats (14 doubles):
 * n_ss, n_iter, n_gmres, n_gmres_min, n_solv, t_fact [s], t_iter [s], residual
 * (reference scaling max(|a|,|b|)), converged, r, residual scaled by |lambda|,
 * device filter time [ms], first refined iteration (0 = none), residual of the
 * first iteration.
 * refine: residual-correction refinement of the shifted solves (see
 * zolo_set_refinement): 0 never, 1 always, -1 automatic (once an iteration has
 * brought the residual below 1e-5 without meeting tol: the remaining gap is the
 * solves' rounding floor, eps / min pivot ratio of the unpivoted LU). */
int zolo_subspace_iteration(zolo_ctx* ctx, int64_t n, int scalar, const int64_t* a_rp, const int64_t* a_ci,
                            const double* a_v, const int64_t* b_rp, const int64_t* b_ci, const double* b_v,
                            const double* design, int r, int64_t n_lambda, int64_t oversample, double tol,
                            int64_t max_iters, double gmres_tol, int64_t gmres_max, uint64_t seed, int refine,
                            double* lambdas, int64_t* n_found, double* vectors, double* stats);

/* Residual-correction (iterative) refinement of every shifted solve:
 * x = K^-1 b, then `steps` times x += K^-1 (b - K x) with K = A - sigma_j B
 * (K^H for the adjoint solves), the residual formed from the pencil's CSR
 * in FP64. The unpivoted LU's rounding (eps / min pivot ratio, band_factor.hpp
 * has no pivoting) then drops to the backward-stable level; each step costs one
 * more sweep pair. Counters keep the reference's meaning (one solve per
 * shifted system). steps in [0, 2]; 0 (default) = the reference's plain solve. */
int zolo_set_refinement(zolo_ctx* ctx, int steps);
/* Relaxed refinement inside zolo_apply_filter (no reference equivalent): with refinement on, a G
 * application skips the correction once the GMRES residuals rho of the iteration before satisfy
 * 10 * rho * (relative residual of the unrefined solves, worst chain, measured once per
 * factorization) <= gmres_tol -- the later an operator application in a Krylov iteration, the less
 * exact it must be. out[0] = that measured residual (-1 before the first refined application),
 * out[1] = G applications of the last zolo_apply_filter that ran unrefined under the rule. */
int zolo_refinement_stats(const zolo_ctx* ctx, double* out);
/* on = 0: every G application of a refined zolo_apply_filter is corrected (default: relaxed). */
int zolo_set_refinement_relaxation(zolo_ctx* ctx, int on);

/* Return the device memory cached by the library's allocator on `device`
 * (blocks of destroyed contexts) to the driver. */
int zolo_pool_trim(int device);

/* Set the context's (or, with NULL, the global) last-error message. */
void zolo_set_error(zolo_ctx* ctx, const char* msg);

/* --- timing of the last device call (CUDA events on the context stream) - */
/* ms[0] = last apply_filter device time, ms[1] = last factorize device time,
 * ms[2] = solve-kernel time summed over the last apply_filter,
 * ms[3] = number of solve-kernel launches in the last apply_filter,
 * ms[4] = kernel launches of the last apply_filter (all kernels),
 * ms[5] = operator applications (sum of active columns) of the last apply_filter,
 * ms[6] = hybrid solve: inner K_p applications (column-steps) of the last apply_filter,
 * ms[7] = device time of the GMRES iterations of the last apply_filter.
 * ms must hold 8 doubles. */
int zolo_last_timings(const zolo_ctx* ctx, double* ms);

/* Structure the triangular sweeps run over (per pole, after zolo_factorize):
 * out[0] block rows (32-row tiles), out[1] off-diagonal tiles of L (= of U),
 * out[2] / out[3] forward / backward DAG task records, out[4] chunk
 * partial-sum slots, out[5] critical path in block rows; work accounting of
 * one pole's sweep tiles (Lt, Ut, DinvL, DinvU: 1024 stored entries each):
 * out[6] nonzero entries (the scalar fill), out[7] entries inside the
 * unmasked 8 x 4 blocks the DMMA loops execute (op N).
 * No equivalent in the reference (development / roofline accounting). */
int zolo_sweep_profile(const zolo_ctx* ctx, int64_t* out);

/* Device timer on the context stream: op 0 records the start event, op 1
 * records the stop event, waits for it and returns the elapsed ms. */
int zolo_timer(zolo_ctx* ctx, int op, double* ms);

/* --- host-only helpers (no GPU needed) ---------------------------------- */
/* Block structure of the nested-dissection factor (no reference equivalent;
 * development / sizing): out[0] padded size, out[1] block rows, out[2]
 * off-diagonal tiles per triangle, out[3] critical path in block rows,
 * out[4] block rows of the largest trailing dense block, out[5] tile-aligned
 * node groups, out[6] trailing-update tile products of the factorization (sum over
 * block columns of the squared column count), out[7] reserved. */
int zolo_nd_structure(int64_t n, const int64_t* rp, const int64_t* ci, int64_t leaf, int64_t* out);
/* Builds the left-looking factor plan of the ND factor of a pattern (symbolic.cpp factor_plan)
 * and checks it on the host (no reference equivalent; test support): out[0] = violations (0 when
 * every tile is completed by exactly one target at the level of its block column, every
 * contribution is a pair L(a,k), U(k,b) of that target with k below it on a lower level, in
 * ascending k also across the parts of split targets, every part is read by one combine entry,
 * and the contributions number sum_k |col(k)|^2), out[1] contributions, out[2] target records,
 * out[3] split targets, out[4] scratch tiles of the widest level, out[5] levels. */
int zolo_factor_plan_check(int64_t n, const int64_t* rp, const int64_t* ci, int64_t leaf, int64_t* out);
/* Builds the DAG sweep schedules (both directions) of the ND factor of a pattern and checks them
 * on the host (no reference equivalent; test support): out[0] = violations (0 when every block
 * row has one row task, every dependency is summed exactly once, every partial slot is written
 * once and the claim order is topological), out[1] tasks, out[2] partial slots, out[3] block rows. */
int zolo_dag_schedule_check(int64_t n, const int64_t* rp, const int64_t* ci, int64_t leaf, int near, int chunk,
                            int order, int64_t* out);
/* reorder_rcm (rcm.hpp:69-115) of a structurally symmetric pattern;
 * perm[new] = old. bw/profile (rcm.hpp:118-147) may be NULL. */
int zolo_rcm(int64_t n, const int64_t* rp, const int64_t* ci, int64_t* perm, int64_t* bw, int64_t* profile);
/* The nested-dissection ordering of ZOLO_ORDER_ND (no reference equivalent):
 * pos[i] = padded device position of row i (tree nodes padded to 32-row
 * tiles), *npad = padded size. */
int zolo_nd_order(int64_t n, const int64_t* rp, const int64_t* ci, int64_t leaf, int64_t* pos, int64_t* npad);

/* random_gaussian<S> (dense.hpp:181-208, raw mt19937_64 bits + Box-Muller),
 * optionally followed by mgs_orthonormalize (dense.hpp:212-229). */
int zolo_random_block(int scalar, int64_t n, int64_t k, uint64_t seed, int orthonormalize, double* out);

/* n uniforms in [0,1) from raw mt19937_64 bits, (x >> 11) * 2^-53 -- the
 * reference's disorder convention (hamiltonian.hpp:52); used by the
 * synthetic config generators. */
int zolo_uniform_stream(uint64_t seed, int64_t n, double* out);

/* Library version / build tag. */
const char* zolo_version(void);

#ifdef __cplusplus
}
#endif

#endif /* ZOLO_B200_H */

#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <memory>
#include <utility>
#include <vector>

namespace zolo {
// Block (32x32-tile) structure of the LU factors under a node ordering
// (symbolic.cpp). Off-diagonal tile ids are row-major slots: row i's tiles
// (i, row_idx[e]) for e in [row_ptr[i], row_ptr[i+1]), k ascending; column
// k's entries (col_idx[e], k) for e in [col_ptr[k], col_ptr[k+1]) carry their
// tile id in col_tile[e]. L(i,k) and U(k,i) share the id.
struct BlockStructure {
  int64_t npad = 0, nb = 0, ntiles = 0, critical_path = 0;
  std::vector<int64_t> pos;  // original row -> padded position
  std::vector<int64_t> inv;  // padded position -> original row, or -1 (identity padding)
  std::vector<int64_t> col_ptr, col_idx, col_tile;
  std::vector<int64_t> row_ptr, row_idx;
  std::vector<int64_t> parent;  // block elimination tree
};
void nd_order(int64_t n, const int64_t* rp, const int64_t* ci, int64_t leaf, std::vector<std::vector<int64_t>>& nodes);
void block_symbolic(int64_t n, const int64_t* rp, const int64_t* ci, const std::vector<std::vector<int64_t>>& nodes,
                    int tile, BlockStructure& bs);
// Level-scheduled left-looking block LU (factor.cu sp_factor): block columns grouped by their
// height in the block elimination tree (columns of one level are independent). Per level: the
// trailing-update targets of its columns -- D(y), L(x, y), U(y, x) -- each with ALL its
// contributions (L(a,k), U(k,b)) in ascending k, so the accumulation order is fixed
// (deterministic factors) and every tile is written once; then the diagonal blocks; then the
// panel tiles.
//   pan: 2 ints per item (k, 2 * tile id + upper)
//   tgt: 2 ints per target (kind 0 = Dt / 1 = Lt / 2 = Ut in bits 30-31 | tile id, first
//        contribution); a target's contributions end where the next target's begin (the lists are
//        laid out in target order; one sentinel entry closes the last)
//        kind 3 = one part of a split target: the id is a scratch slot of the level, the part's
//        product is stored there
//   con: 2 ints per contribution (L tile id, U tile id)
//   cmb: 3 ints per split target (kind | tile id, first scratch slot, parts): tile -= the parts,
//        in part order
// std::vector whose resize leaves new elements uninitialised: the plan's large arrays are sized
// once and filled by the worker threads (which also take their first-touch page faults)
template <class T>
struct NoInit : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = NoInit<U>;
  };
  template <class U, class... A>
  void construct(U* p, A&&... a) {
    if constexpr (sizeof...(A) == 0)
      ::new (static_cast<void*>(p)) U;
    else
      ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
  }
};
using RawInts = std::vector<int, NoInit<int>>;
struct FactorPlan {
  std::vector<int> lvl_ptr, cols, pan_ptr, pan, tgt_ptr, cmb_ptr;
  RawInts tgt, con, cmb;
  int64_t scratch_slots = 0;  // partial-product tiles of the widest level (split targets)
  int64_t contributions = 0;
};
void factor_plan(const BlockStructure& bs, FactorPlan& plan);

// One claim-ordered task of a DAG triangular sweep (trsm.cu dag2_kernel).
// Block row i's dependencies, in processing order q (forward: ascending
// column, backward: descending row), are cut into CHUNK tasks (out >= 0: sum
// op(T~) u_j over q in [qa, qb) into partial slot `out`) and one ROW task
// (out = -1: u_i = pre(b_i) - sum over q in [qa, qb) - partial slots
// [pa, pa + pc)). Every task appears after all tasks it waits on, so
// persistent CTAs claiming in this order cannot deadlock.
// After dag_schedule the chunks of a row ACCUMULATE into K_i = min(DAG_PCHAINS, chunks) partial
// (at least chunks / 63: a chain has at most 64 steps)
// slots [pa, pa + K_i) of a unit of DAG_PCHAINS slots: chunk c writes slot pa + c % K_i as step
// c / K_i of that chain, adding the chain's partial so far (pc = 1) when c >= K_i; the row task adds
// the K_i partials (pc = K_i). A slot's flag stamp is epoch * DAG_GENS + 64 `gen` + step, `gen`
// counting the unit's uses; `aux` = c | K_i << 16 (chunks) or the chunk count (rows). Units are
// reused along the claim order: the first chunk of each chain of a row that takes over a unit waits
// for the row task that last read it (`wait`: its block row).
constexpr int DAG_GENS = 4096;
#ifndef ZOLO_PCHAINS
#define ZOLO_PCHAINS 2  // measured: 1 / 2 / 4 chains: cfg2 1642 / 1679 / 1711, cfg3 125.8 / 125.6 / 124.9 vec/s; cfg5 fits one batch up to 2
#endif
constexpr int DAG_PCHAINS = ZOLO_PCHAINS;
struct DagTask {
  int i, qa, qb, pa, pc, out;
  int gen = 0, wait = -1, aux = 0;
};
// first block row of the largest trailing block [s0, nb) of at most kmax block rows whose
// L pattern is dense (every row holds every earlier row of the block); nb if none
int trailing_dense_start(const BlockStructure& bs, int kmax);
// ptr/idx: forward = (row_ptr, row_idx), backward = (col_ptr, col_idx).
// Rows with more than near + chunk dependencies keep the `near` latest in
// the row task; the rest go to chunks of <= chunk dependencies, each claimed
// right after the row task of its latest dependency. order: 0 = that
// positional order, 1 = by earliest start time (EST), 2 = by longest path to
// the sweep's end (BL), >= 3: EST - (order - 2)/8 * BL (all weighted by tile
// products; all topological). Returns the slot count.
int dag_schedule(int64_t nb, const std::vector<int64_t>& ptr, const std::vector<int64_t>& idx, bool fwd, int chunk,
                 int near, int order, std::vector<DagTask>& tasks);
int accumulate_slots(std::vector<DagTask>& tasks, int64_t nb);
void rcm_order(int64_t n, const int64_t* rp, const int64_t* ci, int64_t* perm);
int64_t bandwidth_under(int64_t n, const int64_t* rp, const int64_t* ci, const int64_t* perm);
int64_t profile_under(int64_t n, const int64_t* rp, const int64_t* ci, const int64_t* perm);
void uniform_stream(uint64_t seed, int64_t n, double* out);
bool random_block(int cx, int64_t n, int64_t k, uint64_t seed, bool orthonormalize, double* out);
}  // namespace zolo

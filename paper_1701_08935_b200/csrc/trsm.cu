// Pipelined multi-RHS block-band triangular solves on the FP64 tensor cores.
//
// Reference: ShiftedFactor::solve / adjoint_solve (band_factor.hpp:53-117)
// sweep the band once per right-hand-side column: forward L / backward U for
// the solve, U^H / L^H for the adjoint. Here every sweep runs over all columns
// of the block at once, as a recurrence over TILE-row blocks:
//
//     x_i = c_i - M_i x_{i-+1},      c_i = Dinv_i (b_i - sum_{d>=2} T_(i,i-+d) x_(i-+d))
//
// with M_i = Dinv_i T_(i,i-+1) precomputed by the factorization (factor.cu).
//   HELPER tasks compute every c_i -- all the flops, off the critical path
//     (they need x only up to block i-+2) -- through an NS-stage cp.async
//     pipeline of envelope tiles;
//   one OWNER task per (chain, column group) walks the chain doing only the
//     M_i x_{i-+1} product, with x_{i-+1} kept in shared memory.
// All tile products are mma.sync.m8n8k4.f64 (DMMA): warp w owns an 8x8
// complex block of the 32 x CG output (4 real MMAs per complex k-step), so no
// cross-lane reduction is needed. All poles, solve + adjoint chains and all
// column groups share ONE persistent launch per sweep direction. The owner
// publishes progress as one monotone (epoch << 32 | steps) counter per chain,
// helpers publish c_i through per-block epoch flags; tasks are claimed in
// dependency order (owners first) from an atomic counter, so the launch is
// deadlock free whenever the owners fit on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "band.cuh"
#include "host.hpp"
#include "mma.cuh"

namespace zolo {

namespace {

constexpr int APAD = TILE + 2; // tile column stride: op N fragment loads conflict free
constexpr int TILE_S = TILE * APAD;
constexpr int XS = CG * XPAD;
constexpr int NS = 3;          // helper pipeline stages
constexpr int SMEM_FIXED = (NS * TILE_S + NS * XS + TILE_S + XS) * static_cast<int>(sizeof(cd));
static_assert(CG == 16, "warp layout assumes 32 x 16 output blocks");

struct SolveArgs {
  const Chain* chains;
  int nchains, ngroups, ncols, nbk, J, epoch, fwd;
  int64_t ld;
  const int* dl;
  unsigned long long* prog;  // per (chain, group): (epoch << 32) | owner steps done
  int* flags_c;              // per (chain, group, block): epoch when c_i is ready
  int* counter;              // [0] task counter, [2] wait-timeout error word
  unsigned long long* trace; // optional: per-step timestamps of chain 0 / group 0
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void dmma(double c[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// acc[2] (complex, the two owned outputs) += op(T)[r0:r0+8, :] X[:, c0:c0+8].
// T padded [col*APAD + row]; X padded [col*XPAD + k]. op H = conjugate transpose.
template <bool OPH>
__device__ __forceinline__ void mma_tile_t(cd acc[2], const cd* ts, const cd* xs, const Frag& f) {
  const int ar = f.r0 + (f.lane >> 2), am = f.lane & 3;
  const int bc = f.c0 + (f.lane >> 2), bm = f.lane & 3;
  // all 16 fragments first (latency overlapped), then 32 DMMAs on 4 chains
  cd a[TILE / 4], b[TILE / 4];
#pragma unroll
  for (int kb = 0; kb < TILE / 4; ++kb) {
    const int k = 4 * kb + am;
    a[kb] = OPH ? ts[ar * APAD + k] : ts[k * APAD + ar];
    b[kb] = xs[bc * XPAD + 4 * kb + bm];
  }
  double re0[2] = {0.0, 0.0}, im0[2] = {0.0, 0.0}, re1[2] = {0.0, 0.0}, im1[2] = {0.0, 0.0};
#pragma unroll
  for (int kb = 0; kb < TILE / 4; ++kb) {
    double* re = (kb & 1) ? re1 : re0;
    double* im = (kb & 1) ? im1 : im0;
    if (OPH) {  // a = conj(t): Re = t.x b.x + t.y b.y, Im = t.x b.y - t.y b.x
      dmma(re, a[kb].x, b[kb].x);
      dmma(re, a[kb].y, b[kb].y);
      dmma(im, a[kb].x, b[kb].y);
      dmma(im, -a[kb].y, b[kb].x);
    } else {
      dmma(re, a[kb].x, b[kb].x);
      dmma(re, -a[kb].y, b[kb].y);
      dmma(im, a[kb].x, b[kb].y);
      dmma(im, a[kb].y, b[kb].x);
    }
  }
  acc[0].x += re0[0] + re1[0];
  acc[1].x += re0[1] + re1[1];
  acc[0].y += im0[0] + im1[0];
  acc[1].y += im0[1] + im1[1];
}

__device__ __forceinline__ void mma_tile(cd acc[2], const cd* ts, const cd* xs, bool opH, const Frag& f) {
  if (opH)
    mma_tile_t<true>(acc, ts, xs, f);
  else
    mma_tile_t<false>(acc, ts, xs, f);
}

__device__ __forceinline__ void load_tile(cd* s, const cd* g) {
#pragma unroll
  for (int q = 0; q < TT / ST; ++q) {
    const int e = threadIdx.x + q * ST;
    cp_async16_cg(&s[(e / TILE) * APAD + (e % TILE)], g + e);
  }
}

// 32 rows x CG columns of a column-major block into [col*XPAD + row].
__device__ __forceinline__ void load_x(cd* xs, const cd* base, int64_t ld, int c0, int nc) {
  const int row = threadIdx.x & 31, cc = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < CG / 8; ++q) {
    const int c = cc + 8 * q;
    if (c < nc)
      cp_async16_cg(&xs[c * XPAD + row], base + row + (c0 + c) * ld);
    else
      xs[c * XPAD + row] = mk(0.0, 0.0);
  }
}

// thread 0 waits for *f >= epoch (bounded: a lost producer is reported through
// err, never a hung GPU), then the CTA synchronises.
__device__ __forceinline__ void wait_flag(const int* f, int epoch, int* err) {
  if (threadIdx.x == 0) {
    int spins = 0;
    while (ld_acquire(f) < epoch) {
      if (++spins > 256) __nanosleep(32);
      if (spins > (1 << 25)) {
        atomicExch(err, 1);
        break;
      }
    }
  }
  __syncthreads();
}

// OWNER: x_i = c_i - op(M_i) x_{i-+1} along the whole chain (one column group).
__device__ void owner_task(const SolveArgs& A, int ci, int gi, cd* smem) {
  cd* m_s[2] = {smem, smem + TILE_S};
  cd* xb[2] = {smem + 2 * TILE_S, smem + 2 * TILE_S + XS};
  const Chain ch = A.chains[ci];
  const bool fwd = A.fwd != 0;
  const bool opH = ch.mode == FWD_UH || ch.mode == BWD_LH;
  const Frag f = frag();
  const int c0 = gi * CG, nc = min(CG, A.ncols - c0);
  const int64_t ld = A.ld;
  unsigned long long* prog = A.prog + static_cast<size_t>(ci) * A.ngroups + gi;
  const unsigned long long tag = static_cast<unsigned long long>(A.epoch) << 32;
  const int* fc = A.flags_c + (static_cast<size_t>(ci) * A.ngroups + gi) * A.nbk;
  cd* cstage = smem + 2 * TILE_S + 2 * XS;  // per-thread c_i staging (own elements only)
  int* dl_s = reinterpret_cast<int*>(cstage + 2 * ST);  // envelope table, read once
  for (int b = threadIdx.x; b < A.nbk; b += ST) dl_s[b] = A.dl[b];
  // Roles inside the owner: thread 0 publishes (its release fence must not
  // wait on any cp.async, so warp 0 issues none for the coupling tiles);
  // thread 32 polls the NEXT step's c flag after the product (no poll sits in
  // front of a barrier); cready_s is double-buffered by step parity.
  __shared__ int cready_s[2];
  if (threadIdx.x == 32) cready_s[0] = ld_acquire(fc + (fwd ? 0 : A.nbk - 1)) >= A.epoch;
  __syncthreads();
  const bool tr = A.trace != nullptr && ci == 0 && gi == 0 && threadIdx.x == 0;
  for (int s = 0; s < A.nbk; ++s) {
    const int i = fwd ? s : A.nbk - 1 - s;
    if (tr) A.trace[s * 16 + 0] = gtimer();
    // coupling tile of the NEXT step: T~(i', i'-+1) is slot 1 of row i' (fwd) or i'+1 (bwd)
    if (s + 1 < A.nbk && threadIdx.x >= 32) {
      const int base = fwd ? i + 1 : i;
      if (dl_s[base] >= 1) {
        const cd* g = ch.off + lt_off(base, 1, A.J);
        cd* sm = m_s[(s + 1) & 1];
        for (int e = threadIdx.x - 32; e < TT; e += ST - 32)
          cp_async16_cg(&sm[(e / TILE) * APAD + (e % TILE)], g + e);
      }
    }
    cp_async_commit();
    cp_async_wait<1>();  // M_i landed (issued one step earlier)
    __syncthreads();
    if (tr) A.trace[s * 16 + 11] = gtimer();
    const bool cready = cready_s[s & 1];
    cd* crow = ch.cbuf + static_cast<int64_t>(i) * TILE + f.row + c0 * ld;
    if (cready) {  // c_i already published: stream it in under the product
#pragma unroll
      for (int q = 0; q < 2; ++q)
        if (f.col + q < nc) cp_async16_cg(&cstage[threadIdx.x * 2 + q], crow + (f.col + q) * ld);
      cp_async_commit();
    }
    // the critical product needs only x_{i-+1} (on chip): do it before c_i arrives
    cd red[2] = {mk(0.0, 0.0), mk(0.0, 0.0)};
    if (s > 0 && dl_s[fwd ? i : i + 1] >= 1) mma_tile(red, m_s[s & 1], xb[(s + 1) & 1], opH, f);
    if (tr) A.trace[s * 16 + 12] = gtimer() + (red[0].x == 1234.5 ? 1 : 0);
    // publish x_{s-1} now: its global stores were ordered by the barriers of
    // the previous step and have landed during the product, so the release
    // fence is cheap and off the chain (helpers need x only 2+ steps later)
    if (threadIdx.x == 0 && s > 0) {
      st_release64(prog, tag | static_cast<unsigned>(s));
      if (A.trace != nullptr && ci == 0 && gi == 0) A.trace[(s - 1) * 16 + 2] = gtimer();
    }
    if (threadIdx.x == 32 && s + 1 < A.nbk)
      cready_s[(s + 1) & 1] = ld_acquire(fc + (fwd ? i + 1 : i - 1)) >= A.epoch;
    if (tr) A.trace[s * 16 + 6] = gtimer() + (red[0].x == 1234.5 ? 1 : 0);
    cd cv[2];
    if (cready) {
      cp_async_wait<0>();  // this thread's own copies: no barrier needed to read them
#pragma unroll
      for (int q = 0; q < 2; ++q) cv[q] = (f.col + q < nc) ? cstage[threadIdx.x * 2 + q] : mk(0.0, 0.0);
    } else {
      wait_flag(fc + i, A.epoch, A.counter + 2);
#pragma unroll
      for (int q = 0; q < 2; ++q) cv[q] = (f.col + q < nc) ? __ldcg(crow + (f.col + q) * ld) : mk(0.0, 0.0);
    }
    if (tr) A.trace[s * 16 + 1] = gtimer();
    cd* xrow = ch.dst + static_cast<int64_t>(i) * TILE + f.row + c0 * ld;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int c = f.col + q;
      const cd x = csub(cv[q], red[q]);
      xb[s & 1][c * XPAD + f.row] = x;
      if (c < nc) xrow[c * ld] = x;
    }
    __syncthreads();
    if (tr) A.trace[s * 16 + 7] = gtimer();
  }
  cp_async_wait<0>();
  __syncthreads();
  if (threadIdx.x == 0) {
    st_release64(prog, tag | static_cast<unsigned>(A.nbk));  // cumulative release after the barrier
    if (A.trace != nullptr && ci == 0 && gi == 0) A.trace[(A.nbk - 1) * 16 + 2] = gtimer();
  }
}

// HELPER: c_i = op(Dinv_i) (b_i - sum_{d>=2} op(T_(i,i-+d)) x_(i-+d)).
__device__ void helper_task(const SolveArgs& A, int s, int ci, int gi, cd* smem, int* dlist) {
  auto tile_s = [smem](int k) { return smem + k * TILE_S; };
  auto x_s = [smem](int k) { return smem + NS * TILE_S + k * XS; };
  cd* dinv_s = smem + NS * TILE_S + NS * XS;
  cd* acc_s = dinv_s + TILE_S;
  __shared__ int nlist_s;
  __shared__ unsigned long long known_s;  // owner progress last acquired by this CTA
  const Chain ch = A.chains[ci];
  const bool fwd = A.fwd != 0;
  const bool opH = ch.mode == FWD_UH || ch.mode == BWD_LH;
  const Frag f = frag();
  const int i = fwd ? s : A.nbk - 1 - s;
  const int c0 = gi * CG, nc = min(CG, A.ncols - c0);
  const int64_t ld = A.ld;
  const int J = A.J;
  const unsigned long long* prog = A.prog + static_cast<size_t>(ci) * A.ngroups + gi;
  const unsigned long long tag = static_cast<unsigned long long>(A.epoch) << 32;
  int* fc = A.flags_c + (static_cast<size_t>(ci) * A.ngroups + gi) * A.nbk;
  const bool tr = A.trace != nullptr && ci == 0 && gi == 0 && threadIdx.x == 0;
  if (tr) A.trace[s * 16 + 3] = gtimer();

  // envelope tiles d >= 2 of this block row, farthest first
  if (threadIdx.x == 0) {
    known_s = ld_acquire64(prog);
    int n = 0;
    const int dli = A.dl[i];
    for (int d = J; d >= 2; --d) {
      const bool ok = fwd ? (d <= dli) : (i + d < A.nbk && d <= A.dl[i + d]);
      if (ok) dlist[n++] = d;
    }
    nlist_s = n;
  }
  // b~_i = op(Dinv_i) b_i (or b_i): off the critical path, before any dependency
  cd bval[2];
  if (ch.pre) {
    load_tile(dinv_s, ch.pre + static_cast<size_t>(i) * TT);
    load_x(acc_s, ch.src + static_cast<int64_t>(i) * TILE, ld, c0, nc);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    bval[0] = bval[1] = mk(0.0, 0.0);
    mma_tile(bval, dinv_s, acc_s, opH, f);
  } else {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int c = f.col + q;
      bval[q] = (c < nc) ? ch.src[static_cast<int64_t>(i) * TILE + f.row + (c0 + c) * ld] : mk(0.0, 0.0);
    }
  }
  __syncthreads();
  const int nl = nlist_s;
  unsigned long long known = known_s;  // identical in every thread
  __syncthreads();                     // known_s may be rewritten from here on
  cd acc[2] = {mk(0.0, 0.0), mk(0.0, 0.0)};

  auto dep = [&](int d) { return fwd ? i - d : i + d; };
  auto tile_ptr = [&](int d) -> const cd* { return ch.off + lt_off(fwd ? i : i + d, d, J); };
  // x of block row j is final once the owner has completed step s_j: the owner
  // publishes in order, so one cached frontier covers all farther rows and
  // only a dependency beyond it costs an L2 round trip. The branch is uniform
  // (every thread holds the same `known`); the slow path re-broadcasts it
  // between two barriers.
  auto ensure = [&](int d) {
    const int j = dep(d);
    const unsigned long long target = tag | static_cast<unsigned>((fwd ? j : A.nbk - 1 - j) + 1);
    if (known < target) {
      if (threadIdx.x == 0) {
        unsigned long long v;
        int spins = 0;
        while ((v = ld_acquire64(prog)) < target) {
          if (++spins > 256) __nanosleep(32);
          if (spins > (1 << 25)) {
            atomicExch(A.counter + 2, 1);
            break;
          }
        }
        known_s = v;
      }
      __syncthreads();
      known = known_s;
      __syncthreads();
    }
  };
  // NS-stage cp.async pipeline over the far tiles (d >= NEAR: tile and x
  // prefetched NS-1 entries ahead); the nearest dependencies (d < NEAR) get
  // their tile prefetched but x loaded only right before use.
  constexpr int NEAR = 4;
  auto issue = [&](int e) {
    const int d = dlist[e], buf = e % NS;
    load_tile(tile_s(buf), tile_ptr(d));
    if (d >= NEAR) {
      ensure(d);
      load_x(x_s(buf), ch.dst + static_cast<int64_t>(dep(d)) * TILE, ld, c0, nc);
    }
  };
#pragma unroll
  for (int e = 0; e < NS - 1; ++e) {
    if (e < nl) issue(e);
    cp_async_commit();
  }
  if (tr) A.trace[s * 16 + 10] = gtimer();
  int nfar = 0;
  for (int q = 0; q < nl; ++q) {
    const int buf = q % NS, d = dlist[q];
    if (d >= NEAR) {
      cp_async_wait<NS - 2>();  // entry q landed; entries q+1..q+NS-2 may be in flight
      ++nfar;
    } else {
      if (tr && nfar >= 0) {
        A.trace[s * 16 + 8] = gtimer();
        A.trace[s * 16 + 9] = nfar;
        nfar = -1000;
      }
      ensure(d);
      load_x(x_s(buf), ch.dst + static_cast<int64_t>(dep(d)) * TILE, ld, c0, nc);
      cp_async_commit();
      cp_async_wait<0>();
    }
    // one barrier per tile: entry q is visible to all warps and every warp has
    // finished entry q-1, whose stage the next issue refills
    __syncthreads();
    if (q + NS - 1 < nl) issue(q + NS - 1);
    cp_async_commit();
    mma_tile(acc, tile_s(buf), x_s(buf), opH, f);
  }
  cp_async_wait<0>();
  if (tr) A.trace[s * 16 + 4] = gtimer();
  // c_i = b~_i - acc: no diagonal work left on the critical path
  cd* crow = ch.cbuf + static_cast<int64_t>(i) * TILE + f.row + c0 * ld;
#pragma unroll
  for (int q = 0; q < 2; ++q)
    if (f.col + q < nc) crow[(f.col + q) * ld] = csub(bval[q], acc[q]);
  __syncthreads();
  if (threadIdx.x == 0) {
    st_release(fc + i, A.epoch);  // cumulative release after the barrier
    if (tr) A.trace[s * 16 + 5] = gtimer();
  }
}

__global__ void __launch_bounds__(ST, 2) trsm_kernel(SolveArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cd* smem = reinterpret_cast<cd*>(smem_raw);
  int* dlist = reinterpret_cast<int*>(smem_raw + SMEM_FIXED);
  __shared__ int task_s;
  const int owners = A.nchains * A.ngroups;
  const int ntasks = owners + A.nbk * owners;
  for (;;) {
    if (threadIdx.x == 0) task_s = atomicAdd(A.counter, 1);
    __syncthreads();
    const int t = task_s;
    __syncthreads();
    if (t >= ntasks) break;
    if (t < owners) {
      owner_task(A, t / A.ngroups, t % A.ngroups, smem);
    } else {
      const int h = t - owners;
      const int s = h / owners, rem = h % owners;
      helper_task(A, s, rem / A.ngroups, rem % A.ngroups, smem, dlist);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// DAG-scheduled sweeps over block-sparse factors (nested dissection etc.)
// ---------------------------------------------------------------------------
#ifndef ZOLO_DNS
#define ZOLO_DNS 3
#endif
#ifndef ZOLO_DAG_MINB
#define ZOLO_DAG_MINB 2
#endif
constexpr int DNS = ZOLO_DNS;            // pipeline stages
constexpr int DAG_TRACE_WORDS = 6;       // start, loop end, done, info, wait ns, first tile ready
constexpr int TSW = TT;                  // swizzled (unpadded) tile
constexpr int DAG_SMEM_FIXED = DNS * (TSW + XS2) * static_cast<int>(sizeof(cd));

struct DagArgs {
  const Chain* chains;
  const int* recs;  // ntask x DAG_REC task records (band.cuh)
  int ntask, nslots;
  int nchains, ngroups, ncols, epoch, fwd;
  int64_t ld, ldp;
  SpGeom s;
  int* flags;    // per (chain, 32-column group, block): epoch when u_i is final
  int* cflags;   // per (chain, 32-column group, slot): epoch when the partial sum is written
  int* counter;  // [0] task counter, [2] wait-timeout error word
  unsigned long long* trace;  // optional: per task (start, dependencies done, done, smid<<48|chunk<<47|i<<16|deps)
  int hints;                  // L2 eviction-priority hints on (development switch ZOLO_DAG_HINTS)
  const int* tmap;            // v2, optional: claim slot k -> record * nchains + chain (groups consecutive)
  int presw;                  // tiles stored pre-swizzled (swizzle_tiles): linear / bulk copies
  int l2pf;                   // v2: L2 prefetch of the next task's tiles / blocks (ZOLO_DAG_L2PF)
  // v2 fused forward + backward launch (dag_fused_launch): the backward sweep's schedule and
  // chains; backward tasks run at epoch + 1 and the tmap entries carry bit 30 for them
  int fused = 0;
  const int* recs_b = nullptr;
  const Chain* chains_b = nullptr;
  int ntask_b = 0, nslots_b = 0;
  int64_t ldp_b = 0;
  int cfs = 0;  // chunk-flag stride per (chain, group): one for both directions, so they never alias
  // ready-queue scheduling: tasks are popped when all their dependencies are done (no claimed
  // task ever waits); the first q_ninit x per_step pops are the initially ready records
  int queue = 0;
  const int* q_cnt0 = nullptr;
  const int* q_dptr = nullptr;
  const int* q_didx = nullptr;
  const int* q_init = nullptr;
  int q_ninit = 0;
  int* q_cnt = nullptr;  // per task: dependencies completed
  int* q_arr = nullptr;  // pushed task ids + 1
  int* q_ctr = nullptr;  // [0] pops, [1] pushes
  // lagged GMRES control (capi apply_filter_impl): the launch covers a superset of the columns
  // still running; a task whose column group has converged entirely is skipped
  const int* gact = nullptr;
  const int* gdone = nullptr;
};

__device__ __forceinline__ int atom_add_acq_rel(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// a tile into the swizzled shared layout: permuted on the way (column-major global
// tile) or copied linearly (tile stored pre-swizzled)
__device__ __forceinline__ void load_tile_any(cd* s, const cd* g, unsigned long long pol, int presw) {
  if (!presw) {
    load_tile_sw(s, g, pol);
    return;
  }
#pragma unroll
  for (int q = 0; q < TT / ST; ++q) {
    const int e = threadIdx.x + q * ST;
    cp_async16_cg_hint(&s[e], g + e, pol);
  }
}

// every thread spins on a share of cnt flags; the barrier publishes them all
__device__ __forceinline__ void wait_flags_par(const int* f, int cnt, int epoch, int* err) {
  for (int p = threadIdx.x; p < cnt; p += ST) {
    int spins = 0;
    while (ld_acquire(f + p) < epoch) {
      if (++spins > 256) __nanosleep(32);
      if (spins > (1 << 25)) {
        atomicExch(err, 1);
        break;
      }
    }
  }
  __syncthreads();
}

// One (task record, chain, 32-column group):
//   row task:   u_i = pre(b_i) - sum_q op(T~(i, j_q)) u_(j_q) - sum_p partial_p
//   chunk task: partial_out = sum_q op(T~(i, j_q)) u_(j_q)
// The pre-transform op(Dinv_i) b_i is pipeline entry 0 with a negated A
// operand, so the accumulator holds S = sum - pre(b) and u_i = -S: no
// serialised prologue. Dependencies come in processing order (earliest
// completed first); their flags are read once, in parallel, at task start,
// so only dependencies still running cost a wait. `rec` is in shared memory
// (prefetched by the previous task); `nrec` is where this task prefetches the
// record of `next` (the CTA's next claimed task) once its first barrier passed.
__device__ void dag_task(const DagArgs& A, const int* rec, int ci, int gi, cd* smem, int* rdy_s, int* nrec,
                         int next_rec, unsigned long long* trc, uint2* mask_s) {
  auto tile_s = [smem](int k) { return smem + k * (TSW + XS2); };
  auto x_s = [smem](int k) { return smem + k * (TSW + XS2) + TSW; };
  const Chain ch = A.chains[ci];
  const int i = rec[0], nd = rec[1], pa = rec[2], pc = rec[3], out = rec[4];
  const int* dq = rec + DAG_REC_HDR;  // (j, tile id) pairs
  const bool chunk = out >= 0;
  const bool opH = ch.mode == FWD_UH || ch.mode == BWD_LH;
  const Frag f = frag();
  const int c0 = gi * DCG, nc = min(DCG, A.ncols - c0);
  const int64_t ld = A.ld;
  const size_t cgi = static_cast<size_t>(ci) * A.ngroups + gi;
  int* flags = A.flags + cgi * A.s.nb;
  int* cflags = A.cflags + cgi * A.nslots;
  const int hp = (!chunk && ch.pre) ? 1 : 0;  // entry 0 = pre-transform
  const int ne = hp + nd;
  // factor tiles and right-hand sides stream through L2 once per column group;
  // the solution blocks u_j are re-read by every later block row that depends on them
  const unsigned long long pol_stream = (A.hints & 1) ? l2_evict_first() : l2_evict_normal();
  const unsigned long long pol_keep = (A.hints & 2) ? l2_evict_last() : l2_evict_normal();
  // tile + occupancy mask of entry e (and the right-hand side for the pre entry): no producer involved
  auto issue_tile = [&](int e) {
    const int buf = e % DNS;
    const uint2* mk_src;
    if (e < hp) {
      load_tile_any(tile_s(buf), ch.pre + static_cast<size_t>(i) * TT, pol_stream, A.presw);
      load_x32(x_s(buf), ch.src + static_cast<int64_t>(i) * TILE, ld, c0, nc, pol_stream);
      mk_src = ch.prem ? ch.prem + i : nullptr;
    } else {
      const int q = e - hp;
      load_tile_any(tile_s(buf), ch.off + static_cast<size_t>(dq[2 * q + 1]) * TT, pol_stream, A.presw);
      mk_src = ch.offm ? ch.offm + dq[2 * q + 1] : nullptr;
    }
    if (threadIdx.x == 0) {
      if (mk_src)
        cp_async8_ca(mask_s + buf, mk_src);
      else
        mask_s[buf] = make_uint2(0xffffffffu, 0xffffffffu);
    }
  };
  // u_j of a dependency entry, when its producer had finished at task start
  auto issue_x = [&](int e) {
    if (e < hp) return;
    const int q = e - hp;
    if (rdy_s[q]) load_x32(x_s(e % DNS), ch.dst + static_cast<int64_t>(dq[2 * q]) * TILE, ld, c0, nc, pol_keep);
  };
  auto issue = [&](int e) {
    issue_tile(e);
    issue_x(e);
  };
  // prologue: the first tiles load while the dependency flags are read
#pragma unroll
  for (int e = 0; e < DNS - 1; ++e)
    if (e < ne) issue_tile(e);
  for (int q = threadIdx.x; q < nd; q += ST) rdy_s[q] = ld_acquire(flags + dq[2 * q]) >= A.epoch;
  cd bval[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int c = ocol(f, q);
    bval[q] = (!chunk && !ch.pre && c < nc) ? ch.src[static_cast<int64_t>(i) * TILE + f.row + (c0 + c) * ld]
                                            : mk(0.0, 0.0);
  }
  __syncthreads();
  if (next_rec >= 0 && threadIdx.x < DAG_REC * 4 / 16)  // prefetch the next task's record
    cp_async16_cg(nrec + 4 * threadIdx.x, A.recs + static_cast<size_t>(next_rec) * DAG_REC + 4 * threadIdx.x);
  auto ready = [&](int e) { return e < hp || rdy_s[e - hp]; };
#pragma unroll
  for (int e = 0; e < DNS - 1; ++e) {
    if (e < ne) issue_x(e);
    cp_async_commit();
  }
  Acc8 acc8;
  acc8_zero(acc8);
  cd acc[4] = {mk(0.0, 0.0), mk(0.0, 0.0), mk(0.0, 0.0), mk(0.0, 0.0)};  // chunk partials
  unsigned long long wsum = 0, tw = 0;  // (trace) time spent waiting on producers
  if (pc > 0) {  // partial sums of the older dependencies, while the first tiles load
    if (trc) tw = gtimer();
    wait_flags_par(cflags + pa, pc, A.epoch, A.counter + 2);
    if (trc) wsum += gtimer() - tw;
    const cd* prow = ch.cbuf + static_cast<int64_t>(pa) * TILE + f.row + c0 * A.ldp;
    for (int p = 0; p < pc; ++p) {
      cd v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = ocol(f, q);
        v[q] = (c < nc) ? __ldcg(prow + static_cast<int64_t>(p) * TILE + c * A.ldp) : mk(0.0, 0.0);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = cadd(acc[q], v[q]);
    }
  }
  for (int e = 0; e < ne; ++e) {
    const int buf = e % DNS;
    if (ready(e)) {
      cp_async_wait<DNS - 2>();
    } else {  // still running at task start: wait for it now, then fetch its u
      const int j = dq[2 * (e - hp)];
      if (trc) tw = gtimer();
      wait_flag(flags + j, A.epoch, A.counter + 2);
      if (trc) wsum += gtimer() - tw;
      load_x32(x_s(buf), ch.dst + static_cast<int64_t>(j) * TILE, ld, c0, nc, pol_keep);
      cp_async_commit();
      cp_async_wait<0>();
    }
    // one barrier per tile: entry e visible to all warps, entry e-1 finished
    __syncthreads();
    if (trc && e == 0 && threadIdx.x == 0) trc[5] = gtimer();
    if (e + DNS - 1 < ne) issue(e + DNS - 1);
    cp_async_commit();
    const uint2 mw = mask_s[buf];
    mma_tile2(acc8, tile_s(buf), x_s(buf), opH, e < hp, f, ((opH ? mw.y : mw.x) >> f.r0) & 0xffu);
  }
  cp_async_wait<0>();
  if (trc && threadIdx.x == 0) trc[1] = gtimer();
  {
    cd prod[4];
    acc8_fold(acc8, prod);
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q] = cadd(acc[q], prod[q]);
  }
  if (chunk) {
    cd* prow = ch.cbuf + static_cast<int64_t>(out) * TILE + f.row + c0 * A.ldp;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = ocol(f, q);
      if (c < nc) prow[c * A.ldp] = acc[q];
    }
  } else {
    cd* urow = ch.dst + static_cast<int64_t>(i) * TILE + f.row + c0 * ld;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = ocol(f, q);
      if (c < nc) urow[c * ld] = csub(bval[q], acc[q]);  // hp: bval = 0, acc = S
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    st_release(chunk ? cflags + out : flags + i, A.epoch);  // cumulative release after the barrier
    if (trc) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      trc[2] = gtimer();
      trc[4] = wsum;
      trc[3] = (static_cast<unsigned long long>(smid) << 48) | (static_cast<unsigned long long>(chunk) << 47) |
               (static_cast<unsigned long long>(i) << 16) | static_cast<unsigned>(nd);
    }
  }
}

// Persistent CTAs claim (record, chain, group) tasks in schedule order; each
// claims its NEXT task when it starts the current one and prefetches that
// task's record behind the current tile pipeline.
__global__ void __launch_bounds__(ST, ZOLO_DAG_MINB) dag_kernel(DagArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cd* smem = reinterpret_cast<cd*>(smem_raw);
  int* recb = reinterpret_cast<int*>(smem_raw + DAG_SMEM_FIXED);  // 2 x DAG_REC
  int* rdy_s = recb + 2 * DAG_REC;
  __shared__ int cur_s, next_s;
  __shared__ uint2 mask_s[DNS];
  const int per_step = A.nchains * A.ngroups;
  const int ntasks = A.ntask * per_step;
  if (threadIdx.x == 0) cur_s = atomicAdd(A.counter, 1);
  __syncthreads();
  int t = cur_s, b = 0;
  if (t < ntasks && threadIdx.x < DAG_REC * 4 / 16)
    cp_async16_cg(recb + 4 * threadIdx.x, A.recs + static_cast<size_t>(t / per_step) * DAG_REC + 4 * threadIdx.x);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  while (t < ntasks) {
    unsigned long long* trc = A.trace ? A.trace + DAG_TRACE_WORDS * static_cast<size_t>(t) : nullptr;
    if (trc && threadIdx.x == 0) trc[0] = gtimer();
    if (threadIdx.x == 0) next_s = atomicAdd(A.counter, 1);
    __syncthreads();
    const int tn = next_s;
    const int rem = t % per_step;
    dag_task(A, recb + b * DAG_REC, rem / A.ngroups, rem % A.ngroups, smem, rdy_s, recb + (b ^ 1) * DAG_REC,
             tn < ntasks ? tn / per_step : -1, trc, mask_s);
    __syncthreads();  // (dag_task ends with cp.async.wait_all: the next record has landed)
    t = tn;
    b ^= 1;
  }
}

// ---------------------------------------------------------------------------
// Warp-specialised DAG sweep (v2): one persistent CTA per SM = 8 consumer warps
// (DMMA) + 1 producer warp. The producer claims tasks, waits on their producers'
// flags and streams (tile, u_j) / add-block entries into an NST2-deep ring of
// shared-memory stages with cp.async + mbarriers, running ahead across task
// boundaries; consumers never touch global memory except for the task's output,
// and no CTA-wide barrier sits on the per-tile path.
// ---------------------------------------------------------------------------
#ifndef ZOLO_NST2
#define ZOLO_NST2 3
#endif
#ifndef ZOLO_V2_MINB
#define ZOLO_V2_MINB 2
#endif
constexpr int NST2 = ZOLO_NST2;
constexpr int P2T = ST + 32;  // threads: 8 consumer warps + the producer warp
struct Meta2 {
  int kind;  // 0 MMA(tile, x, neg = sign), 1 ADD(x block * sign), 2 END
  int sign;
  unsigned mx, my;  // occupancy mask (op N / op H)
  int last, i, ci, gi, out, nc, pad0, pad1;
};
constexpr int DAG2_CHAINS = 32;
constexpr int DAG2_SMEM = NST2 * (TSW + XS2) * static_cast<int>(sizeof(cd)) + NST2 * static_cast<int>(sizeof(Meta2)) +
                          2 * NST2 * 8 + 2 * DAG2_CHAINS * static_cast<int>(sizeof(Chain)) + DAG_REC * 4;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, int count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, int parity) {
  const unsigned a = smem_u32(b);
  unsigned ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
// bulk (TMA-engine) global -> shared copy completing `bytes` on the mbarrier's transaction count
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                          unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void l2_prefetch(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(ST) : "memory"); }

// lane 0 spins on *f >= epoch (bounded), then the warp reconverges
__device__ __forceinline__ void warp_wait_flag(const int* f, int epoch, int* err) {
  if ((threadIdx.x & 31) == 0) {
    int spins = 0;
    while (ld_acquire(f) < epoch) {
      if (++spins > 64) __nanosleep(64);
      if (spins > (1 << 24)) {
        atomicExch(err, 1);
        break;
      }
    }
  }
  __syncwarp();
}

__global__ void __launch_bounds__(P2T, ZOLO_V2_MINB) dag2_kernel(DagArgs A) {
  extern __shared__ __align__(16) unsigned char sm2[];
  cd* ring = reinterpret_cast<cd*>(sm2);
  Meta2* meta = reinterpret_cast<Meta2*>(sm2 + NST2 * (TSW + XS2) * sizeof(cd));
  unsigned long long* full = reinterpret_cast<unsigned long long*>(meta + NST2);
  unsigned long long* empty = full + NST2;
  Chain* chs = reinterpret_cast<Chain*>(empty + NST2);
  int* recp = reinterpret_cast<int*>(chs + 2 * DAG2_CHAINS);
  auto tile_s = [ring](int s) { return ring + s * (TSW + XS2); };
  auto x_s = [ring](int s) { return ring + s * (TSW + XS2) + TSW; };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int q = threadIdx.x; q < A.nchains; q += blockDim.x) {
    chs[q] = A.chains[q];
    if (A.fused) chs[DAG2_CHAINS + q] = A.chains_b[q];
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST2; ++s) {
      mbar_init(full + s, 1);    // the producer's arrive (+ the stage's bulk-copy bytes)
      mbar_init(empty + s, ST / 32);
    }
  }
  __syncthreads();
  const int per_step = A.nchains * A.ngroups;
  const int ntasks_f = A.ntask * per_step;
  const int ntasks = ntasks_f + (A.fused ? A.ntask_b * per_step : 0);
  if (warp == ST / 32) {
    // ------------------------------ producer ------------------------------
    const unsigned long long pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
    int g = 0;
    // one ring entry: tile (optional) + a 32 x 32 block with column stride `stride`
    int cur_t = 0;  // claim index of the task being produced (trace)
    int cur_dir = 0;  // fused launch: 1 while producing a backward task
    auto produce = [&](int kind, int sign, const cd* tile, uint2 mw, const cd* blk, int64_t stride, int c0,
                       int nc, unsigned long long pol, int last, int i, int ci, int gi, int out) {
      const int s = g % NST2, round = g / NST2;
      mbar_wait(empty + s, (round & 1) ^ 1);
      // bulk copies: the (pre-swizzled) tile in one, the block's columns one per lane
      const unsigned bytes = (tile ? static_cast<unsigned>(TT * sizeof(cd)) : 0u) +
                             static_cast<unsigned>(nc) * TILE * static_cast<unsigned>(sizeof(cd));
      if (lane == 0) mbar_expect_tx(full + s, bytes);
      __syncwarp();
      if (tile && lane == 0) bulk_copy(tile_s(s), tile, TT * sizeof(cd), full + s, pol_stream);
      cd* xs = x_s(s);
#ifdef ZOLO_XPROBE  // (development timing probe, wrong results) one contiguous copy per block
      if (lane == 0) bulk_copy(xs, blk + c0 * stride, nc * TILE * sizeof(cd), full + s, pol);
#else
      if (lane < nc)
        bulk_copy(xs + lane * XPAD, blk + (c0 + lane) * stride, TILE * sizeof(cd), full + s, pol);
      else
        for (int r = 0; r < TILE; ++r) xs[lane * XPAD + r] = mk(0.0, 0.0);
#endif
      __syncwarp();
      if (lane == 0) {
        Meta2 m;
        m.kind = kind;
        m.sign = sign;
        m.mx = mw.x;
        m.my = mw.y;
        m.last = last;
        m.i = i;
        m.ci = ci;
        m.gi = gi;
        m.out = out;
        m.nc = nc;
        m.pad0 = cur_t;
        m.pad1 = cur_dir;
        meta[s] = m;
        mbar_arrive(full + s);
      }
      ++g;
    };
    auto decode = [&](int tt, int& r, int& ci, int& gi, int& dir) {
      if (A.tmap) {  // chains staggered in the claim order (each chain keeps its topological order)
        int rc = A.tmap[tt / A.ngroups];
        dir = (rc >> 30) & 1;
        rc &= (1 << 30) - 1;
        r = rc / A.nchains;
        ci = rc % A.nchains;
        gi = tt % A.ngroups;
      } else {
        dir = tt >= ntasks_f;
        if (dir) tt -= ntasks_f;
        r = tt / per_step;
        const int rem = tt % per_step;
        ci = rem / A.ngroups;
        gi = rem % A.ngroups;
      }
    };
    auto recs_of = [&](int dir) { return dir ? A.recs_b : A.recs; };
    // lagged GMRES control: the column groups whose columns have all converged (read once)
    unsigned gmask = 0;
    if (A.gdone && A.ngroups <= 32) {
      for (int gg = 0; gg < A.ngroups; ++gg) {
        const int cg0 = gg * DCG, ncg = min(DCG, A.ncols - cg0);
        if (__all_sync(0xffffffffu, lane >= ncg || A.gdone[A.gact[cg0 + lane]] != 0)) gmask |= 1u << gg;
      }
      if (gmask == (A.ngroups == 32 ? ~0u : (1u << A.ngroups) - 1u)) {  // nothing left: leave at once
        produce(2, 0, nullptr, make_uint2(0u, 0u), A.chains[0].src, 0, 0, 0, pol_stream, 1, 0, 0, 0, -1);
        return;
      }
    }
    // ready queue: pop position -> task id (the initial records directly, later ones once pushed)
    const int q_base = A.q_ninit * per_step;
    auto resolve = [&](int pos) {
      int id = ntasks;
      if (lane == 0 && pos < ntasks) {
        if (pos < q_base) {
          id = A.q_init[pos / per_step] * per_step + pos % per_step;
        } else {
          int spins = 0;
          while ((id = ld_acquire(A.q_arr + (pos - q_base))) == 0) {
            if (++spins > 64) __nanosleep(64);
            if (spins > (1 << 26)) {
              atomicExch(A.counter + 2, 1);
              break;
            }
          }
          id = id > 0 ? id - 1 : ntasks;
        }
      }
      return __shfl_sync(0xffffffffu, id, 0);
    };
    // Claims run two tasks ahead: when task T starts, T+1's id has arrived (its record load is
    // issued now and lands while T streams) and the atomic for T+2 goes out. (Ready-queue mode:
    // one task at a time, popped when the previous one has been issued.)
    int t = 0;
    if (lane == 0) t = atomicAdd(A.queue ? A.q_ctr : A.counter, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (A.queue) t = resolve(t);
    int rec_lo = 0, rec_hi = 0;  // this lane's two words of the current task's record
    if (t < ntasks) {
      int r0, c0_, g0_, d0_;
      decode(t, r0, c0_, g0_, d0_);
      rec_lo = recs_of(d0_)[static_cast<size_t>(r0) * DAG_REC + lane];
      rec_hi = recs_of(d0_)[static_cast<size_t>(r0) * DAG_REC + lane + 32];
    }
    int tn_raw = 0;
    if (lane == 0 && !A.queue) tn_raw = atomicAdd(A.counter, 1);
    for (;;) {
      if (t >= ntasks) {
        produce(2, 0, nullptr, make_uint2(0u, 0u), A.chains[0].src, 0, 0, 0, pol_stream, 1, 0, 0, 0, -1);
        break;
      }
      const int tn = A.queue ? ntasks : __shfl_sync(0xffffffffu, tn_raw, 0);
      int nrec_lo = 0, nrec_hi = 0;
      if (tn < ntasks) {
        int rn_, cn_, gn_, dn_;
        decode(tn, rn_, cn_, gn_, dn_);
        nrec_lo = recs_of(dn_)[static_cast<size_t>(rn_) * DAG_REC + lane];
        nrec_hi = recs_of(dn_)[static_cast<size_t>(rn_) * DAG_REC + lane + 32];
      }
      if (lane == 0 && !A.queue) tn_raw = atomicAdd(A.counter, 1);
      if (A.l2pf && tn < ntasks) {
        // warm L2 with the next task's tiles and solution blocks while this one streams
        int rn, cin, gin;
        if (A.tmap) {
          const int rc = A.tmap[tn / A.ngroups];
          rn = rc / A.nchains;
          cin = rc % A.nchains;
          gin = tn % A.ngroups;
        } else {
          rn = tn / per_step;
          cin = (tn % per_step) / A.ngroups;
          gin = (tn % per_step) % A.ngroups;
        }
        const int* rgn = A.recs + static_cast<size_t>(rn) * DAG_REC;
        const int in = rgn[0], ndn = rgn[1], outn = rgn[4];
        const Chain& chn = chs[cin];
        const int c0n = gin * DCG, ncn = min(DCG, A.ncols - c0n);
        const cd* tsrc = nullptr;
        const cd* xsrc = nullptr;
        if (lane < ndn) {
          tsrc = chn.off + static_cast<size_t>(rgn[DAG_REC_HDR + 2 * lane + 1]) * TT;
          xsrc = chn.dst + static_cast<int64_t>(rgn[DAG_REC_HDR + 2 * lane]) * TILE;
        } else if (lane == ndn && outn < 0) {
          tsrc = chn.pre ? chn.pre + static_cast<size_t>(in) * TT : nullptr;
          xsrc = chn.src + static_cast<int64_t>(in) * TILE;
        }
        if (tsrc) l2_prefetch(tsrc, TT * sizeof(cd));
        if (xsrc)
          for (int c = 0; c < ncn; ++c) l2_prefetch(xsrc + (c0n + c) * A.ld, TILE * sizeof(cd));
      }
      cur_t = t;
      unsigned long long* trp = A.trace ? A.trace + DAG_TRACE_WORDS * static_cast<size_t>(t) : nullptr;
      unsigned long long wsum = 0;
      if (trp && lane == 0) trp[0] = gtimer();
      int r, ci, gi, dir;
      decode(t, r, ci, gi, dir);
      cur_dir = dir;
      const int epoch = A.epoch + dir;
      const int64_t ldp = dir ? A.ldp_b : A.ldp;
      recp[lane] = rec_lo;
      recp[lane + 32] = rec_hi;
      __syncwarp();
      const int i = recp[0], nd = recp[1], pa = recp[2], pc = recp[3], out = recp[4], tf = recp[5];
      const bool chunk = out >= 0;
      // task kinds of the selectively inverted trailing block (host.hpp DT_*)
      const bool slotdep = tf & DT_SLOTDEP, srcdep = tf & DT_SRCDEP, invdep = slotdep || srcdep;
      const bool bentry = (!chunk || (tf & DT_BENTRY)) && !(tf & DT_NOB);
      const Chain& ch = chs[ci + dir * DAG2_CHAINS];
      const int c0 = gi * DCG, nc = min(DCG, A.ncols - c0);
      const size_t cgi = static_cast<size_t>(ci) * A.ngroups + gi;
      const int* flags = A.flags + cgi * A.s.nb;
      const int* cflags = A.cflags + cgi * A.cfs;
      const int* dflags = slotdep ? cflags : flags;  // where dependency q's readiness lives
      // every task of a fully converged column group skips (its dependents are in the same group)
      const bool skip = (gmask >> gi) & 1u;
      if (!skip) {
      // occupancy masks of all the task's tiles (lane q: dependency q, lane 31: the pre-transform)
      // and readiness of every dependency, each read in parallel (one round trip)
      uint2 my_mask = make_uint2(0xffffffffu, 0xffffffffu);
      if (lane < nd) {
        if (ch.offm && !invdep) my_mask = ch.offm[recp[DAG_REC_HDR + 2 * lane + 1]];
      } else if (lane == 31 && bentry && ch.pre && ch.prem) {
        my_mask = ch.prem[i];
      }
      const unsigned dep_ready = __ballot_sync(
          0xffffffffu,
          lane >= nd || srcdep || A.queue || ld_acquire(dflags + recp[DAG_REC_HDR + 2 * lane]) >= epoch);
      auto mask_of = [&](int q) {
        return make_uint2(__shfl_sync(0xffffffffu, my_mask.x, q), __shfl_sync(0xffffffffu, my_mask.y, q));
      };
      const int nent = (bentry ? 1 : 0) + pc + nd;
      int e = 0;
      // fused launch: a backward task's b_i is the forward sweep's u_i of the same chain, which may
      // still be in flight when the task is claimed (claims are topological, completions are not)
      if (A.fused && dir && bentry && ld_acquire(flags + i) < A.epoch) {
        const unsigned long long tw = trp ? gtimer() : 0;
        warp_wait_flag(flags + i, A.epoch, A.counter + 2);
        if (trp) wsum += gtimer() - tw;
      }
      if (bentry) {
        ++e;
        const uint2 pm = mask_of(31);
        if (ch.pre)
          produce(0, 1, ch.pre + static_cast<size_t>(i) * TT, pm, ch.src + static_cast<int64_t>(i) * TILE, A.ld, c0,
                  nc, pol_stream, e == nent, i, ci + dir * DAG2_CHAINS, gi, out);
        else
          produce(1, -1, nullptr, pm, ch.src + static_cast<int64_t>(i) * TILE, A.ld, c0, nc, pol_stream, e == nent,
                  i, ci + dir * DAG2_CHAINS, gi, out);
      }
      for (int p0 = 0; p0 < pc; p0 += 32) {
        const unsigned prdy = __ballot_sync(
            0xffffffffu, p0 + lane >= pc || A.queue || ld_acquire(cflags + pa + p0 + lane) >= epoch);
        for (int p = p0; p < pc && p < p0 + 32; ++p) {
          if (!((prdy >> (p - p0)) & 1u)) {
            const unsigned long long tw = trp ? gtimer() : 0;
            warp_wait_flag(cflags + pa + p, epoch, A.counter + 2);
            if (trp) wsum += gtimer() - tw;
          }
          ++e;
          produce(1, 1, nullptr, make_uint2(0xffffffffu, 0xffffffffu), ch.cbuf + static_cast<int64_t>(pa + p) * TILE,
                  ldp, c0, nc, pol_stream, e == nent, i, ci + dir * DAG2_CHAINS, gi, out);
        }
      }
      for (int q = 0; q < nd; ++q) {
        const int j = recp[DAG_REC_HDR + 2 * q], tid = recp[DAG_REC_HDR + 2 * q + 1];
        if (!((dep_ready >> q) & 1u)) {
          const unsigned long long tw = trp ? gtimer() : 0;
          warp_wait_flag(dflags + j, epoch, A.counter + 2);
          if (trp) wsum += gtimer() - tw;
        }
        ++e;
        const int cix = ci + dir * DAG2_CHAINS;
        if (!invdep)
          produce(0, 0, ch.off + static_cast<size_t>(tid) * TT, mask_of(q), ch.dst + static_cast<int64_t>(j) * TILE,
                  A.ld, c0, nc, pol_keep, e == nent, i, cix, gi, out);
        else if (slotdep)  // M(i,k) S_k, S_k = -c_k from its slot
          produce(0, 0, ch.minv + static_cast<size_t>(tid) * TT, mask_of(q),
                  ch.cbuf + static_cast<int64_t>(j) * TILE, ldp, c0, nc, pol_stream, e == nent, i, cix, gi, out);
        else  // -W(i,k) b_k (b_k staged into slot j before the launch: the sweep runs in place)
          produce(0, 1, ch.minv + static_cast<size_t>(tid) * TT, mask_of(q), ch.cbuf + static_cast<int64_t>(j) * TILE,
                  ldp, c0, nc, pol_stream, e == nent, i, cix, gi, out);
      }
      }  // !skip
      __syncwarp();
      if (trp && lane == 0) {
        trp[4] = wsum;
        trp[5] = gtimer();
      }
      if (A.queue) {  // pop the next ready task and load its record
        int pos = 0;
        if (lane == 0) pos = atomicAdd(A.q_ctr, 1);
        t = resolve(__shfl_sync(0xffffffffu, pos, 0));
        if (t < ntasks) {
          int rq, cq, gq, dq;
          decode(t, rq, cq, gq, dq);
          rec_lo = recs_of(dq)[static_cast<size_t>(rq) * DAG_REC + lane];
          rec_hi = recs_of(dq)[static_cast<size_t>(rq) * DAG_REC + lane + 32];
        }
      } else {
        t = tn;
        rec_lo = nrec_lo;
        rec_hi = nrec_hi;
      }
    }
    return;
  }
  // ------------------------------ consumers ------------------------------
  const Frag f = frag();
  Acc8 acc;
  acc8_zero(acc);
  int ntiles_task = 0;  // (trace) tile products of the current task
  for (int g = 0;; ++g) {
    const int s = g % NST2, round = g / NST2;
    mbar_wait(full + s, round & 1);
    const Meta2 m = meta[s];
    if (m.kind == 2) break;
    const Chain& ch = chs[m.ci];
    const bool opH = ch.mode == FWD_UH || ch.mode == BWD_LH;
    const int mdir = m.pad1;
    ntiles_task += m.kind == 0;
    if (m.kind == 0) {
      mma_tile2(acc, tile_s(s), x_s(s), opH, m.sign != 0, f, ((opH ? m.my : m.mx) >> f.r0) & 0xffu);
#ifdef ZOLO_DMMA2X  // (development timing probe, wrong results) twice the tensor work per stage
      mma_tile2(acc, tile_s(s), x_s(s), opH, m.sign != 0, f, ((opH ? m.my : m.mx) >> f.r0) & 0xffu);
#endif
    } else {
      const cd* xs = x_s(s);
      const double sg = static_cast<double>(m.sign);
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int e2 = 0; e2 < 2; ++e2) {
          const cd v = xs[ocol(f, 2 * h + e2) * XPAD + f.row];
          acc.v[h][0][0][e2] += sg * v.x;
          acc.v[h][0][1][e2] += sg * v.y;
        }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + s);
    if (m.last) {
      cd o[4];
      acc8_fold(acc, o);
      acc8_zero(acc);
      const bool chunk = m.out >= 0;
      const int c0 = m.gi * DCG;
      if (chunk) {
        const int64_t ldp = mdir ? A.ldp_b : A.ldp;
        cd* prow = ch.cbuf + static_cast<int64_t>(m.out) * TILE + f.row + c0 * ldp;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = ocol(f, q);
          if (c < m.nc) prow[c * ldp] = o[q];
        }
      } else {
        cd* urow = ch.dst + static_cast<int64_t>(m.i) * TILE + f.row + c0 * A.ld;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = ocol(f, q);
          if (c < m.nc) urow[c * A.ld] = mk(-o[q].x, -o[q].y);
        }
      }
      consumers_sync();
      if (threadIdx.x == 0) {
        const size_t cgi = static_cast<size_t>(m.ci - mdir * DAG2_CHAINS) * A.ngroups + m.gi;
        st_release(chunk ? A.cflags + cgi * A.cfs + m.out : A.flags + cgi * A.s.nb + m.i, A.epoch + mdir);
      }
      if (A.queue) {  // this task is done: count it in its dependents and push the ones now ready
        consumers_sync();
        __threadfence();
        const int r = m.pad0 / (A.nchains * A.ngroups), rem = m.pad0 % (A.nchains * A.ngroups);
        for (int q = A.q_dptr[r] + static_cast<int>(threadIdx.x); q < A.q_dptr[r + 1]; q += ST) {
          const int d = A.q_didx[q];
          const int idd = d * A.nchains * A.ngroups + rem;
          if (atom_add_acq_rel(A.q_cnt + idd, 1) + 1 == A.q_cnt0[d]) {
            const int pos = atomicAdd(A.q_ctr + 1, 1);
            st_release(A.q_arr + pos, idd + 1);
          }
        }
      }
      if (threadIdx.x == 0) {
        if (A.trace) {
          unsigned long long* trc = A.trace + DAG_TRACE_WORDS * static_cast<size_t>(m.pad0);
          unsigned smid;
          asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
          trc[2] = gtimer();
          trc[3] = (static_cast<unsigned long long>(smid) << 48) | (static_cast<unsigned long long>(chunk) << 47) |
                   (static_cast<unsigned long long>(m.i) << 16) | static_cast<unsigned>(ntiles_task);
        }
      }
      ntiles_task = 0;
    }
  }
}

// cbuf[dst_row0 + r, c] = src[row0 + r, c] for every chain: the sweep input of the selectively
// inverted block staged where the in-place backward sweep cannot overwrite it (host.hpp DT_SRCDEP)
__global__ void stage_rows_kernel(const Chain* chains, int64_t row0, int64_t rows, int64_t ld, int64_t ldp,
                                  int64_t dst_row0) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  const Chain& ch = chains[blockIdx.z];
  const int64_t c = blockIdx.y;
  ch.cbuf[dst_row0 + r + c * ldp] = ch.src[row0 + r + c * ld];
}

// x_i <- op(D_i) x_i per (block row, 16-column group): the adjoint post-pass.
__global__ void __launch_bounds__(ST) blockdiag_kernel(const cd* D, bool opH, cd* x, int ncols, int64_t ld,
                                                      int swizzled) {
  __shared__ __align__(16) cd ds[TILE_S];
  __shared__ __align__(16) cd xs[XS];
  const int i = blockIdx.x, c0 = blockIdx.y * CG, nc = min(CG, ncols - c0);
  const Frag f = frag();
  if (swizzled) {  // undo the sweep layout into the padded column-major copy
    const cd* g = D + static_cast<size_t>(i) * TT;
#pragma unroll
    for (int q = 0; q < TT / ST; ++q) {
      const int e = threadIdx.x + q * ST, col = e / TILE, row = e % TILE;
      cp_async16_cg(&ds[col * APAD + row], g + col * TILE + (row ^ swz(col)));
    }
  } else {
    load_tile(ds, D + static_cast<size_t>(i) * TT);
  }
  load_x(xs, x + static_cast<int64_t>(i) * TILE, ld, c0, nc);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  cd out[2] = {mk(0.0, 0.0), mk(0.0, 0.0)};
  mma_tile(out, ds, xs, opH, f);
  cd* row = x + static_cast<int64_t>(i) * TILE + f.row + c0 * ld;
#pragma unroll
  for (int q = 0; q < 2; ++q)
    if (f.col + q < nc) row[(f.col + q) * ld] = out[q];
}

}  // namespace

void blockdiag_apply(cudaStream_t st, int nb, const cd* D, bool opH, cd* x, int ncols, int64_t ld, bool swizzled) {
  if (ncols > 0)
    blockdiag_kernel<<<dim3(nb, (ncols + CG - 1) / CG), ST, 0, st>>>(D, opH, x, ncols, ld, swizzled ? 1 : 0);
}

int dag_groups(int ncols) { return (ncols + DCG - 1) / DCG; }

void dag_stage_inputs(cudaStream_t st, const Chain* d_chains, int nchains, int64_t row0, int64_t rows, int ncols,
                      int64_t ld, int64_t ldp, int64_t dst_row0) {
  if (rows <= 0 || ncols <= 0 || nchains <= 0) return;
  stage_rows_kernel<<<dim3(static_cast<unsigned>((rows + 255) / 256), ncols, nchains), 256, 0, st>>>(
      d_chains, row0, rows, ld, ldp, dst_row0);
}

// Forward and backward sweeps of all chains in ONE persistent launch (v2 kernel): backward tasks
// (epoch + 1) are claimed after the forward tasks of their chain (tmap bit 30), and a backward
// root waits on the forward flag of its own row (DT_FWDWAIT) -- every other backward row depends
// on it transitively, as does every forward row of its chain. Lets one chain's narrow top-level
// phase overlap another chain's wide phase instead of every chain draining at a kernel boundary.
int dag_fused_launch(cudaStream_t st, const SpGeom& s, const DagSched& sf, const DagSched& sb, const Chain* d_fwd,
                     const Chain* d_bwd, int nchains, int ncols, int64_t ld, int* flags, int* cflags, int epoch,
                     int* counter, int num_sms, const int* tmap) {
  if (nchains > DAG2_CHAINS) return -1;
  DagArgs a;
  a.chains = d_fwd;
  a.nchains = nchains;
  a.ngroups = (ncols + DCG - 1) / DCG;
  a.ncols = ncols;
  a.epoch = epoch;
  a.fwd = 1;
  a.ld = ld;
  a.ldp = static_cast<int64_t>(sf.nslots) * TILE;
  a.recs = sf.recs;
  a.ntask = sf.ntask;
  a.nslots = sf.nslots;
  a.s = s;
  a.flags = flags;
  a.cflags = cflags;
  a.counter = counter;
  a.trace = nullptr;
  a.hints = 3;
  a.tmap = tmap;
  a.presw = 1;
  a.l2pf = 0;
  a.fused = 1;
  a.recs_b = sb.recs;
  a.chains_b = d_bwd;
  a.ntask_b = sb.ntask;
  a.nslots_b = sb.nslots;
  a.ldp_b = static_cast<int64_t>(sb.nslots) * TILE;
  a.cfs = std::max(sf.nslots, sb.nslots);
  static bool attr2 = false;
  if (!attr2) {
    cudaFuncSetAttribute(dag2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, DAG2_SMEM);
    attr2 = true;
  }
  cudaMemsetAsync(counter, 0, sizeof(int), st);
  const int ntasks = (sf.ntask + sb.ntask) * nchains * a.ngroups;
  const int grid = std::min(ntasks, num_sms * ZOLO_V2_MINB);
  if (grid > 0) dag2_kernel<<<grid, P2T, DAG2_SMEM, st>>>(a);
  return grid;
}

int dag_trsm_launch(cudaStream_t st, const SpGeom& s, const DagSched& sched, const Chain* d_chains, int nchains,
                    int ncols, int64_t ld, int* flags, int* cflags, int epoch, int* counter, int fwd, int num_sms,
                    unsigned long long* trace, const int* tmap, bool presw, bool need_v2,
                    const DagQueueWork* qw, const int* gact, const int* gdone) {
  const int smem = DAG_SMEM_FIXED + (2 * DAG_REC + DAG_REC_DEPS + 8) * static_cast<int>(sizeof(int));
  static int attr_set = 0;
  if (smem > attr_set) {
    cudaFuncSetAttribute(dag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr_set = smem;
  }
  DagArgs a;
  a.chains = d_chains;
  a.nchains = nchains;
  a.ngroups = (ncols + DCG - 1) / DCG;
  a.ncols = ncols;
  a.epoch = epoch;
  a.fwd = fwd;
  a.ld = ld;
  a.ldp = static_cast<int64_t>(sched.nslots) * TILE;
  a.recs = sched.recs;
  a.ntask = sched.ntask;
  a.nslots = sched.nslots;
  a.cfs = sched.nslots;
  a.s = s;
  a.flags = flags;
  a.cflags = cflags;
  a.counter = counter;
  a.trace = trace;
  static const int hints = [] {
    const char* v = std::getenv("ZOLO_DAG_HINTS");
    return v ? std::atoi(v) : 3;
  }();
  a.hints = hints;
  a.tmap = tmap;
  a.presw = presw ? 1 : 0;
  static const int l2pf = [] {
    const char* v = std::getenv("ZOLO_DAG_L2PF");  // off: measured slower (the producer is on the path)
    return v ? std::atoi(v) : 0;
  }();
  a.l2pf = l2pf;
  cudaMemsetAsync(counter, 0, sizeof(int), st);
  const int ntasks = sched.ntask * nchains * a.ngroups;
  if (qw && sched.q_cnt0 && !tmap) {  // ready-queue scheduling
    a.queue = 1;
    a.q_cnt0 = sched.q_cnt0;
    a.q_dptr = sched.q_dptr;
    a.q_didx = sched.q_didx;
    a.q_init = sched.q_init;
    a.q_ninit = sched.q_ninit;
    a.q_cnt = qw->cnt;
    a.q_arr = qw->q;
    a.q_ctr = qw->ctr;
    cudaMemsetAsync(qw->cnt, 0, sizeof(int) * ntasks, st);
    cudaMemsetAsync(qw->q, 0, sizeof(int) * ntasks, st);
    cudaMemsetAsync(qw->ctr, 0, sizeof(int) * 2, st);
  }
  if (!a.queue && gdone) {  // lagged GMRES control: converged column groups skip their tasks
    a.gact = gact;
    a.gdone = gdone;
  }
  static const int v2 = [] {
    const char* v = std::getenv("ZOLO_DAG_V2");
    return v ? std::atoi(v) : 1;
  }();
  if (v2 && presw && nchains <= DAG2_CHAINS) {
    static bool attr2 = false;
    if (!attr2) {
      cudaFuncSetAttribute(dag2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, DAG2_SMEM);
      attr2 = true;
    }
    const int grid = std::min(ntasks, num_sms * ZOLO_V2_MINB);
    if (grid > 0) dag2_kernel<<<grid, P2T, DAG2_SMEM, st>>>(a);
    return grid;
  }
  if (need_v2) return -1;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dag_kernel, ST, smem);
  if (per_sm < 1) per_sm = 1;
  const int grid = std::min(ntasks, num_sms * per_sm);
  if (grid > 0) dag_kernel<<<grid, ST, smem, st>>>(a);
  return grid;
}

int trsm_launch(cudaStream_t st, const BandGeom& g, const Chain* d_chains, int nchains, int ncols, int64_t ld,
                unsigned long long* prog, int* flags_c, int epoch, int* counter, int fwd, int num_sms,
                unsigned long long* trace) {
  const int smem = SMEM_FIXED + (g.J + 8) * static_cast<int>(sizeof(int));
  static int attr_set = 0;
  if (smem > attr_set) {
    cudaFuncSetAttribute(trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr_set = smem;
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
  a.dl = g.dl;
  a.prog = prog;
  a.flags_c = flags_c;
  a.counter = counter;
  a.trace = trace;
  cudaMemsetAsync(counter, 0, sizeof(int), st);
  const int owners = nchains * a.ngroups;
  const int ntasks = owners + g.nbk * owners;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, trsm_kernel, ST, smem);
  if (per_sm < 1) per_sm = 1;
  const int resident = num_sms * per_sm;
  if (owners >= resident) return -1;  // owners must leave room for helpers
  const int grid = std::min(ntasks, resident);
  if (grid > 0) trsm_kernel<<<grid, ST, smem, st>>>(a);
  return grid;
}

}  // namespace zolo

// DAG-scheduled multi-RHS triangular sweeps over the block-sparse factors on
// the FP64 tensor cores.
//
// Reference: ShiftedFactor::solve / adjoint_solve (band_factor.hpp:53-117)
// sweep the factor once per right-hand-side column -- forward L (:62-69) and
// backward U (:71-80) for the solve, U^H (:98-105) then L^H (:107-112) for the
// adjoint. Here every sweep runs over all columns of the block at once as a
// recurrence over 32-row block rows of row-scaled tiles T~ (factor.cu):
//
//     u_i = pre(b_i) - sum_{j in deps(i)} op(T~(i, j)) u_j
//
// scheduled as a DAG (host symbolic.cpp dag_schedule: block rows with many
// dependencies are split into chunk tasks that sum into partial slots). All
// poles, the solve and adjoint chains and all 32-column groups share ONE
// persistent launch per sweep direction; dependencies are per-(chain, group,
// block row) epoch flags (release / acquire). Tile products are
// mma.sync.m8n8k4.f64 (DMMA, the only FP64 tensor-core path on sm_100a:
// tcgen05.mma has no f64 kind), fed by a warp-specialised producer through a
// ring of shared-memory stages filled with cp.async.bulk (the TMA engine).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "host.hpp"
#include "mma.cuh"
#include "tiles.cuh"

namespace zolo {

namespace {

constexpr int APAD = TILE + 2; // padded tile column stride (the adjoint post-pass): fragment loads conflict free
constexpr int TILE_S = TILE * APAD;
constexpr int XS = CG * XPAD;
static_assert(CG == 16, "warp layout assumes 32 x 16 output blocks");

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

// ---------------------------------------------------------------------------
// Warp-specialised DAG sweep: persistent CTAs (2 per SM) of 8 consumer warps
// (DMMA) + 1 producer warp. The producer claims tasks two ahead, reads every
// dependency / partial-slot flag of a task in parallel (one ld.acquire per
// lane + ballot), waits only on the ones still running, and streams each
// entry -- a (tile, u_j) pair, the pre-transform, or an add-block (b_i,
// partial sums) -- into an NST2-deep ring of shared-memory stages with
// cp.async.bulk (tile: one 16 KiB copy of the pre-swizzled tile; block: one
// 512 B copy per column), completing on the stage's transaction-count
// mbarrier. Consumers wait on the stage's full barrier, run the DMMA tile
// product or add the block into the accumulators, and release the stage on
// its empty barrier. The ring runs across task boundaries, and no CTA-wide
// barrier sits on the per-tile path; only the epilogue syncs the consumer
// warps: the last one to finish a task (a per-stage shared-memory count) releases u_i.
// ---------------------------------------------------------------------------
// Sweep task shape (template W): W columns per task (one tile load serves W columns); 8 consumer
// warps, each 8 rows x W / 2 columns (W / 16 8-column DMMA blocks, 16 apart); a ring of NST
// stages (tile + x block), MINB CTAs per SM. W = 64 for wide blocks (half the tile traffic and
// task overhead per column), 32 when the block has fewer than 128 columns (zolo_ctx::swc).
template <int W>
struct Shape {
  static constexpr int NB = W / 16;               // DMMA column blocks per warp
  static constexpr int NST = W == 64 ? 4 : 3;     // ring stages
  static constexpr int MINB = W == 64 ? 1 : 2;    // CTAs per SM
  static constexpr int XS = W * TILE;             // x block: W columns x 32 rows, 128-byte swizzled (mma.cuh xsw)
};
constexpr int DAG_TRACE_WORDS = 6;  // claim, -, consumer done, info, wait ns, producer done (tools/dag2_trace_analyze.py)
constexpr int TSW = TT;             // swizzled (unpadded) tile
constexpr int CW = ST / 32;         // consumer warps
constexpr int P2T = ST + 32;        // threads: the consumer warps + the producer warp
constexpr int DAG2_CHAINS = 32;

struct DagArgs {
  const Chain* chains;
  const int* recs;  // ntask x DAG_REC task records (tiles.cuh)
  int ntask, nslots;
  int nchains, ngroups, ncols, epoch;
  int64_t ld, ldp;
  SpGeom s;
  int* flags;    // per (chain, 32-column group, block): epoch when u_i is final
  int* cflags;   // per (chain, 32-column group, slot): epoch when the partial sum is written
  int* counter;  // [0] task counter, [2] wait-timeout error word
  unsigned long long* trace;  // optional: per task (claim, -, done, smid<<48|chunk<<47|i<<16|tiles, wait ns, produced)
  // lagged GMRES control (capi apply_filter_impl): the launch covers a superset of the columns
  // still running; a task whose column group has converged entirely is skipped
  const int* gact = nullptr;
  const int* gdone = nullptr;
  int policy = 1 | (2 << 2);  // L2 eviction priority: bits 0-1 tiles, bits 2-3 solution blocks (0 first, 1 normal, 2 last)
};

__device__ __forceinline__ unsigned long long l2_policy(int code) {
  return code == 0 ? l2_evict_first() : (code == 1 ? l2_evict_normal() : l2_evict_last());
}

// (development) timing probe: the tensor copies fetch 1 / ZOLO_PROBE_XDIV of every x block's rows
// (results wrong by construction): how much of a sweep is the L2 -> SM traffic of the x blocks
#ifndef ZOLO_PROBE_XDIV
#define ZOLO_PROBE_XDIV 1
#endif
struct Meta2 {
  int kind;  // 0 MMA(tile, x, neg = sign), 1 ADD(x block * sign), 2 END
  int sign;
  unsigned mx, my;  // occupancy mask (op N / op H)
  int last, i, ci, gi, out, nc, t, pad;
};
// stages are 1024-byte aligned (the 128-byte swizzle pattern of the tensor copies repeats every 1 KiB)
template <int W>
constexpr int dag2_smem() {
  return 1024 + Shape<W>::NST * (TSW + Shape<W>::XS) * static_cast<int>(sizeof(cd)) +
         Shape<W>::NST * static_cast<int>(sizeof(Meta2)) + 2 * Shape<W>::NST * 8 +
         DAG2_CHAINS * static_cast<int>(sizeof(Chain)) + DAG_REC * 4 + Shape<W>::NST * 4;
}

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
// 32 rows (row groups 4 rb .. 4 rb + 3 of the map's 8-row groups) x 32 columns (c0 ..) of a
// block through its tensor map (encode_xblock_map), one TMA instruction, completing on the
// stage's mbarrier; columns beyond the map's extent are zero-filled
__device__ __forceinline__ void tma_xblock(void* dst, const unsigned char* tmap, int rb, int c0,
                                           unsigned long long* bar, unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(0), "r"(c0), "r"(4 * rb), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// lane 0 spins on *f >= epoch (bounded: a lost producer is reported through err, never a hung
// GPU), then the warp reconverges
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
    asm volatile("fence.proxy.async.global;" ::: "memory");  // the block is then read by a tensor copy
  }
  __syncwarp();
}

// One task = (schedule record, chain, 32-column group):
//   row task:   u_i = pre(b_i) - sum_q op(T~(i, j_q)) u_(j_q) - sum_p partial_p
//   chunk task: partial_out = sum_q op(T~(i, j_q)) u_(j_q)
// The pre-transform op(Dinv_i) b_i is ring entry 0 with a negated A operand,
// so the accumulator holds S = sum - pre(b) and u_i = -S.
template <int W>
__global__ void __launch_bounds__(P2T, Shape<W>::MINB) dag2_kernel(DagArgs A) {
  constexpr int NST2 = Shape<W>::NST, XSW = Shape<W>::XS, NBW = Shape<W>::NB, SWC = W;
  extern __shared__ __align__(1024) unsigned char sm2_raw[];
  unsigned char* sm2 = sm2_raw + ((1024u - (smem_u32(sm2_raw) & 1023u)) & 1023u);
  cd* ring = reinterpret_cast<cd*>(sm2);
  Meta2* meta = reinterpret_cast<Meta2*>(sm2 + NST2 * (TSW + XSW) * sizeof(cd));
  unsigned long long* full = reinterpret_cast<unsigned long long*>(meta + NST2);
  unsigned long long* empty = full + NST2;
  Chain* chs = reinterpret_cast<Chain*>(empty + NST2);
  int* recp = reinterpret_cast<int*>(chs + DAG2_CHAINS);
  unsigned* done = reinterpret_cast<unsigned*>(recp + DAG_REC);  // per stage: consumer warps done with a task
  auto tile_s = [ring](int s) { return ring + s * (TSW + XSW); };
  auto x_s = [ring](int s) { return ring + s * (TSW + XSW) + TSW; };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int q = threadIdx.x; q < A.nchains; q += blockDim.x) chs[q] = A.chains[q];
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST2; ++s) {
      mbar_init(full + s, 1);  // the producer's arrive (+ the stage's bulk-copy bytes)
      mbar_init(empty + s, CW);
      done[s] = 0;
    }
  }
  __syncthreads();
  const int per_step = A.nchains * A.ngroups;
  const int ntasks = A.ntask * per_step;
  if (warp == CW) {
    // ------------------------------ producer ------------------------------
    const unsigned long long pol_stream = l2_evict_first(), pol_tile = l2_policy(A.policy & 3),
                             pol_keep = l2_policy((A.policy >> 2) & 3);
    int g = 0;
    int cur_t = 0;  // claim index of the task being produced (trace)
    int cur_gen = 0;  // the partial-slot generation the task writes (chunk tasks)
    // one ring entry: tile (optional) + the 32 x 32 block (block row rb, columns c0..) of the
    // chain's buffer behind tensor map `xmap` (kind 2, the end marker: nothing)
    auto produce = [&](int kind, int sign, const cd* tile, uint2 mw, const unsigned char* xmap, int rb, int c0,
                       int nc, unsigned long long pol, int last, int i, int ci, int gi, int out) {
      const int s = g % NST2, round = g / NST2;
      mbar_wait(empty + s, (round & 1) ^ 1);
      if (lane == 0) {
        const unsigned bytes = (tile ? static_cast<unsigned>(TT * sizeof(cd)) : 0u) +
                               (kind != 2 ? static_cast<unsigned>(XSW * sizeof(cd)) / ZOLO_PROBE_XDIV : 0u);
        mbar_expect_tx(full + s, bytes);
        if (tile) bulk_copy(tile_s(s), tile, TT * sizeof(cd), full + s, pol_tile);
        if (kind != 2) tma_xblock(x_s(s), xmap, rb, c0, full + s, pol);
      }
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
        m.t = cur_t;
        m.pad = cur_gen;
        meta[s] = m;
        mbar_arrive(full + s);
      }
      ++g;
    };
    auto decode = [&](int tt, int& r, int& ci, int& gi) {
      r = tt / per_step;
      const int rem = tt % per_step;
      ci = rem / A.ngroups;
      gi = rem % A.ngroups;
    };
    // lagged GMRES control: the column groups whose columns have all converged (read once)
    unsigned gmask = 0;
    if (A.gdone && A.ngroups <= 32) {
      for (int gg = 0; gg < A.ngroups; ++gg) {
        const int cg0 = gg * SWC, ncg = min(SWC, A.ncols - cg0);
        bool all = true;
        for (int h = 0; h < SWC; h += 32)
          all = __all_sync(0xffffffffu, h + lane >= ncg || A.gdone[A.gact[cg0 + h + lane]] != 0) && all;
        if (all) gmask |= 1u << gg;
      }
      if (gmask == (A.ngroups == 32 ? ~0u : (1u << A.ngroups) - 1u)) {  // nothing left: leave at once
        produce(2, 0, nullptr, make_uint2(0u, 0u), nullptr, 0, 0, 0, pol_stream, 1, 0, 0, 0, -1);
        return;
      }
    }
    // Claims run two tasks ahead: when task T starts, T+1's id has arrived (its record load is
    // issued now and lands while T streams) and the atomic for T+2 goes out.
    int t = 0;
    if (lane == 0) t = atomicAdd(A.counter, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    int rec_lo = 0, rec_hi = 0;  // this lane's two words of the current task's record
    if (t < ntasks) {
      int r0, c0_, g0_;
      decode(t, r0, c0_, g0_);
      rec_lo = A.recs[static_cast<size_t>(r0) * DAG_REC + lane];
      rec_hi = A.recs[static_cast<size_t>(r0) * DAG_REC + lane + 32];
    }
    int tn_raw = 0;
    if (lane == 0) tn_raw = atomicAdd(A.counter, 1);
    for (;;) {
      if (t >= ntasks) {
        produce(2, 0, nullptr, make_uint2(0u, 0u), nullptr, 0, 0, 0, pol_stream, 1, 0, 0, 0, -1);
        break;
      }
      const int tn = __shfl_sync(0xffffffffu, tn_raw, 0);
      int nrec_lo = 0, nrec_hi = 0;
      if (tn < ntasks) {
        int rn_, cn_, gn_;
        decode(tn, rn_, cn_, gn_);
        nrec_lo = A.recs[static_cast<size_t>(rn_) * DAG_REC + lane];
        nrec_hi = A.recs[static_cast<size_t>(rn_) * DAG_REC + lane + 32];
      }
      if (lane == 0) tn_raw = atomicAdd(A.counter, 1);
      cur_t = t;
      unsigned long long* trp = A.trace ? A.trace + DAG_TRACE_WORDS * static_cast<size_t>(t) : nullptr;
      unsigned long long wsum = 0;
      if (trp && lane == 0) trp[0] = gtimer();
      int r, ci, gi;
      decode(t, r, ci, gi);
      recp[lane] = rec_lo;
      recp[lane + 32] = rec_hi;
      __syncwarp();
      const int i = recp[0], nd = recp[1], pa = recp[2], pc = recp[3], out = recp[4], wait = recp[5], gen = recp[6],
                aux = recp[7];
      const bool chunk = out >= 0;
      // partial-slot stamps (DagTask): a chunk writes step c / K_i of its chain and reads the step
      // before; the row task reads the last step of each of its K_i = pc chains
      const int cstep = chunk ? (aux & 0xffff) / (aux >> 16) : 0;
      cur_gen = 64 * gen + cstep;
      const Chain& ch = chs[ci];
      const int c0 = gi * SWC, nc = min(SWC, A.ncols - c0);
      const size_t cgi = static_cast<size_t>(ci) * A.ngroups + gi;
      const int* flags = A.flags + cgi * A.s.nb;
      const int* cflags = A.cflags + cgi * A.nslots;
      // every task of a fully converged column group skips (its dependents are in the same group)
      if (!((gmask >> gi) & 1u)) {
        // the dependencies' blocks were written by generic stores (published by st.release); the
        // tensor copies read them through the async proxy: order the acquires before them
        asm volatile("fence.proxy.async.global;" ::: "memory");
        // occupancy masks of all the task's tiles (lane q: dependency q, lane 31: the pre-transform)
        // and readiness of every dependency, each read in parallel (one round trip)
        uint2 my_mask = make_uint2(0xffffffffu, 0xffffffffu);
        if (lane < nd)
          my_mask = ch.offm[recp[DAG_REC_HDR + 2 * lane + 1]];
        else if (lane == 31 && !chunk && ch.pre)
          my_mask = ch.prem[i];
        const unsigned dep_ready =
            __ballot_sync(0xffffffffu, lane >= nd || ld_acquire(flags + recp[DAG_REC_HDR + 2 * lane]) >= A.epoch);
        auto mask_of = [&](int q) {
          return make_uint2(__shfl_sync(0xffffffffu, my_mask.x, q), __shfl_sync(0xffffffffu, my_mask.y, q));
        };
        const int nent = (chunk ? 0 : 1) + pc + nd;
        int e = 0;
        // a chunk that takes over a partial slot waits until the row task that read it is done
        if (wait >= 0 && ld_acquire(flags + wait) < A.epoch) warp_wait_flag(flags + wait, A.epoch, A.counter + 2);
        auto pstamp = [&](int q) {  // the stamp partial q of this task must carry
          return A.epoch * DAG_GENS + 64 * gen + (chunk ? cstep - 1 : (aux - 1 - q) / pc);
        };
        if (!chunk) {  // the pre-transform op(Dinv_i) b_i (negated), or b_i itself (negated add)
          ++e;
          const uint2 pm = mask_of(31);
          if (ch.pre)
            produce(0, 1, ch.pre + static_cast<size_t>(i) * TT, pm, ch.tmaps, i, c0, nc, pol_stream, e == nent, i, ci,
                    gi, out);
          else
            produce(1, -1, nullptr, pm, ch.tmaps, i, c0, nc, pol_stream, e == nent, i, ci, gi, out);
        }
        for (int p0 = 0; p0 < pc; p0 += 32) {
          const unsigned prdy =
              __ballot_sync(0xffffffffu, p0 + lane >= pc || ld_acquire(cflags + pa + p0 + lane) >= pstamp(p0 + lane));
          for (int p = p0; p < pc && p < p0 + 32; ++p) {
            if (!((prdy >> (p - p0)) & 1u)) {
              const unsigned long long tw = trp ? gtimer() : 0;
              warp_wait_flag(cflags + pa + p, pstamp(p), A.counter + 2);
              if (trp) wsum += gtimer() - tw;
            }
            ++e;
            produce(1, 1, nullptr, make_uint2(0xffffffffu, 0xffffffffu), ch.tmaps + 2 * XMAP_BYTES, pa + p, c0, nc,
                    pol_stream, e == nent, i, ci, gi, out);
          }
        }
        for (int q = 0; q < nd; ++q) {
          const int j = recp[DAG_REC_HDR + 2 * q], tid = recp[DAG_REC_HDR + 2 * q + 1];
          if (!((dep_ready >> q) & 1u)) {
            const unsigned long long tw = trp ? gtimer() : 0;
            warp_wait_flag(flags + j, A.epoch, A.counter + 2);
            if (trp) wsum += gtimer() - tw;
          }
          ++e;
          produce(0, 0, ch.off + static_cast<size_t>(tid) * TT, mask_of(q), ch.tmaps + XMAP_BYTES, j, c0, nc, pol_keep,
                  e == nent, i, ci, gi, out);
        }
      }
      __syncwarp();
      if (trp && lane == 0) {
        trp[4] = wsum;
        trp[5] = gtimer();
      }
      t = tn;
      rec_lo = nrec_lo;
      rec_hi = nrec_hi;
    }
    return;
  }
  // ------------------------------ consumers ------------------------------
  // warp w: rows as frag(), columns 8 ((w / 4) % 2) + 16 h, h < NBW, of the task's SWC
  const Frag f = frag();
  const TileOff toff = tile_off<SWC>(f);
  Acc3<NBW> acc;  // 3M complex products (mma.cuh)
  acc3_zero(acc);
  int ntiles_task = 0;  // (trace) tile products of the current task
  for (int g = 0;; ++g) {
    const int s = g % NST2, round = g / NST2;
    mbar_wait(full + s, round & 1);
    const Meta2 m = meta[s];
    if (m.kind == 2) break;
    const Chain& ch = chs[m.ci];
    const bool opH = ch.mode == FWD_UH || ch.mode == BWD_LH;
    ntiles_task += m.kind == 0;
    if (m.kind == 0) {
      mma_tile3<SWC, NBW>(acc, tile_s(s), x_s(s), opH, m.sign != 0, toff, ((opH ? m.my : m.mx) >> f.r0) & 0xffu);
    } else {
      const cd* xs = x_s(s);
      const double sg = static_cast<double>(m.sign);
#pragma unroll
      for (int h = 0; h < NBW; ++h)
#pragma unroll
        for (int e2 = 0; e2 < 2; ++e2) {
          const cd v = xs[xsw<SWC>(ocol_sw(f, 2 * h + e2), f.row)];
          acc3_add(acc, h, e2, v, sg);
        }
    }
    if (m.last) {
      cd o[2 * NBW];
      acc3_fold(acc, o);
      acc3_zero(acc);
      const bool chunk = m.out >= 0;
      const int c0 = m.gi * SWC;
      if (chunk) {
        cd* prow = ch.cbuf + static_cast<int64_t>(m.out) * TILE + f.row + c0 * A.ldp;
#pragma unroll
        for (int q = 0; q < 2 * NBW; ++q) {
          const int c = ocol_sw(f, q);
          if (c < m.nc) prow[c * A.ldp] = o[q];
        }
      } else {
        cd* urow = ch.dst + static_cast<int64_t>(m.i) * TILE + f.row + c0 * A.ld;
#pragma unroll
        for (int q = 0; q < 2 * NBW; ++q) {
          const int c = ocol_sw(f, q);
          if (c < m.nc) urow[c * A.ld] = mk(-o[q].x, -o[q].y);
        }
      }
      // the last consumer warp to finish the task publishes it: each warp's stores are ordered
      // before its acq_rel count (syncwarp + cta-scope release), the last warp's gpu-scope release
      // is cumulative over them. The stage is released only after the count, so the counter of
      // stage s is reset before the stage can carry another task's last entry.
      __syncwarp();
      unsigned prev = 0;
      if (lane == 0)
        asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(prev) : "r"(smem_u32(done + s)) : "memory");
      if (lane == 0 && prev == CW - 1) {
        done[s] = 0;
        const size_t cgi = static_cast<size_t>(m.ci) * A.ngroups + m.gi;
        if (chunk)
          st_release(A.cflags + cgi * A.nslots + m.out, A.epoch * DAG_GENS + m.pad);
        else
          st_release(A.flags + cgi * A.s.nb + m.i, A.epoch);
        if (A.trace) {
          unsigned long long* trc = A.trace + DAG_TRACE_WORDS * static_cast<size_t>(m.t);
          unsigned smid;
          asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
          trc[2] = gtimer();
          trc[3] = (static_cast<unsigned long long>(smid) << 48) | (static_cast<unsigned long long>(chunk) << 47) |
                   (static_cast<unsigned long long>(m.i) << 16) | static_cast<unsigned>(ntiles_task);
        }
      }
      ntiles_task = 0;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + s);
  }
}

// x_i <- op(D_i) x_i, the adjoint post-pass: one CTA per (block row, chain) keeps the diagonal
// tile in shared memory and walks the block's 16-column groups with a two-stage cp.async ring
// (one launch for all adjoint chains; per-group CTAs re-read the tile for every group: 307 us per
// chain at config 3).
struct BdArgs {
  const cd* D[DAG2_CHAINS];
  cd* x[DAG2_CHAINS];
};
__global__ void __launch_bounds__(ST) blockdiag_kernel(BdArgs A, bool opH, int ncols, int64_t ld) {
  __shared__ __align__(16) cd ds[TILE_S];
  __shared__ __align__(16) cd xs[2][XS];
  const int i = blockIdx.x;
  cd* x = A.x[blockIdx.y];
  const Frag f = frag();
  {  // undo the sweep layout (tiles are stored swizzled) into the padded column-major copy
    const cd* g = A.D[blockIdx.y] + static_cast<size_t>(i) * TT;
#pragma unroll
    for (int q = 0; q < TT / ST; ++q) {
      const int e = threadIdx.x + q * ST, col = e / TILE, row = e % TILE;
      cp_async16_cg(&ds[col * APAD + row], g + col * TILE + (row ^ swz(col)));
    }
  }
  const int ngroups = (ncols + CG - 1) / CG;
  load_x(xs[0], x + static_cast<int64_t>(i) * TILE, ld, 0, min(CG, ncols));
  cp_async_commit();
  for (int g = 0; g < ngroups; ++g) {
    const int c0 = g * CG, nc = min(CG, ncols - c0);
    if (g + 1 < ngroups) {
      load_x(xs[(g + 1) & 1], x + static_cast<int64_t>(i) * TILE, ld, c0 + CG, min(CG, ncols - c0 - CG));
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    cd out[2] = {mk(0.0, 0.0), mk(0.0, 0.0)};
    mma_tile(out, ds, xs[g & 1], opH, f);
    cd* row = x + static_cast<int64_t>(i) * TILE + f.row + c0 * ld;
#pragma unroll
    for (int q = 0; q < 2; ++q)
      if (f.col + q < nc) row[(f.col + q) * ld] = out[q];
    __syncthreads();  // the stage is refilled two groups later
  }
}

}  // namespace

bool encode_xblock_map(void* map, const cd* base, int64_t ld, int64_t ncols, int swc) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static const Encode encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<Encode>(nullptr);
    return reinterpret_cast<Encode>(fn);
  }();
  static_assert(sizeof(CUtensorMap) == XMAP_BYTES, "tensor map size");
  if (!encode || !base || ld % TILE != 0 || ncols < 1 || (swc != 32 && swc != 64)) return false;
  // doubles, 3D: (16 doubles = 8 complex rows: one 128-byte swizzle line, ncols, ld / 8 row groups);
  // the box lands as [row group][column][8 rows] (mma.cuh xsw)
  const cuuint64_t dims[3] = {16, static_cast<cuuint64_t>(ncols), static_cast<cuuint64_t>(ld / 8)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld) * sizeof(cd), 128};
  const cuuint32_t box[3] = {16, static_cast<cuuint32_t>(swc), TILE / 8 / ZOLO_PROBE_XDIV};
  const cuuint32_t estr[3] = {1, 1, 1};
  return encode(static_cast<CUtensorMap*>(map), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<cd*>(base), dims,
                strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void blockdiag_apply(cudaStream_t st, int nb, const cd* const* D, cd* const* x, int nchains, bool opH, int ncols,
                     int64_t ld) {
  for (int c0 = 0; c0 < nchains && ncols > 0; c0 += DAG2_CHAINS) {
    BdArgs a;
    const int nc = std::min(DAG2_CHAINS, nchains - c0);
    for (int q = 0; q < nc; ++q) a.D[q] = D[c0 + q], a.x[q] = x[c0 + q];
    blockdiag_kernel<<<dim3(nb, nc), ST, 0, st>>>(a, opH, ncols, ld);
  }
}

int dag_groups(int ncols, int swc) { return (ncols + swc - 1) / swc; }

int dag_trsm_launch(cudaStream_t st, const SpGeom& s, const DagSched& sched, const Chain* d_chains, int nchains,
                    int ncols, int swc, int64_t ld, int64_t ldp, int* flags, int* cflags, int epoch, int* counter,
                    int num_sms, unsigned long long* trace, const int* gact, const int* gdone) {
  if (nchains > DAG2_CHAINS) return -1;
  DagArgs a;
  a.chains = d_chains;
  a.nchains = nchains;
  a.ngroups = dag_groups(ncols, swc);
  a.ncols = ncols;
  a.epoch = epoch;
  a.ld = ld;
  a.ldp = ldp;  // the chains' cbuf (and their tensor maps) are sized for the larger of the two schedules
  a.recs = sched.recs;
  a.ntask = sched.ntask;
  a.nslots = sched.nslots;
  a.s = s;
  a.flags = flags;
  a.cflags = cflags;
  a.counter = counter;
  a.trace = trace;
  a.gact = gact;
  a.gdone = gdone;
  static const int policy = [] {
    const char* v = std::getenv("ZOLO_L2_POLICY");  // (development) see DagArgs::policy
    return v && *v ? std::atoi(v) : (1 | (2 << 2));  // tiles evict_normal (+3% on cfg3), blocks evict_last
  }();
  a.policy = policy;
  // the attribute is per device: set it on every launch (a process may drive several GPUs)
  if (swc != 32 && swc != 64) return -1;
  cudaFuncSetAttribute(dag2_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, dag2_smem<32>());
  cudaFuncSetAttribute(dag2_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, dag2_smem<64>());
  cudaMemsetAsync(counter, 0, sizeof(int), st);
  const int ntasks = sched.ntask * nchains * a.ngroups;
  const int grid = std::min(ntasks, num_sms * (swc == 64 ? Shape<64>::MINB : Shape<32>::MINB));
  if (grid > 0) {
    if (swc == 64)
      dag2_kernel<64><<<grid, P2T, dag2_smem<64>(), st>>>(a);
    else
      dag2_kernel<32><<<grid, P2T, dag2_smem<32>(), st>>>(a);
  }
  return grid;
}

}  // namespace zolo

// C ABI implementation (include/zolo_b200.h): context, device memory, and the
// host-side orchestration of FilterOperator<S>::apply_g / apply_filter
// (filter_engine.hpp:56-155) on the B200.
//
// One context = one device + one private stream. The multi-shift GMRES of
// the reference runs one column at a time (gmres.hpp:98-182, one call per
// column from filter_engine.hpp:109-111); here all columns of the block run
// in lock step: each iteration applies G once to the compacted set of still
// active columns (so g_applications == sum_col m_col, exactly as the
// reference counts), then CGS2 + the batched shifted least squares decide
// which columns finish. Everything stays in the factor ordering P v on the
// device; only the input block is permuted in and the output permuted out.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <map>
#include <mutex>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/zolo_b200.h"
#include "host.hpp"
#include "krylov.cuh"
#include "tiles.cuh"
#include "shard.hpp"

namespace zolo {
void gmres_init(cudaStream_t st, GmresDev g);
// the caching device allocator below, for the other translation units (driver.cu)
void* device_alloc(size_t bytes, size_t* got, cudaStream_t st);
void device_free(void* p, size_t bytes, cudaStream_t st);
}

using namespace zolo;

namespace {

struct ZoloError : std::runtime_error {
  int code;
  ZoloError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CK(call)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      throw ZoloError(ZOLO_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));         \
  } while (0)

// Process-wide caching device allocator: freed blocks stay mapped and are handed to later
// requests of up to 2x smaller size on the same device, so repeated contexts (every eigensolver
// call builds one: factors, workspaces, Krylov basis) skip cudaMalloc / cudaFree, driver round
// trips that cost milliseconds each on a busy host. A block is released with an event recorded
// on the stream that last used it; its next user's stream waits on that event (no device-wide
// synchronisation). At most ZOLO_POOL_CAP_GB (default 16) stay cached per device: larger frees go
// back to the driver, and zolo_pool_trim / zolo_ctx_destroy of the last context return the rest.
struct Cached {
  void* p;
  cudaEvent_t done;
};
struct DevPool {
  std::mutex mu;
  std::map<int, std::multimap<size_t, Cached>> cache;
  std::map<int, size_t> cached;
  std::map<int, int> live_ctx;  // contexts per device
};
DevPool& dev_pool() {
  static DevPool* pool = new DevPool;  // never destroyed: blocks live until process exit
  return *pool;
}
size_t pool_cap() {
  static const size_t cap = [] {
    const char* v = std::getenv("ZOLO_POOL_CAP_GB");
    return static_cast<size_t>((v && *v ? std::atof(v) : 16.0) * double(size_t(1) << 30));
  }();
  return cap;
}
size_t pool_cached_bytes() {
  int dev = 0;
  cudaGetDevice(&dev);
  DevPool& P = dev_pool();
  std::lock_guard<std::mutex> lock(P.mu);
  return P.cached[dev];
}
void pool_trim(int dev) {
  DevPool& P = dev_pool();
  std::lock_guard<std::mutex> lock(P.mu);
  for (auto& kv : P.cache[dev]) {
    cudaEventSynchronize(kv.second.done);
    cudaEventDestroy(kv.second.done);
    cudaFree(kv.second.p);
  }
  P.cache[dev].clear();
  P.cached[dev] = 0;
}
// returns the block and its size (>= b), or nullptr; `st` (may be null = legacy stream) is where
// the block will be used next: it waits for the block's previous user
void* pool_alloc(size_t b, size_t* got, cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  DevPool& P = dev_pool();
  {
    std::lock_guard<std::mutex> lock(P.mu);
    auto& m = P.cache[dev];
    auto it = m.lower_bound(b);
    if (it != m.end() && it->first <= 2 * b + (size_t(1) << 20)) {
      Cached c = it->second;
      *got = it->first;
      P.cached[dev] -= it->first;
      m.erase(it);
      if (st)
        cudaStreamWaitEvent(st, c.done, 0);
      else
        cudaEventSynchronize(c.done);
      cudaEventDestroy(c.done);
      return c.p;
    }
  }
  void* p = nullptr;
  if (cudaMalloc(&p, b) != cudaSuccess) {
    cudaGetLastError();
    pool_trim(dev);  // give the cached blocks back and retry once
    if (cudaMalloc(&p, b) != cudaSuccess) return nullptr;
  }
  *got = b;
  return p;
}
// `st`: the last stream that used the block (null: synchronise the device, the conservative default)
void pool_free(void* p, size_t b, cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  DevPool& P = dev_pool();
  cudaEvent_t ev = nullptr;
  bool keep = false;
  {
    std::lock_guard<std::mutex> lock(P.mu);
    keep = P.cached[dev] + b <= pool_cap();
    if (keep) P.cached[dev] += b;  // reserve the room
  }
  if (keep && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess &&
      cudaEventRecord(ev, st) == cudaSuccess) {
    if (!st) cudaEventSynchronize(ev);  // legacy stream: unknown users, wait for the device
    std::lock_guard<std::mutex> lock(P.mu);
    P.cache[dev].emplace(b, Cached{p, ev});
    return;
  }
  if (ev) cudaEventDestroy(ev);
  if (keep) {
    std::lock_guard<std::mutex> lock(P.mu);
    P.cached[dev] -= b;
  }
  cudaFree(p);  // synchronises the device
}

// the stream of the context whose entry point is running on this thread (guarded): the stream
// new device blocks are bound to
thread_local cudaStream_t tls_stream = nullptr;

struct DevMem {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t st = nullptr;  // the stream this block is used on (its context's)
  DevMem() = default;
  DevMem(const DevMem&) = delete;
  DevMem& operator=(const DevMem&) = delete;
  ~DevMem() { release(); }
  void release() {
    if (p) pool_free(p, bytes, st);
    p = nullptr;
    bytes = 0;
  }
  // grow-only; returns true when (re)allocated. Blocks of a context live on its stream
  // (bind): every kernel that touches them runs there.
  bool ensure(size_t b) {
    if (b <= bytes && p) return false;
    release();
    if (b == 0) b = 16;
    st = tls_stream;
    size_t got = 0;
    p = pool_alloc(b, &got, st);
    if (!p) {
      cudaError_t e = cudaGetLastError();
      throw ZoloError(ZOLO_ERR_CUDA, "cudaMalloc(" + std::to_string(b) + " B): " + cudaGetErrorString(e));
    }
    b = got;
    static const bool zero = std::getenv("ZOLO_ZERO_ALLOC") != nullptr;  // (debug) zero-fill allocations
    if (zero) {
      cudaMemset(p, 0, b);
      cudaDeviceSynchronize();
    }
    bytes = b;
    return true;
  }
  template <class T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

// NVTX range around a phase of the path (factorization, filter application, G application,
// Arnoldi, Rayleigh-Ritz): visible in Nsight Systems / ncu --nvtx, free without a tool attached
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};

// development knobs (schedule tuning); defaults are the shipped configuration
int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

// Host -> device copy of setup data. Large pageable arrays (the factor plan: ~0.8 GB at config 5)
// go through two pinned bounce buffers: the CPU fills one while the DMA drains the other
// (pageable copies run at ~2 GB/s, pinned ones at ~25 GB/s).
void h2d_setup(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  constexpr size_t CH = size_t(32) << 20;
  if (bytes < 2 * CH) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    return;
  }
  struct Bounce {
    char* pin[2] = {nullptr, nullptr};
    cudaEvent_t done[2];
  };
  static std::map<int, Bounce> per_device;  // events belong to a device
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  CK(cudaGetDevice(&dev));
  Bounce& bb = per_device[dev];
  char** pin = bb.pin;
  cudaEvent_t* done = bb.done;
  if (!pin[0]) {
    for (int q = 0; q < 2; ++q) {
      CK(cudaMallocHost(&pin[q], CH));
      CK(cudaEventCreateWithFlags(&done[q], cudaEventDisableTiming));
      CK(cudaEventRecord(done[q], st));
    }
  }
  for (size_t off = 0, q = 0; off < bytes; off += CH, q ^= 1) {
    const size_t len = std::min(CH, bytes - off);
    CK(cudaEventSynchronize(done[q]));  // the DMA out of this buffer has finished
    {  // the staging copy on four host threads (one thread fills a pinned buffer at ~8 GB/s)
      constexpr int NT = 4;
      const char* from = static_cast<const char*>(src) + off;
      char* to = pin[q];
      std::thread part[NT - 1];
      for (int t = 1; t < NT; ++t)
        part[t - 1] = std::thread([=] { std::memcpy(to + len * t / NT, from + len * t / NT, len * (t + 1) / NT - len * t / NT); });
      std::memcpy(to, from, len / NT);
      for (auto& th : part) th.join();
    }
    CK(cudaMemcpyAsync(static_cast<char*>(dst) + off, pin[q], len, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(done[q], st));
  }
}

template <class T, class A>
void upload(DevMem& m, const std::vector<T, A>& v, cudaStream_t st) {
  m.ensure(sizeof(T) * std::max<size_t>(v.size(), 1));
  if (!v.empty()) h2d_setup(m.p, v.data(), sizeof(T) * v.size(), st);
  CK(cudaStreamSynchronize(st));
}

}  // namespace

namespace zolo {
cudaStream_t ctx_stream(const zolo_ctx* c);
void* device_alloc(size_t bytes, size_t* got, cudaStream_t st) { return pool_alloc(bytes, got, st); }
void device_free(void* p, size_t bytes, cudaStream_t st) { pool_free(p, bytes, st); }
}  // namespace zolo

struct zolo_ctx {
  int device = 0;
  cudaStream_t st = nullptr;
  int num_sms = 148;
  std::string err;

  // pencil (host copy, original ordering)
  int64_t n = 0;
  int cx = 0;
  bool b_identity = true;
  std::vector<int64_t> a_rp, a_ci, b_rp, b_ci;
  std::vector<double> a_v, b_v;
  bool have_pencil = false;

  // design
  int r = 0;
  std::vector<double> design;
  std::vector<std::complex<double>> eff_w, shifts;
  std::vector<double> coef;
  double constant_term = 0.0;
  bool have_design = false;

  // ordering + device pencil in the factor ordering
  std::vector<int64_t> perm;
  bool have_perm = false;
  DevGeom geom;
  DevMem perm_d, arp_d, aci_d, av_d, brp_d, bci_d, bv_d, bvc_d;
  // BSR copies of A and B in the device ordering (zolo_set_block_size): atoms of `bsr` rows
  int64_t bsr = 1, bsr_na = 0;
  bool bsr_dev = false;  // the device ordering keeps every atom's rows contiguous: SpMMs use BSR
  DevMem abrp_d, abci_d, abv_d, bbrp_d, bbci_d, bbv_d, brow0_d;

  // factors
  bool factored = false;
  DevMem tiles_mem, rownorm_mem, fstate_mem;
  std::vector<FactorTiles> tiles;
  std::vector<cudaStream_t> pole_streams;
  DevMem weights_d, shifts_d, coef_d;

  // solve workspace
  int64_t ncap = 0;  // columns the workspace is sized for
  DevMem vin_orig, vin, vout, w, bbuf, chains_fwd, chains_bwd, flags, counter;
  std::vector<std::unique_ptr<DevMem>> xbuf, cbuf;
  // residual-correction refinement of the shifted solves (zolo_set_refinement): per chain the
  // residual / correction block, the in-place sweep chains over it and the chain's shift
  int refine = 0;
  // relaxed refinement inside apply_filter (inexact Krylov): the measured relative residual of the
  // unrefined solves (worst chain), and whether the G application being enqueued may skip the
  // correction because the GMRES residuals are already small enough
  double unrefined_res = -1.0;
  bool refine_skip = false;
  bool refine_relax = true;  // zolo_set_refinement_relaxation
  int refine_skipped = 0;  // G applications of the last apply_filter that ran unrefined under that rule
  DevMem norm_buf;
  std::vector<std::unique_ptr<DevMem>> rbuf;
  DevMem chains_fwd_ref, chains_bwd_ref, chain_sigma;
  DevMem tmaps_fwd, tmaps_bwd, tmaps_fwd_ref, tmaps_bwd_ref;  // the chains' x-block tensor maps
  DevMem trace_buf;
  DevMem host_in, host_out;  // staging of the host-buffer entry points
  bool trace_done = false;

  // block-sparse factors (nested dissection, or the reference's RCM order)
  int order_mode = ZOLO_ORDER_ND;
  int64_t nd_leaf = 192;
  SpGeom sgeom;
  int64_t critical_path = 0;
  int64_t work_nnz = 0, work_exec = 0;  // pole 0's sweep tiles: nonzero entries / entries in unmasked 8x4 blocks
  int iters_seen = 0;         // largest Krylov dimension an apply_filter on this context has needed
  const int* lag_done = nullptr;  // lagged GMRES control: per-column done flags the sweeps may skip on
  int* act_hq[4] = {};   // pinned active lists / done flags, one per lagged-loop slot
  int* done_hq[4] = {};
  DevMem sp_row_ptr, sp_row_idx, sp_col_ptr, sp_col_idx, sp_col_tile, sp_tile_row, sp_pad_rows, sp_err;
  DevMem sp_sched_fwd, sp_sched_bwd, sp_masks;
  DevMem sp_er, sp_ec, sp_ea, sp_eb;  // scatter lists of the union pattern in the factor ordering
  int64_t sp_nnz = 0;
  int sp_npads = 0;
  bool sym_ready = false;
  FactorPlan fplan;                         // level-scheduled factorization (host level ranges)
  DevMem fp_lmask;  // per pole and L tile: occupancy mask written by the panel step (SpFactor::lmask)
  DevMem fp_cols, fp_pan, fp_tgt, fp_con, fp_cmb, fp_scratch;  // its device arrays; partial products of split targets
  DagSched sched_fwd, sched_bwd;
  int sp_nslots = 0;
  int swc = 32;  // sweep task width (columns): 64 for blocks of >= 128 columns (ensure_workspace)
  std::vector<cd*> sp_dt;
  int64_t flags_cap = 0, prog_cap = 0, cflags_off = 0;
  int epoch = 0;

  // GMRES state
  int maxit_cap = 0;
  std::vector<std::unique_ptr<DevMem>> basis;
  DevMem basis_ptrs, gH, gR, gG, gROT, gY, gZ, gres, gfrozen, gmlen, gbeta, gmcol, ghappy, gdone, gwnorm;
  DevMem partial, hsave, act_d, rr_partial, rr_tmp, rr_out, tmp1, tmp2, tmp3;
  int* act_h = nullptr;
  int* done_h = nullptr;

  int64_t inner_solves = 0, g_apps = 0;
  double last_ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  cudaEvent_t tev0 = nullptr, tev1 = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr, ev3 = nullptr;
  cudaEvent_t ev4 = nullptr, ev5 = nullptr;  // device-busy time of the GMRES iterations
  cudaEvent_t lag_ev[20] = {};                // lagged GMRES loop: done-copy, sweep and busy events x 4 slots
  cudaEvent_t ev2_use = nullptr, ev3_use = nullptr;  // apply_g_device's sweep events when set

  // hybrid inner solve (BASELINE config 2): one factored pole,
  // shift-invariant GMRES on K_p^{-1} B for the others
  int hybrid = 0, hy_pole = 0, hy_max = 256;
  double hy_tol = 1e-14;
  int64_t hy_inner_its = 0;  // inner Arnoldi steps (summed over columns) of the last apply_filter
  DevMem hy_x0[2], hy_y[2], hy_w, hy_weights, hy_shifts[2], hy_ccoef[2], act_in_d;
  DevMem iH, iR, iG, iROT, iY, iZ, ires, ifrozen, imlen, ibeta, imcol, ihappy, idone, iwnorm, ipartial, ihsave,
      ibasis_ptrs;
  std::vector<std::unique_ptr<DevMem>> ibasis;
  int imaxit_cap = 0;
  int64_t incap = 0;
  int* act_in_h = nullptr;

  // pole sharding: this context factors the poles own[] of the design
  int shard_rank = 0, shard_size = 1;
  std::vector<int> own;
  Collective* coll = nullptr;  // the group's collectives (NCCL, or host-staged through a callback)
  // Row-sharded Arnoldi (default with a communicator; ZOLO_ROW_SHARD=0: replicated, G all-reduced):
  // rank g owns rows [g rb, min(ld, (g + 1) rb)) of every Krylov vector. A G application ends with
  // a reduce-scatter of the ranks' partial sums over row blocks, the CGS2 inner products are
  // all-reduced (n_active x (m + 1) scalars), and the next basis vector is all-gathered (every
  // rank's poles need all of its rows): per iteration the bytes of one all-reduce, and the Arnoldi
  // work divided by the ranks.
  bool row_shard = false;
  bool in_filter = false;  // inside apply_filter (the row-sharded layout applies; zolo_apply_g stays replicated)
  int64_t rb = 0;
  DevMem wc, wloc, vpack, vgath;  // blocked partial G | this rank's reduced block | basis block out / in

  size_t es() const { return cx ? 16 : 8; }
  int nloc() const { return static_cast<int>(own.size()); }
  int nchains() const { return cx ? 2 * nloc() : nloc(); }
  double local_constant() const { return shard_rank == 0 ? constant_term : 0.0; }
};

namespace {

std::string g_create_err;

// Runs an entry point on the context's device and stream; the caller's current device is
// restored afterwards (a library call must not move the caller's CUDA state).
struct DeviceScope {
  int saved = -1;
  cudaStream_t saved_stream;
  DeviceScope(const zolo_ctx* ctx) : saved_stream(tls_stream) {
    if (ctx && cudaGetDevice(&saved) == cudaSuccess && saved != ctx->device) cudaSetDevice(ctx->device);
    if (ctx) tls_stream = ctx->st;
  }
  ~DeviceScope() {
    int cur = -1;
    if (saved >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != saved) cudaSetDevice(saved);
    tls_stream = saved_stream;
  }
};

template <class F>
int guarded(zolo_ctx* ctx, F&& f) {
  DeviceScope scope(ctx);
  try {
    f();
    return ZOLO_OK;
  } catch (const ZoloError& e) {
    if (ctx) ctx->err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    if (ctx) ctx->err = "host allocation failed";
    return ZOLO_ERR_NUMERICAL;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what();
    return ZOLO_ERR_NUMERICAL;
  }
}

void require(bool ok, const std::string& msg) {
  if (!ok) throw ZoloError(ZOLO_ERR_DOMAIN, msg);
}

// fn(lo, hi) over [0, n) in contiguous ranges on the host cores (setup loops over the pencil's
// rows: each range writes its own output rows, so the result does not depend on the threading);
// the first exception of a range is rethrown on the caller
template <class F>
void par_rows(int64_t n, F&& fn, int64_t grain = 2048) {  // grain: rows worth a thread of their own
  const int nt = static_cast<int>(std::min<int64_t>(std::min(16u, std::max(1u, std::thread::hardware_concurrency())),
                                                    std::max<int64_t>(1, n / grain)));
  if (nt < 2) {
    fn(int64_t{0}, n);
    return;
  }
  std::vector<std::exception_ptr> err(nt);
  std::vector<std::thread> pool;
  for (int q = 0; q < nt; ++q)
    pool.emplace_back([&, q] {
      try {
        fn(n * q / nt, n * (q + 1) / nt);
      } catch (...) {
        err[q] = std::current_exception();
      }
    });
  for (auto& t : pool) t.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}

// Union pattern of A and B (B = I when absent): assemble_shifted (sparse.hpp:153-186).
struct Union {
  std::vector<int64_t> rp;
  std::vector<int64_t, NoInit<int64_t>> ci;
  std::vector<double, NoInit<double>> av, bv;  // interleaved when complex
};

Union union_pattern(const zolo_ctx& c) {
  Union u;
  const int64_t n = c.n;
  const int w = c.cx ? 2 : 1;
  u.rp.assign(n + 1, 0);
  // the rows' merges are independent: count, prefix sum, fill (all host cores)
  auto merge_row = [&](int64_t i, auto&& emit) {
    int64_t ka = c.a_rp[i], kb = c.b_identity ? 0 : c.b_rp[i];
    const int64_t ea = c.a_rp[i + 1], eb = c.b_identity ? 1 : c.b_rp[i + 1];
    while (ka < ea || kb < eb) {
      const int64_t ja = ka < ea ? c.a_ci[ka] : n;
      const int64_t jb = kb < eb ? (c.b_identity ? i : c.b_ci[kb]) : n;
      const int64_t j = std::min(ja, jb);
      emit(j, ja == j ? ka : int64_t{-1}, jb == j ? kb : int64_t{-1});
      if (ja == j) ++ka;
      if (jb == j) ++kb;
    }
  };
  par_rows(n, [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) {
      int64_t cnt = 0;
      merge_row(i, [&](int64_t, int64_t, int64_t) { ++cnt; });
      u.rp[i + 1] = cnt;
    }
  });
  for (int64_t i = 0; i < n; ++i) u.rp[i + 1] += u.rp[i];
  const size_t nnz = static_cast<size_t>(u.rp[n]);
  u.ci.resize(nnz);
  u.av.resize(nnz * w);
  u.bv.resize(nnz * w);
  par_rows(n, [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) {
      int64_t at = u.rp[i];
      merge_row(i, [&](int64_t j, int64_t ka, int64_t kb) {
        u.ci[at] = j;
        for (int q = 0; q < w; ++q) {
          u.av[at * w + q] = ka >= 0 ? c.a_v[ka * w + q] : 0.0;
          u.bv[at * w + q] = kb >= 0 ? (c.b_identity ? (q == 0 ? 1.0 : 0.0) : c.b_v[kb * w + q]) : 0.0;
        }
        ++at;
      });
    }
  });
  return u;
}

// P M P^T as int32 CSR over the npad device positions (padding rows empty),
// sorted columns. inv: position -> original row or -1; pos: original -> position.
void permuted_csr(int64_t npad, const std::vector<int64_t>& inv, const std::vector<int>& pos,
                  const std::vector<int64_t>& rp, const std::vector<int64_t>& ci, const std::vector<double>& v, int w,
                  std::vector<int>& prp, std::vector<int, NoInit<int>>& pci,
                  std::vector<double, NoInit<double>>& pv) {
  prp.assign(npad + 1, 0);
  for (int64_t t = 0; t < npad; ++t) {
    const int64_t i = inv[t];
    prp[t + 1] = prp[t] + (i >= 0 ? static_cast<int>(rp[i + 1] - rp[i]) : 0);
  }
  pci.resize(static_cast<size_t>(prp[npad]));
  pv.resize(static_cast<size_t>(prp[npad]) * w);
  par_rows(npad, [&](int64_t lo, int64_t hi) {  // every device row sorts and writes its own range
    std::vector<std::pair<int, int64_t>> row;
    for (int64_t t = lo; t < hi; ++t) {
      const int64_t i = inv[t];
      if (i < 0) continue;
      row.clear();
      for (int64_t k = rp[i]; k < rp[i + 1]; ++k) row.emplace_back(pos[ci[k]], k);
      std::sort(row.begin(), row.end());
      int64_t at = prp[t];
      for (auto& e : row) {
        pci[at] = e.first;
        for (int q = 0; q < w; ++q) pv[at * w + q] = v[e.second * w + q];
        ++at;
      }
    }
  });
}

// Device copies of the pencil in the factor ordering + the position map.
// M (CSR, original ordering) as BSR over atoms of b rows, atoms in device order (rank), dense
// row-major blocks, block columns ascending by rank; row0[rank] = device row of the atom's first row.
void bsr_from_csr(int64_t na, int b, const std::vector<int64_t>& rank_of, const std::vector<int64_t>& atom_of_rank,
                  const std::vector<int64_t>& rp, const std::vector<int64_t>& ci, const std::vector<double>& v, int w,
                  std::vector<int>& brp, std::vector<int>& bci, std::vector<double>& bval) {
  brp.assign(na + 1, 0);
  bci.clear();
  bval.clear();
  std::vector<int64_t> slot(na, -1), cols;
  for (int64_t I = 0; I < na; ++I) {
    const int64_t atom = atom_of_rank[I];
    cols.clear();
    for (int r = 0; r < b; ++r)
      for (int64_t q = rp[atom * b + r]; q < rp[atom * b + r + 1]; ++q) {
        const int64_t J = rank_of[ci[q] / b];
        if (slot[J] < 0) {
          slot[J] = 0;
          cols.push_back(J);
        }
      }
    std::sort(cols.begin(), cols.end());
    const size_t base = bci.size();
    for (size_t k = 0; k < cols.size(); ++k) {
      slot[cols[k]] = static_cast<int64_t>(base + k);
      bci.push_back(static_cast<int>(cols[k]));
    }
    bval.resize(bci.size() * b * b * w, 0.0);
    for (int r = 0; r < b; ++r)
      for (int64_t q = rp[atom * b + r]; q < rp[atom * b + r + 1]; ++q) {
        const int64_t J = rank_of[ci[q] / b], kk = ci[q] % b;
        const size_t e = ((static_cast<size_t>(slot[J]) * b + r) * b + kk) * w;
        for (int z = 0; z < w; ++z) bval[e + z] = v[q * w + z];
      }
    for (int64_t J : cols) slot[J] = -1;
    brp[I + 1] = static_cast<int>(bci.size());
  }
}

void upload_device_bsr(zolo_ctx& c, const std::vector<int>& pos) {
  c.bsr_dev = false;
  const int64_t b = c.bsr, n = c.n;
  if (b <= 1 || n % b) return;
  const int64_t na = n / b;
  for (int64_t a = 0; a < na; ++a)
    for (int64_t r = 1; r < b; ++r)
      if (pos[a * b + r] != pos[a * b] + r) return;  // an atom split by the ordering: CSR SpMMs
  std::vector<int64_t> atom_of_rank(na), rank_of(na);
  for (int64_t a = 0; a < na; ++a) atom_of_rank[a] = a;
  std::sort(atom_of_rank.begin(), atom_of_rank.end(), [&](int64_t x, int64_t y) { return pos[x * b] < pos[y * b]; });
  std::vector<int> row0(na);
  for (int64_t I = 0; I < na; ++I) {
    rank_of[atom_of_rank[I]] = I;
    row0[I] = pos[atom_of_rank[I] * b];
  }
  const int w = c.cx ? 2 : 1;
  std::vector<int> brp, bci;
  std::vector<double> bval;
  bsr_from_csr(na, static_cast<int>(b), rank_of, atom_of_rank, c.a_rp, c.a_ci, c.a_v, w, brp, bci, bval);
  upload(c.abrp_d, brp, c.st);
  upload(c.abci_d, bci, c.st);
  upload(c.abv_d, bval, c.st);
  if (!c.b_identity) {
    bsr_from_csr(na, static_cast<int>(b), rank_of, atom_of_rank, c.b_rp, c.b_ci, c.b_v, w, brp, bci, bval);
    upload(c.bbrp_d, brp, c.st);
    upload(c.bbci_d, bci, c.st);
    upload(c.bbv_d, bval, c.st);
  }
  upload(c.brow0_d, row0, c.st);
  c.bsr_na = na;
  c.bsr_dev = true;
}

void upload_device_pencil(zolo_ctx& c, const std::vector<int64_t>& inv, const std::vector<int>& pos) {
  const int w = c.cx ? 2 : 1;
  const int64_t npad = static_cast<int64_t>(inv.size());
  std::vector<int> prp, brp;
  std::vector<int, NoInit<int>> pci, bci;
  std::vector<double, NoInit<double>> pv, bv;
  // B's permuted copy on a host thread beside A's (plain host work; bad_alloc is the only failure)
  std::exception_ptr berr;
  std::thread tb;
  if (!c.b_identity)
    tb = std::thread([&] {
      try {
        permuted_csr(npad, inv, pos, c.b_rp, c.b_ci, c.b_v, w, brp, bci, bv);
      } catch (...) {
        berr = std::current_exception();
      }
    });
  struct Join {
    std::thread& t;
    ~Join() {
      if (t.joinable()) t.join();
    }
  } join_b{tb};
  upload_device_bsr(c, pos);
  permuted_csr(npad, inv, pos, c.a_rp, c.a_ci, c.a_v, w, prp, pci, pv);
  upload(c.arp_d, prp, c.st);
  upload(c.aci_d, pci, c.st);
  upload(c.av_d, pv, c.st);
  if (!c.b_identity) {
    tb.join();
    if (berr) std::rethrow_exception(berr);
    prp.swap(brp);
    pci.swap(bci);
    pv.swap(bv);
    upload(c.brp_d, prp, c.st);
    upload(c.bci_d, pci, c.st);
    upload(c.bv_d, pv, c.st);
    if (!c.cx) {  // complex copy for the hybrid solve's inner Krylov space (complex even for real pencils)
      std::vector<double> pvc(2 * pv.size(), 0.0);
      for (size_t q = 0; q < pv.size(); ++q) pvc[2 * q] = pv[q];
      upload(c.bvc_d, pvc, c.st);
    }
  }
  std::vector<int> p32(inv.begin(), inv.end());
  upload(c.perm_d, p32, c.st);
  c.have_perm = true;
}

void ensure_perm_csr(zolo_ctx& c) {
  if (c.have_perm) return;
  require(c.have_pencil, "no pencil uploaded");
  c.geom.n = c.n;
  c.geom.nbk = static_cast<int>((c.n + TILE - 1) / TILE);
  c.geom.npad = static_cast<int64_t>(c.geom.nbk) * TILE;
  std::vector<int64_t> inv(c.geom.npad, -1);
  std::vector<int> pos(c.n);
  for (int64_t i = 0; i < c.n; ++i) {
    inv[i] = i;
    pos[i] = static_cast<int>(i);
  }
  upload_device_pencil(c, inv, pos);
}

// Block-sparse factors for every pole: under nested dissection (symbolic.cpp),
// under the reference's RCM ordering (ZOLO_ORDER_RCM, band_factor.hpp:203-204:
// one node, so pivot positions are RCM positions as in the reference's
// FactorizationError), or under a caller ordering given as perm.
void do_factorize_sparse(zolo_ctx& c, const int64_t* perm_in, zolo_factor_stats* stats);

void do_factorize(zolo_ctx& c, const int64_t* perm_in, zolo_factor_stats* stats) {
  Nvtx range("zolo::factorize");
  require(c.have_pencil, "zolo_factorize: no pencil uploaded");
  require(c.have_design, "zolo_factorize: no design installed");
  if (c.order_mode == ZOLO_ORDER_RCM && !perm_in) {
    Union u = union_pattern(c);
    std::vector<int64_t> rcm(c.n);
    rcm_order(c.n, u.rp.data(), u.ci.data(), rcm.data());  // band_factor.hpp:203-204
    c.sym_ready = false;
    do_factorize_sparse(c, rcm.data(), stats);
    if (stats) {  // FactorProfile.bandwidth (band_factor.hpp:31-35): the half-bandwidth under RCM
      const int64_t bw = bandwidth_under(c.n, u.rp.data(), u.ci.data(), rcm.data());
      for (int j = 0; j < c.nloc(); ++j) stats[j].bandwidth = bw;
    }
    return;
  }
  do_factorize_sparse(c, perm_in, stats);
}

// Ordering + block symbolic analysis + sweep schedules + the device pencil and
// scatter lists in the factor ordering: everything shift-independent.
// (development) ZOLO_SETUP_TIMES=1 prints the host setup phases
struct SetupClock {
  bool on = std::getenv("ZOLO_SETUP_TIMES") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[setup] %-22s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

void sparse_symbolic(zolo_ctx& c, const int64_t* perm_in) {
  SetupClock clk;
  const int64_t n = c.n;
  Union u = union_pattern(c);
  clk.mark("union pattern");
  std::vector<std::vector<int64_t>> nodes;
  if (perm_in) {
    std::vector<char> seen(n, 0);
    std::vector<int64_t> one(n);
    for (int64_t i = 0; i < n; ++i) {
      require(perm_in[i] >= 0 && perm_in[i] < n && !seen[perm_in[i]], "zolo_factorize: invalid permutation");
      seen[perm_in[i]] = 1;
      one[i] = perm_in[i];
    }
    nodes.push_back(std::move(one));
  } else if (c.bsr > 1 && n % c.bsr == 0) {
    // atoms of bsr rows (BSR pencils): dissect the block graph, then expand every atom into its
    // rows in order, so atoms stay contiguous in the device ordering (BSR SpMMs)
    const int64_t b = c.bsr, na = n / b;
    std::vector<int64_t> brp(na + 1, 0), bci;
    std::vector<std::vector<int64_t>> nbr(na);
    par_rows(na, [&](int64_t lo, int64_t hi) {  // atoms are independent: each range its own marks
      std::vector<int64_t> mark(na, -1);
      for (int64_t I = lo; I < hi; ++I) {
        for (int64_t i = I * b; i < (I + 1) * b; ++i)
          for (int64_t q = u.rp[i]; q < u.rp[i + 1]; ++q) {
            const int64_t J = u.ci[q] / b;
            if (mark[J] != I) {
              mark[J] = I;
              nbr[I].push_back(J);
            }
          }
        std::sort(nbr[I].begin(), nbr[I].end());
      }
    }, 16);
    for (int64_t I = 0; I < na; ++I) {
      bci.insert(bci.end(), nbr[I].begin(), nbr[I].end());
      brp[I + 1] = static_cast<int64_t>(bci.size());
    }
    std::vector<std::vector<int64_t>> anodes;
    nd_order(na, brp.data(), bci.data(), std::max<int64_t>(1, c.nd_leaf / b), anodes);
    for (const auto& an : anodes) {
      std::vector<int64_t> rows;
      rows.reserve(an.size() * b);
      for (int64_t a : an)
        for (int64_t r = 0; r < b; ++r) rows.push_back(a * b + r);
      nodes.push_back(std::move(rows));
    }
  } else {
    nd_order(n, u.rp.data(), u.ci.data(), c.nd_leaf, nodes);
  }
  clk.mark("nested dissection");
  BlockStructure bs;
  block_symbolic(n, u.rp.data(), u.ci.data(), nodes, TILE, bs);
  clk.mark("block symbolic");
  require(bs.ntiles < (int64_t(1) << 31) && bs.npad < (int64_t(1) << 31), "zolo_factorize: structure too large");
  const int nb = static_cast<int>(bs.nb);
  std::vector<int> pos(n);
  for (int64_t i = 0; i < n; ++i) pos[i] = static_cast<int>(bs.pos[i]);
  c.perm.assign(n, 0);
  for (int64_t t = 0, q = 0; t < bs.npad; ++t)
    if (bs.inv[t] >= 0) c.perm[q++] = bs.inv[t];
  c.critical_path = bs.critical_path;

  DevGeom g;
  g.n = n;
  g.npad = bs.npad;
  g.nbk = nb;
  c.geom = g;

  // The factor plan and the two sweep schedules depend on the block structure only: host threads
  // build them while this thread uploads the structure, the scatter lists and the device pencil.
  std::exception_ptr bg_err[3];
  std::vector<int> rec_f, rec_b;
  int ntask_f = 0, ntask_b = 0, sf = 0, sb = 0;
  // claim-ordered sweep schedules: wide block rows split into chunk tasks
  static const int near = std::min(std::max(env_int("ZOLO_DAG_NEAR", 4), 0), DAG_REC_DEPS - 1),
                   chunk = std::min(std::max(env_int("ZOLO_DAG_CHUNK", 16), 1), DAG_REC_DEPS - near),
                   order = env_int("ZOLO_DAG_ORDER", 3);
  // self-contained task records: header + the (j, tile id) pairs in processing order
  auto schedule = [&](bool fwd, std::vector<int>& rec, int& ntask, int& nslots) {
    std::vector<DagTask> ts;
    nslots = fwd ? dag_schedule(nb, bs.row_ptr, bs.row_idx, true, chunk, near, order, ts)
                 : dag_schedule(nb, bs.col_ptr, bs.col_idx, false, chunk, near, order, ts);
    ntask = static_cast<int>(ts.size());
    rec.assign(ts.size() * DAG_REC, 0);
    for (size_t t = 0; t < ts.size(); ++t) {
      const DagTask& k = ts[t];
      int* r = rec.data() + t * DAG_REC;
      const int64_t e0 = fwd ? bs.row_ptr[k.i] : bs.col_ptr[k.i];
      const int ndall = static_cast<int>((fwd ? bs.row_ptr[k.i + 1] : bs.col_ptr[k.i + 1]) - e0);
      const int nd = k.qb - k.qa;
      require(nd <= DAG_REC_DEPS, "zolo_factorize: DAG task record overflow");
      r[0] = k.i, r[1] = nd, r[2] = k.pa, r[3] = k.pc, r[4] = k.out, r[5] = k.wait, r[6] = k.gen, r[7] = k.aux;
      for (int q = 0; q < nd; ++q) {
        const int64_t e = fwd ? e0 + k.qa + q : e0 + ndall - 1 - (k.qa + q);
        r[DAG_REC_HDR + 2 * q] = static_cast<int>(fwd ? bs.row_idx[e] : bs.col_idx[e]);
        r[DAG_REC_HDR + 2 * q + 1] = static_cast<int>(fwd ? e : bs.col_tile[e]);
      }
    }
  };
  auto guard_bg = [&](int slot, auto&& fn) {
    return std::thread([&bg_err, slot, fn] {
      try {
        fn();
      } catch (...) {
        bg_err[slot] = std::current_exception();
      }
    });
  };
  std::thread bg[3] = {guard_bg(0, [&] { factor_plan(bs, c.fplan); }),
                       guard_bg(1, [&] { schedule(true, rec_f, ntask_f, sf); }),
                       guard_bg(2, [&] { schedule(false, rec_b, ntask_b, sb); })};
  struct JoinAll {
    std::thread* t;
    ~JoinAll() {
      for (int k = 0; k < 3; ++k)
        if (t[k].joinable()) t[k].join();
    }
  } join_all{bg};

  auto to32 = [](const std::vector<int64_t>& v) { return std::vector<int>(v.begin(), v.end()); };
  std::vector<int> tile_row(bs.ntiles);
  for (int64_t i = 0; i < nb; ++i)
    for (int64_t e = bs.row_ptr[i]; e < bs.row_ptr[i + 1]; ++e) tile_row[e] = static_cast<int>(i);
  upload(c.sp_row_ptr, to32(bs.row_ptr), c.st);
  upload(c.sp_row_idx, to32(bs.row_idx), c.st);
  upload(c.sp_col_ptr, to32(bs.col_ptr), c.st);
  upload(c.sp_col_idx, to32(bs.col_idx), c.st);
  upload(c.sp_col_tile, to32(bs.col_tile), c.st);
  upload(c.sp_tile_row, tile_row, c.st);
  int max_deps = 0;
  for (int i = 0; i < nb; ++i) {
    max_deps = std::max(max_deps, static_cast<int>(bs.row_ptr[i + 1] - bs.row_ptr[i]));
    max_deps = std::max(max_deps, static_cast<int>(bs.col_ptr[i + 1] - bs.col_ptr[i]));
  }
  SpGeom s;
  s.n = n;
  s.npad = bs.npad;
  s.nb = nb;
  s.ntiles = bs.ntiles;
  s.max_deps = max_deps;
  s.row_ptr = c.sp_row_ptr.as<int>();
  s.row_idx = c.sp_row_idx.as<int>();
  s.col_ptr = c.sp_col_ptr.as<int>();
  s.col_idx = c.sp_col_idx.as<int>();
  s.col_tile = c.sp_col_tile.as<int>();
  s.tile_row = c.sp_tile_row.as<int>();
  c.sgeom = s;

  const int64_t nnz = static_cast<int64_t>(u.ci.size());
  std::vector<int, NoInit<int>> er(nnz), ec(nnz);
  std::vector<int> pads;
  par_rows(n, [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i)
      for (int64_t k = u.rp[i]; k < u.rp[i + 1]; ++k) {
        er[k] = pos[i];
        ec[k] = pos[u.ci[k]];
      }
  });
  for (int64_t t = 0; t < bs.npad; ++t)
    if (bs.inv[t] < 0) pads.push_back(static_cast<int>(t));
  upload(c.sp_er, er, c.st);
  upload(c.sp_ec, ec, c.st);
  upload(c.sp_ea, u.av, c.st);
  upload(c.sp_eb, u.bv, c.st);
  upload(c.sp_pad_rows, pads, c.st);
  c.sp_nnz = nnz;
  c.sp_npads = static_cast<int>(pads.size());
  upload_device_pencil(c, bs.inv, pos);
  clk.mark("device pencil");
  for (int k = 0; k < 3; ++k) bg[k].join();
  for (int k = 0; k < 3; ++k)
    if (bg_err[k]) std::rethrow_exception(bg_err[k]);
  clk.mark("plan + schedules (wait)");
  upload(c.sp_sched_fwd, rec_f, c.st);
  upload(c.sp_sched_bwd, rec_b, c.st);
  c.sched_fwd = DagSched{c.sp_sched_fwd.as<int>(), ntask_f, sf};
  c.sched_bwd = DagSched{c.sp_sched_bwd.as<int>(), ntask_b, sb};
  c.sp_nslots = std::max(sf, sb);
  upload(c.fp_cols, c.fplan.cols, c.st);
  upload(c.fp_pan, c.fplan.pan, c.st);
  upload(c.fp_tgt, c.fplan.tgt, c.st);
  upload(c.fp_con, c.fplan.con, c.st);
  upload(c.fp_cmb, c.fplan.cmb, c.st);
  clk.mark("plan upload");
  c.sym_ready = true;
}

// Numeric block-sparse LU of A - sigma_k B for each shift into `store`
// (Dt, DinvL, DinvU: nb tiles; Lt, Ut: ntiles), one stream per shift;
// masks (tile_masks) when `mstore` is given. fail[k] / min_ratio[k] per shift.
void sparse_numeric(zolo_ctx& c, const std::vector<std::complex<double>>& sig, DevMem& store, DevMem* mstore,
                    std::vector<FactorTiles>& tiles, std::vector<cd*>& dt, std::vector<int>& fail,
                    std::vector<double>& min_ratio, size_t* per_pole_out) {
  const int nb = c.sgeom.nb;
  const int64_t ntiles = c.sgeom.ntiles;
  const int r = static_cast<int>(sig.size());
  const size_t per_diag = static_cast<size_t>(nb) * TT;
  const size_t per_off = static_cast<size_t>(ntiles) * TT;
  const size_t per_pole = 3 * per_diag + 2 * per_off;
  if (per_pole_out) *per_pole_out = per_pole;
  size_t free_b = 0, total_b = 0;
  SetupClock clk;
  store.release();
  CK(cudaMemGetInfo(&free_b, &total_b));
  free_b += pool_cached_bytes();  // cached blocks are reusable
  const size_t need = per_pole * r * sizeof(cd);
  if (need + (size_t(1) << 30) > free_b)
    throw ZoloError(ZOLO_ERR_DOMAIN, "zolo_factorize: factors need " + std::to_string(need >> 20) +
                                         " MiB, device has " + std::to_string(free_b >> 20) + " MiB free");
  store.ensure(need);
  c.rownorm_mem.ensure(sizeof(double) * c.sgeom.npad * r);
  c.fstate_mem.ensure(sizeof(unsigned long long) * 2 * r);
  c.sp_err.ensure(sizeof(int) * 4 + 2 * sizeof(unsigned long long));
  CK(cudaMemsetAsync(c.sp_err.p, 0, sizeof(int) * 4, c.st));
  tiles.assign(r, FactorTiles());
  dt.assign(r, nullptr);
  cd* base = store.as<cd>();
  for (int j = 0; j < r; ++j) {
    cd* p = base + per_pole * j;
    dt[j] = p;
    tiles[j].DinvL = p + per_diag;
    tiles[j].DinvU = p + 2 * per_diag;
    tiles[j].Lt = p + 3 * per_diag;
    tiles[j].Ut = p + 3 * per_diag + per_off;
  }
  if (mstore) {
    const size_t mper = 2 * static_cast<size_t>(nb) + 2 * static_cast<size_t>(ntiles);
    mstore->ensure(sizeof(uint2) * mper * r);
    for (int j = 0; j < r; ++j) {
      uint2* m = mstore->as<uint2>() + mper * j;
      tiles[j].mDL = m;
      tiles[j].mDU = m + nb;
      tiles[j].mLt = m + 2 * nb;
      tiles[j].mUt = m + 2 * nb + ntiles;
    }
  }
  std::vector<unsigned long long> fs(2 * r);
  const double inf = std::numeric_limits<double>::infinity();
  unsigned long long infbits;
  std::memcpy(&infbits, &inf, 8);
  for (int j = 0; j < r; ++j) {
    fs[2 * j] = 0xffffffffffffffffull;
    fs[2 * j + 1] = infbits;
  }
  CK(cudaMemcpyAsync(c.fstate_mem.p, fs.data(), fs.size() * 8, cudaMemcpyHostToDevice, c.st));
  CK(cudaStreamSynchronize(c.st));
  clk.mark("factor storage");
  while (static_cast<int>(c.pole_streams.size()) < r) {
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    c.pole_streams.push_back(st);
  }
  FactorPlanDev pd;
  pd.lvl_ptr = &c.fplan.lvl_ptr;
  pd.pan_ptr = &c.fplan.pan_ptr;
  pd.tgt_ptr = &c.fplan.tgt_ptr;
  pd.cmb_ptr = &c.fplan.cmb_ptr;
  pd.cmb = c.fp_cmb.as<int>();
  const size_t scratch_per_pole = static_cast<size_t>(std::max<int64_t>(c.fplan.scratch_slots, 1)) * TT;
  c.fp_scratch.ensure(sizeof(cd) * scratch_per_pole * r);
  const size_t lmask_per_pole = static_cast<size_t>(std::max<int64_t>(ntiles, 1));
  c.fp_lmask.ensure(sizeof(unsigned) * lmask_per_pole * r);
  CK(cudaMemsetAsync(c.fp_lmask.p, 0xff, sizeof(unsigned) * lmask_per_pole * r, c.st));
  pd.cols = c.fp_cols.as<int>();
  pd.pan = c.fp_pan.as<int>();
  pd.tgt = c.fp_tgt.as<int>();
  pd.con = c.fp_con.as<int>();
  CK(cudaStreamSynchronize(c.st));
  CK(cudaEventRecord(c.ev0, c.st));
  for (int j = 0; j < r; ++j) CK(cudaStreamWaitEvent(c.pole_streams[j], c.ev0, 0));
  for (int j = 0; j < r; ++j) {
    SpFactor f;
    f.Dt = dt[j];
    f.Lt = tiles[j].Lt;
    f.Ut = tiles[j].Ut;
    f.DinvL = tiles[j].DinvL;
    f.DinvU = tiles[j].DinvU;
    f.lmask = c.fp_lmask.as<unsigned>() + lmask_per_pole * j;
    FactorDevState ds;
    ds.fail_index = reinterpret_cast<int*>(c.fstate_mem.as<unsigned long long>() + 2 * j);
    ds.min_ratio_bits = c.fstate_mem.as<unsigned long long>() + 2 * j + 1;
    pd.scratch = c.fp_scratch.as<cd>() + scratch_per_pole * j;
    sp_factor(c.pole_streams[j], c.sgeom, f, c.sp_nnz, c.sp_er.as<int>(), c.sp_ec.as<int>(), c.sp_ea.as<double>(),
              c.sp_eb.as<double>(), c.cx, sig[j].real(), sig[j].imag(), c.rownorm_mem.as<double>() + c.sgeom.npad * j,
              c.sp_pad_rows.as<int>(), c.sp_npads, ds, c.sp_err.as<int>(), pd);
    if (mstore) {  // sweep factors: occupancy masks, then the swizzled sweep layout
      tile_masks(c.pole_streams[j], tiles[j].DinvL, nb, tiles[j].mDL);
      tile_masks(c.pole_streams[j], tiles[j].DinvU, nb, tiles[j].mDU);
      tile_masks(c.pole_streams[j], tiles[j].Lt, ntiles, tiles[j].mLt);
      tile_masks(c.pole_streams[j], tiles[j].Ut, ntiles, tiles[j].mUt);
      if (j == 0) {  // work accounting of the sweeps (one pole: all share the structure)
        c.sp_err.ensure(sizeof(int) * 4 + 2 * sizeof(unsigned long long));
        unsigned long long* wk = reinterpret_cast<unsigned long long*>(c.sp_err.as<int>() + 4);
        CK(cudaMemsetAsync(wk, 0, 2 * sizeof(unsigned long long), c.pole_streams[0]));
        tile_work(c.pole_streams[0], tiles[0].DinvL, tiles[0].mDL, nb, wk);
        tile_work(c.pole_streams[0], tiles[0].DinvU, tiles[0].mDU, nb, wk);
        tile_work(c.pole_streams[0], tiles[0].Lt, tiles[0].mLt, ntiles, wk);
        tile_work(c.pole_streams[0], tiles[0].Ut, tiles[0].mUt, ntiles, wk);
      }
      swizzle_tiles(c.pole_streams[j], tiles[j].DinvL, nb);
      swizzle_tiles(c.pole_streams[j], tiles[j].DinvU, nb);
      swizzle_tiles(c.pole_streams[j], tiles[j].Lt, ntiles);
      swizzle_tiles(c.pole_streams[j], tiles[j].Ut, ntiles);
      tiles[j].swz = true;
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(c.ev2, c.pole_streams[j]));
    CK(cudaStreamWaitEvent(c.st, c.ev2, 0));
  }
  CK(cudaEventRecord(c.ev1, c.st));
  CK(cudaStreamSynchronize(c.st));
  for (int j = 0; j < r; ++j) CK(cudaStreamSynchronize(c.pole_streams[j]));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, c.ev0, c.ev1));
  c.last_ms[1] = ms;
  clk.mark("numeric (launch+device)");
  int serr = 0;
  unsigned long long wk[2] = {0, 0};
  CK(cudaMemcpyAsync(&serr, c.sp_err.p, sizeof(int), cudaMemcpyDeviceToHost, c.st));
  if (mstore)
    CK(cudaMemcpyAsync(wk, c.sp_err.as<int>() + 4, sizeof(wk), cudaMemcpyDeviceToHost, c.st));
  CK(cudaStreamSynchronize(c.st));
  if (mstore) {
    c.work_nnz = static_cast<int64_t>(wk[0]);
    c.work_exec = static_cast<int64_t>(wk[1]);
  }
  if (serr) throw ZoloError(ZOLO_ERR_NUMERICAL, "zolo_factorize: symbolic structure does not cover the fill");
  CK(cudaMemcpyAsync(fs.data(), c.fstate_mem.p, fs.size() * 8, cudaMemcpyDeviceToHost, c.st));
  CK(cudaStreamSynchronize(c.st));
  fail.assign(r, -1);
  min_ratio.assign(r, 0.0);
  for (int j = 0; j < r; ++j) {
    fail[j] = static_cast<int>(static_cast<uint32_t>(fs[2 * j] & 0xffffffffull));
    std::memcpy(&min_ratio[j], &fs[2 * j + 1], 8);
  }
}

void do_factorize_sparse(zolo_ctx& c, const int64_t* perm_in, zolo_factor_stats* stats) {
  sparse_symbolic(c, perm_in);
  const double* poles = c.design.data() + ZOLO_DESIGN_HEAD;
  std::vector<std::complex<double>> sig;
  for (int j : c.own) sig.emplace_back(poles[2 * j], poles[2 * j + 1]);
  std::vector<int> fail;
  std::vector<double> mr;
  size_t per_pole = 0;
  sparse_numeric(c, sig, c.tiles_mem, &c.sp_masks, c.tiles, c.sp_dt, fail, mr, &per_pole);
  int fail_any = -1;
  for (size_t j = 0; j < sig.size(); ++j) {
    if (stats) {
      stats[j].bandwidth = -1;
      stats[j].stored_entries = static_cast<int64_t>(per_pole);
      stats[j].min_pivot_ratio = mr[j];
      stats[j].pivot_index = fail[j];
    }
    if (fail[j] >= 0 && fail_any < 0) fail_any = fail[j];
  }
  c.factored = fail_any < 0;
  c.ncap = 0;
  c.unrefined_res = -1.0;  // measured again with the new factors
  if (fail_any >= 0)
    throw ZoloError(ZOLO_ERR_FACTORIZATION, "factorize: pivot " + std::to_string(fail_any) + " below threshold");
}

// poles of this context (j = rank, rank + nranks, ... < r) and their weights, local order
void refresh_own(zolo_ctx& c) {
  c.own.clear();
  if (c.hybrid)
    c.own.push_back(c.hy_pole);
  else
    for (int j = c.shard_rank; j < c.r; j += c.shard_size) c.own.push_back(j);
  std::vector<cd> w(std::max<size_t>(c.own.size(), 1), mk(0.0, 0.0));
  for (size_t k = 0; k < c.own.size(); ++k) w[k] = mk(c.eff_w[c.own[k]].real(), c.eff_w[c.own[k]].imag());
  upload(c.weights_d, w, c.st);
  c.factored = false;
  c.ncap = 0;
}

void ensure_workspace(zolo_ctx& c, int64_t ncols) {
  const int64_t ld = c.geom.npad;
  const size_t es = c.es();
  if (ncols <= c.ncap) return;
  const int64_t nc = ncols;
  c.vin_orig.ensure(es * c.n * nc);
  c.vin.ensure(es * ld * nc);
  c.vout.ensure(es * ld * nc);
  c.w.ensure(es * ld * nc);
  c.bbuf.ensure(sizeof(cd) * ld * nc);
  const int nch = c.nchains();
  while (static_cast<int>(c.xbuf.size()) < nch) c.xbuf.emplace_back(new DevMem());
  while (static_cast<int>(c.cbuf.size()) < nch) c.cbuf.emplace_back(new DevMem());
  // cbuf: the DAG chunk partials (32 x nslots rows)
  const int64_t crows = static_cast<int64_t>(TILE) * std::max(c.sp_nslots, 1);
  for (int i = 0; i < nch; ++i) {
    c.xbuf[i]->ensure(sizeof(cd) * ld * nc);
    c.cbuf[i]->ensure(sizeof(cd) * crows * nc);
  }
  // sweep task width: 64 columns halve the tile traffic and the per-task overhead per column, but
  // pad a block of fewer than 128 columns too much (ZOLO_SWEEP_COLS: development override)
  static const int swc_env = env_int("ZOLO_SWEEP_COLS", 0);
  c.swc = (swc_env == 32 || swc_env == 64) ? swc_env : (nc >= 128 ? 64 : 32);
  std::vector<Chain> fwd(nch), bwd(nch);
  for (int p = 0; p < c.nloc(); ++p) {
    const FactorTiles& t = c.tiles[p];
    const cd* b = c.bbuf.as<cd>();
    if (c.cx) {
      cd* x = c.xbuf[2 * p]->as<cd>();
      cd* xa = c.xbuf[2 * p + 1]->as<cd>();
      cd* cb = c.cbuf[2 * p]->as<cd>();
      cd* cba = c.cbuf[2 * p + 1]->as<cd>();
      // solve:   y = DinvL b - L~ y ;  x = DinvU y - U~ x
      // adjoint: z = b - U~^H z (z_i = U_ii^H y_i) ; w = DinvU^H z - L~^H w (w_i = L_ii^H x_i),
      //          then x_i = DinvL_i^H w_i (blockdiag post-pass)
      fwd[2 * p] = Chain{t.Lt, t.DinvL, t.mLt, t.mDL, b, x, cb, FWD_L, 0, nullptr};
      bwd[2 * p] = Chain{t.Ut, t.DinvU, t.mUt, t.mDU, x, x, cb, BWD_U, 0, nullptr};
      fwd[2 * p + 1] = Chain{t.Ut, nullptr, t.mUt, nullptr, b, xa, cba, FWD_UH, 0, nullptr};
      bwd[2 * p + 1] = Chain{t.Lt, t.DinvU, t.mLt, t.mDU, xa, xa, cba, BWD_LH, 0, nullptr};
    } else {
      cd* x = c.xbuf[p]->as<cd>();
      cd* cb = c.cbuf[p]->as<cd>();
      fwd[p] = Chain{t.Lt, t.DinvL, t.mLt, t.mDL, b, x, cb, FWD_L, 0, nullptr};
      bwd[p] = Chain{t.Ut, t.DinvU, t.mUt, t.mDU, x, x, cb, BWD_U, 0, nullptr};
    }
  }
  // the sweeps' x-block tensor maps (src, dst, cbuf per chain), sized for the workspace's columns
  auto with_maps = [&](std::vector<Chain>& chs, DevMem& maps) {
    struct alignas(64) XMap {
      unsigned char b[XMAP_BYTES];
    };
    std::vector<XMap> hm(3 * chs.size());
    maps.ensure(sizeof(XMap) * hm.size());
    for (size_t ch = 0; ch < chs.size(); ++ch) {
      const cd* bufs[3] = {chs[ch].src, chs[ch].dst, chs[ch].cbuf};
      const int64_t lds[3] = {ld, ld, crows};
      for (int k = 0; k < 3; ++k)
        if (!encode_xblock_map(&hm[3 * ch + k], bufs[k], lds[k], nc, c.swc))
          throw ZoloError(ZOLO_ERR_CUDA, "cuTensorMapEncodeTiled failed for a sweep block");
      chs[ch].tmaps = maps.as<unsigned char>() + 3 * ch * sizeof(XMap);
    }
    upload(maps, hm, c.st);
  };
  with_maps(fwd, c.tmaps_fwd);
  with_maps(bwd, c.tmaps_bwd);
  upload(c.chains_fwd, fwd, c.st);
  upload(c.chains_bwd, bwd, c.st);
  if (c.refine) {  // refinement sweeps: same factors, in place over the residual blocks
    while (static_cast<int>(c.rbuf.size()) < nch) c.rbuf.emplace_back(new DevMem());
    std::vector<cd> sig(nch);
    const double* poles = c.design.data() + ZOLO_DESIGN_HEAD;
    for (int ch = 0; ch < nch; ++ch) {
      c.rbuf[ch]->ensure(sizeof(cd) * ld * nc);
      cd* rb = c.rbuf[ch]->as<cd>();
      fwd[ch].src = rb;
      fwd[ch].dst = rb;
      bwd[ch].src = rb;
      bwd[ch].dst = rb;
      // chain 2p solves K_p = A - sigma_p B; chain 2p + 1 (complex pencils) K_p^H = A - conj(sigma_p) B
      const int p = c.cx ? ch / 2 : ch;
      const double im = poles[2 * c.own[p] + 1];
      sig[ch] = mk(poles[2 * c.own[p]], (c.cx && (ch & 1)) ? -im : im);
    }
    with_maps(fwd, c.tmaps_fwd_ref);
    with_maps(bwd, c.tmaps_bwd_ref);
    upload(c.chains_fwd_ref, fwd, c.st);
    upload(c.chains_bwd_ref, bwd, c.st);
    upload(c.chain_sigma, sig, c.st);
  }
  const int64_t ngroups = (nc + CG - 1) / CG;
  // [(reserved) nch x ngroups uint64 | block flags: nch x ngroups x nbk int |
  //  DAG chunk flags: nch x dag_groups x nslots int]; all epoch-stamped, zeroed with the epoch
  const int64_t nbflags = static_cast<int64_t>(nch) * ngroups * c.geom.nbk;
  const int64_t nflags = nbflags + static_cast<int64_t>(nch) * dag_groups(nc, 32) * c.sp_nslots;
  if (nflags > c.flags_cap || static_cast<int64_t>(nch) * ngroups > c.prog_cap) {
    c.prog_cap = static_cast<int64_t>(nch) * ngroups;
    const size_t bytes = sizeof(unsigned long long) * c.prog_cap + sizeof(int) * nflags;
    c.flags.ensure(bytes);
    CK(cudaMemsetAsync(c.flags.p, 0, c.flags.bytes, c.st));
    c.flags_cap = nflags;
    c.epoch = 0;
  }
  c.cflags_off = nbflags;
  if (c.counter.ensure(sizeof(int) * 4)) CK(cudaMemsetAsync(c.counter.p, 0, sizeof(int) * 4, c.st));
  c.act_d.ensure(sizeof(int) * nc);
  for (int** hp : {&c.act_h, &c.done_h, &c.act_hq[0], &c.act_hq[1], &c.act_hq[2], &c.act_hq[3], &c.done_hq[0],
                    &c.done_hq[1], &c.done_hq[2], &c.done_hq[3]}) {
    if (*hp) cudaFreeHost(*hp);
    CK(cudaMallocHost(hp, sizeof(int) * nc));
  }
  c.ncap = nc;
  c.maxit_cap = 0;  // GMRES state is sized per (ncap, maxit)
}

// this rank's Krylov rows [r0, r1) (all rows unless row-sharded)
inline int64_t row_lo(const zolo_ctx& c) { return c.row_shard ? std::min<int64_t>(c.geom.npad, c.shard_rank * c.rb) : 0; }
inline int64_t row_hi(const zolo_ctx& c) {
  return c.row_shard ? std::min<int64_t>(c.geom.npad, (c.shard_rank + 1) * c.rb) : c.geom.npad;
}

// w[:, act] = (rank 0: constant v) + the context's poles' terms (filter_engine.hpp:60-80).
// Pole-sharded, row-sharded Arnoldi: written row-blocked, reduce-scattered over the ranks (each
// rank receives its row block of G v, summed over all poles) and unpacked into w's local rows.
// Pole-sharded, replicated Arnoldi: computed compacted, all-reduced, scattered -- every rank ends
// with the same bits. Without a communicator (nranks > 1, no unique id) the rank's partial sum
// is returned.
void combine_g(zolo_ctx& c, const void* vsrc, const int* act, int na, std::vector<cd*>& xs, void* wdst) {
  const int64_t ld = c.geom.npad, n = ld;
  const bool sharded = c.shard_size > 1;
  if (sharded && c.row_shard && c.in_filter) {
    const int P = c.shard_size;
    const int64_t rb = c.rb;
    c.wc.ensure(c.es() * rb * P * std::max(na, 1));
    c.wloc.ensure(c.es() * rb * std::max(na, 1));
    if (c.cx)
      Krylov<cd>::combine_blocked(c.st, ld, rb, P, c.local_constant(), reinterpret_cast<const cd*>(vsrc), act, na,
                                  xs.data(), c.weights_d.as<cd>(), c.nloc(), c.wc.as<cd>());
    else
      Krylov<double>::combine_blocked(c.st, ld, rb, P, c.local_constant(), reinterpret_cast<const double*>(vsrc),
                                      act, na, xs.data(), c.weights_d.as<cd>(), c.nloc(), c.wc.as<double>());
    c.coll->reduce_scatter(c.wc.as<double>(), c.wloc.as<double>(), static_cast<size_t>(rb) * na * (c.es() / 8), c.st);
    const int64_t r0 = row_lo(c), rows = row_hi(c) - r0;
    if (c.cx)
      Krylov<cd>::unpack_rows(c.st, c.wloc.as<cd>(), r0, rows, rb, act, na, reinterpret_cast<cd*>(wdst), ld);
    else
      Krylov<double>::unpack_rows(c.st, c.wloc.as<double>(), r0, rows, rb, act, na, reinterpret_cast<double*>(wdst),
                                  ld);
    return;
  }
  void* out = wdst;
  if (sharded) {
    c.wc.ensure(c.es() * ld * std::max(na, 1));
    out = c.wc.p;
  }
  if (c.cx)
    Krylov<cd>::combine(c.st, n, ld, c.local_constant(), reinterpret_cast<const cd*>(vsrc), act, na, xs.data(),
                        c.weights_d.as<cd>(), c.nloc(), reinterpret_cast<cd*>(out), sharded);
  else
    Krylov<double>::combine(c.st, n, ld, c.local_constant(), reinterpret_cast<const double*>(vsrc), act, na,
                            xs.data(), c.weights_d.as<cd>(), c.nloc(), reinterpret_cast<double*>(out), sharded);
  if (!sharded) return;
  if (c.coll) c.coll->allreduce(c.wc.as<double>(), static_cast<size_t>(ld) * na * (c.es() / 8), c.st);
  if (c.cx)
    Krylov<cd>::scatter_cols(c.st, ld, c.wc.as<cd>(), act, na, reinterpret_cast<cd*>(wdst));
  else
    Krylov<double>::scatter_cols(c.st, ld, c.wc.as<double>(), act, na, reinterpret_cast<double*>(wdst));
}

// DAG sweeps (forward, backward, and the adjoint post-pass) of the chains
// [first, first + nsub) on bbuf's first na (compacted) columns -> their xbuf.
// refinement = true: the in-place sweeps over the chains' residual blocks (rbuf).
void sweep_sparse(zolo_ctx& c, int first, int nsub, int na, unsigned long long* trace = nullptr,
                  bool refinement = false) {
  const int64_t ld = c.geom.npad;
  unsigned long long* fx = c.flags.as<unsigned long long>();
  int* fc = reinterpret_cast<int*>(fx + c.prog_cap);
  int* cf = fc + c.cflags_off;
  const Chain* cfw = (refinement ? c.chains_fwd_ref : c.chains_fwd).as<Chain>() + first;
  const Chain* cbw = (refinement ? c.chains_bwd_ref : c.chains_bwd).as<Chain>() + first;
  const int64_t ldp = static_cast<int64_t>(TILE) * std::max(c.sp_nslots, 1);  // cbuf rows (ensure_workspace)
  if ((static_cast<int64_t>(c.epoch) + 3) * DAG_GENS >= (int64_t(1) << 31)) {  // partial-slot stamps near overflow
    CK(cudaMemsetAsync(c.flags.p, 0, c.flags.bytes, c.st));
    c.epoch = 0;
  }
  const int g1 = dag_trsm_launch(c.st, c.sgeom, c.sched_fwd, cfw, nsub, na, c.swc, ld, ldp, fc, cf, ++c.epoch,
                                 c.counter.as<int>(), c.num_sms, trace, c.act_d.as<int>(), c.lag_done);
  const int g2 = dag_trsm_launch(c.st, c.sgeom, c.sched_bwd, cbw, nsub, na, c.swc, ld, ldp, fc, cf, ++c.epoch,
                                 c.counter.as<int>(), c.num_sms, nullptr, c.act_d.as<int>(), c.lag_done);
  if (g1 < 0 || g2 < 0) throw ZoloError(ZOLO_ERR_DOMAIN, "triangular solve: more than 32 chains in one launch");
  if (c.cx) {  // the adjoint chains' post-pass x_i = DinvL_i^H w_i, one launch
    std::vector<const cd*> dv;
    std::vector<cd*> xv;
    for (int ci = first; ci < first + nsub; ++ci)
      if (ci & 1) {
        dv.push_back(c.tiles[ci / 2].DinvL);
        xv.push_back((refinement ? c.rbuf[ci] : c.xbuf[ci])->as<cd>());
      }
    blockdiag_apply(c.st, c.geom.nbk, dv.data(), xv.data(), static_cast<int>(dv.size()), true, na, ld);
  }
}

// Residual-correction refinement of every chain's solution (zolo_set_refinement):
// r = b - K x (K^H for the adjoint chains) from the pencil in FP64, d = K^-1 r by the same
// sweeps in place over r, x += d.
void refine_solves(zolo_ctx& c, int na, int first = 0, int nsub = -1) {
  Nvtx range("zolo::refine");
  const int64_t ld = c.geom.npad, n = ld;
  const int nch = nsub < 0 ? c.nchains() : nsub;
  std::vector<cd*> xs(nch), rs(nch);
  for (int i = 0; i < nch; ++i) xs[i] = c.xbuf[first + i]->as<cd>(), rs[i] = c.rbuf[first + i]->as<cd>();
  for (int step = 0; step < c.refine; ++step) {
    if (c.cx)
      Krylov<cd>::shifted_residual(c.st, n, ld, c.arp_d.as<int>(), c.aci_d.as<int>(), c.av_d.as<cd>(),
                                   c.b_identity ? nullptr : c.brp_d.as<int>(), c.bci_d.as<int>(), c.bv_d.as<cd>(),
                                   c.bbuf.as<cd>(), xs.data(), rs.data(), c.chain_sigma.as<cd>() + first, nch, na);
    else
      Krylov<double>::shifted_residual(c.st, n, ld, c.arp_d.as<int>(), c.aci_d.as<int>(), c.av_d.as<double>(),
                                       c.b_identity ? nullptr : c.brp_d.as<int>(), c.bci_d.as<int>(),
                                       c.bv_d.as<double>(), c.bbuf.as<cd>(), xs.data(), rs.data(),
                                       c.chain_sigma.as<cd>() + first, nch, na);
    if (step == 0 && c.in_filter && c.unrefined_res < 0.0 && first == 0 && na > 0) {
      // ||b - K x||_F / ||b||_F of the unrefined solves, worst chain (once per factorization)
      c.norm_buf.ensure(sizeof(double) * static_cast<size_t>(nch + 1) * na);
      double* nb = c.norm_buf.as<double>();
      for (int ch = 0; ch < nch; ++ch) Krylov<cd>::col_norms(c.st, rs[ch], ld, ld, na, nb + static_cast<size_t>(ch) * na);
      Krylov<cd>::col_norms(c.st, c.bbuf.as<cd>(), ld, ld, na, nb + static_cast<size_t>(nch) * na);
      std::vector<double> h(static_cast<size_t>(nch + 1) * na);
      CK(cudaMemcpyAsync(h.data(), nb, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, c.st));
      CK(cudaStreamSynchronize(c.st));
      double b2 = 0.0, worst = 0.0;
      for (int a = 0; a < na; ++a) b2 += h[static_cast<size_t>(nch) * na + a] * h[static_cast<size_t>(nch) * na + a];
      for (int ch = 0; ch < nch; ++ch) {
        double r2 = 0.0;
        for (int a = 0; a < na; ++a) r2 += h[static_cast<size_t>(ch) * na + a] * h[static_cast<size_t>(ch) * na + a];
        worst = std::max(worst, r2);
      }
      c.unrefined_res = b2 > 0.0 && std::isfinite(worst) ? std::sqrt(worst / b2) : 1.0;
    }
    sweep_sparse(c, first, nch, na, nullptr, true);
    add_corrections(c.st, ld, xs.data(), rs.data(), nch, na);
  }
}

// out[:, a] = B v[:, act[a]] (complex, the sweeps' input) over the device rows: BSR kernel when
// the pencil has atoms (zolo_set_block_size) kept contiguous by the ordering, CSR otherwise.
void device_apply_b(zolo_ctx& c, const void* v, const int* act, int na, cd* out) {
  const int64_t ld = c.geom.npad, n = ld;
  if (c.bsr_dev && !c.b_identity) {
    if (c.cx)
      Krylov<cd>::bsr_spmm(c.st, c.bsr_na, static_cast<int>(c.bsr), c.bbrp_d.as<int>(), c.bbci_d.as<int>(),
                           c.bbv_d.as<cd>(), c.brow0_d.as<int>(), reinterpret_cast<const cd*>(v), ld, act, na, nullptr,
                           out);
    else
      Krylov<double>::bsr_spmm(c.st, c.bsr_na, static_cast<int>(c.bsr), c.bbrp_d.as<int>(), c.bbci_d.as<int>(),
                               c.bbv_d.as<double>(), c.brow0_d.as<int>(), reinterpret_cast<const double*>(v), ld, act,
                               na, nullptr, out);
    zero_rows(c.st, c.sp_pad_rows.as<int>(), c.sp_npads, out, ld, na);
    return;
  }
  if (c.cx)
    Krylov<cd>::apply_b(c.st, n, ld, c.b_identity ? nullptr : c.brp_d.as<int>(), c.bci_d.as<int>(), c.bv_d.as<cd>(),
                        reinterpret_cast<const cd*>(v), act, na, out);
  else
    Krylov<double>::apply_b(c.st, n, ld, c.b_identity ? nullptr : c.brp_d.as<int>(), c.bci_d.as<int>(),
                            c.bv_d.as<double>(), reinterpret_cast<const double*>(v), act, na, out);
}

// out (ld x k, device rows) = M x, M = A (which 0) or B (which 1); BSR when available
template <class S>
void device_spmm(zolo_ctx& c, int which, const S* x, int64_t k, S* out) {
  const int64_t ld = c.geom.npad;
  if (c.bsr_dev) {
    Krylov<S>::bsr_spmm(c.st, c.bsr_na, static_cast<int>(c.bsr), (which ? c.bbrp_d : c.abrp_d).template as<int>(),
                        (which ? c.bbci_d : c.abci_d).template as<int>(), (which ? c.bbv_d : c.abv_d).template as<S>(),
                        c.brow0_d.as<int>(), x, ld, nullptr, k, out, nullptr);
    return;
  }
  if (which == 0)
    Krylov<S>::spmm(c.st, ld, ld, c.arp_d.as<int>(), c.aci_d.as<int>(), c.av_d.as<S>(), x, k, out);
  else
    Krylov<S>::spmm(c.st, ld, ld, c.brp_d.as<int>(), c.bci_d.as<int>(), c.bv_d.as<S>(), x, k, out);
}

float apply_g_hybrid(zolo_ctx& c, const void* vsrc, int na, void* wdst);

// G applied to the columns act[0..na) of vsrc (ld x ncap, S) -> w[:, act].
float apply_g_device(zolo_ctx& c, const void* vsrc, int na, void* wdst) {
  Nvtx range("zolo::apply_g");
  if (c.hybrid) return apply_g_hybrid(c, vsrc, na, wdst);
  const int64_t ld = c.geom.npad;  // device rows: padding rows (anywhere in ND order) are zero
  const int* act = c.act_d.as<int>();
  const int nch = c.nchains();
  std::vector<cd*> xs(nch);
  for (int i = 0; i < nch; ++i) xs[i] = c.xbuf[i]->as<cd>();
  device_apply_b(c, vsrc, act, na, c.bbuf.as<cd>());
  CK(cudaEventRecord(c.ev2_use ? c.ev2_use : c.ev2, c.st));
  // ZOLO_TRACE=<file>: per-task timestamps of the first forward sweep (development aid,
  // tools/dag2_trace_analyze.py)
  static const char* dag_trace = std::getenv("ZOLO_TRACE");
  unsigned long long* dtr = nullptr;
  const size_t ntask = static_cast<size_t>(c.sched_fwd.ntask) * nch * dag_groups(na, c.swc);
  if (dag_trace && !c.trace_done) {
    c.trace_buf.ensure(sizeof(unsigned long long) * 6 * ntask);
    CK(cudaMemsetAsync(c.trace_buf.p, 0, sizeof(unsigned long long) * 6 * ntask, c.st));
    dtr = c.trace_buf.as<unsigned long long>();
  }
  sweep_sparse(c, 0, nch, na, dtr);
  if (c.refine && !c.refine_skip) refine_solves(c, na);
  if (dtr) {
    std::vector<unsigned long long> h(6 * ntask);
    CK(cudaMemcpyAsync(h.data(), dtr, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    if (FILE* fh = std::fopen(dag_trace, "w")) {
      std::fprintf(fh, "# nb %d chains %d groups %d critical_path %lld schedule %d slots %d\n", c.geom.nbk, nch,
                   dag_groups(na, c.swc), static_cast<long long>(c.critical_path), c.sched_fwd.ntask, c.sched_fwd.nslots);
      for (size_t q = 0; q < ntask; ++q)
        std::fprintf(fh, "%llu %llu %llu %llu %llu %llu\n", h[6 * q], h[6 * q + 1], h[6 * q + 2], h[6 * q + 3],
                     h[6 * q + 4], h[6 * q + 5]);
      std::fclose(fh);
    }
    c.trace_done = true;
  }
  CK(cudaEventRecord(c.ev3_use ? c.ev3_use : c.ev3, c.st));
  CK(cudaGetLastError());
  combine_g(c, vsrc, act, na, xs, wdst);
  CK(cudaGetLastError());
  return 0.0f;
}

template <class S>
void ensure_gmres(zolo_ctx& c, int maxit) {
  if (maxit <= c.maxit_cap) return;
  const int64_t nv = c.ncap;
  const int q = 2 * c.r;
  const size_t es = sizeof(S);
  c.gH.ensure(es * nv * (maxit + 1) * maxit);
  c.gR.ensure(sizeof(cd) * nv * q * maxit * maxit);
  c.gG.ensure(sizeof(cd) * nv * q * (maxit + 1));
  c.gROT.ensure(sizeof(cd) * nv * q * 2 * maxit);
  c.gY.ensure(sizeof(cd) * nv * q * maxit);
  c.gZ.ensure(sizeof(cd) * nv * maxit);
  c.gres.ensure(sizeof(double) * nv * q);
  c.gfrozen.ensure(sizeof(int) * nv * q);
  c.gmlen.ensure(sizeof(int) * nv * q);
  c.gbeta.ensure(sizeof(double) * nv);
  c.gmcol.ensure(sizeof(int) * nv);
  c.ghappy.ensure(sizeof(int) * nv);
  c.gdone.ensure(sizeof(int) * nv);
  c.gwnorm.ensure(sizeof(double) * nv);
  const int64_t nchunk = (c.geom.npad + CHUNK - 1) / CHUNK;
  c.partial.ensure(3 * es * nv * nchunk * (maxit + 1) + 64);
  c.hsave.ensure(es * nv * (maxit + 1));
  c.basis_ptrs.ensure(sizeof(void*) * (maxit + 1));
  c.maxit_cap = maxit;
}

GmresDev gmres_view(zolo_ctx& c, int maxit) {
  GmresDev g;
  g.maxit = maxit;
  g.q = 2 * c.r;
  g.nv = static_cast<int>(c.ncap);
  g.H = c.gH.p;
  g.R = c.gR.as<cd>();
  g.G = c.gG.as<cd>();
  g.ROT = c.gROT.as<cd>();
  g.Y = c.gY.as<cd>();
  g.Z = c.gZ.as<cd>();
  g.res = c.gres.as<double>();
  g.frozen = c.gfrozen.as<int>();
  g.mlen = c.gmlen.as<int>();
  g.beta = c.gbeta.as<double>();
  g.mcol = c.gmcol.as<int>();
  g.happy = c.ghappy.as<int>();
  g.done = c.gdone.as<int>();
  g.wnorm = c.gwnorm.as<double>();
  g.shifts = c.shifts_d.as<cd>();
  g.coef = c.coef_d.as<double>();
  return g;
}

void* basis_block(zolo_ctx& c, int i) {
  const size_t bytes = c.es() * c.geom.npad * c.ncap;
  while (static_cast<int>(c.basis.size()) <= i) c.basis.emplace_back(new DevMem());
  if (c.basis[i]->ensure(bytes)) {
    void* p = c.basis[i]->p;
    CK(cudaMemcpyAsync(c.basis_ptrs.as<void*>() + i, &p, sizeof(void*), cudaMemcpyHostToDevice, c.st));
    CK(cudaStreamSynchronize(c.st));
  }
  return c.basis[i]->p;
}

// ---- hybrid inner solve (BASELINE config 2) --------
// Only pole p is factored. With M = K_p^{-1} B and delta_j = s_j - s_p,
//   K_j^{-1} B v = (I - delta_j M)^{-1} K_p^{-1} B v = -(1/delta_j) (M - I/delta_j)^{-1} x0,
// x0 = K_p^{-1} B v, so one Krylov space K_m(M, x0) per column serves every
// other pole (shift-invariance): the batched multi-shift GMRES of the outer
// loop (krylov.cu) runs on M with shifts -1/delta_j and folds the weighted
// solutions sum_j w_j (-1/delta_j) y_j into one block (complex coefficients).
// Complex pencils repeat it for the adjoint solves with M' = K_p^{-H} B and the
// conjugated shifts / weights.
void ensure_inner(zolo_ctx& c, int64_t nv, int q, int maxit) {
  const int64_t ld = c.geom.npad;
  if (nv > c.incap) {
    for (int k = 0; k < 2; ++k) {
      c.hy_x0[k].ensure(sizeof(cd) * ld * nv);
      c.hy_y[k].ensure(sizeof(cd) * ld * nv);
    }
    c.hy_w.ensure(sizeof(cd) * ld * nv);
    c.act_in_d.ensure(sizeof(int) * nv);
    if (c.act_in_h) cudaFreeHost(c.act_in_h);
    CK(cudaMallocHost(&c.act_in_h, sizeof(int) * nv));
    c.imaxit_cap = 0;
    for (auto& b : c.ibasis) b->release();
    c.incap = nv;
  }
  if (maxit > c.imaxit_cap) {
    nv = c.incap;
    const size_t es = sizeof(cd);
    c.iH.ensure(es * nv * (maxit + 1) * maxit);
    c.iR.ensure(sizeof(cd) * nv * q * maxit * maxit);
    c.iG.ensure(sizeof(cd) * nv * q * (maxit + 1));
    c.iROT.ensure(sizeof(cd) * nv * q * 2 * maxit);
    c.iY.ensure(sizeof(cd) * nv * q * maxit);
    c.iZ.ensure(sizeof(cd) * nv * maxit);
    c.ires.ensure(sizeof(double) * nv * q);
    c.ifrozen.ensure(sizeof(int) * nv * q);
    c.imlen.ensure(sizeof(int) * nv * q);
    c.ibeta.ensure(sizeof(double) * nv);
    c.imcol.ensure(sizeof(int) * nv);
    c.ihappy.ensure(sizeof(int) * nv);
    c.idone.ensure(sizeof(int) * nv);
    c.iwnorm.ensure(sizeof(double) * nv);
    const int64_t nchunk = (ld + CHUNK - 1) / CHUNK;
    c.ipartial.ensure(2 * es * nv * nchunk * (maxit + 1) + 64);
    c.ihsave.ensure(es * nv * (maxit + 1));
    c.ibasis_ptrs.ensure(sizeof(void*) * (maxit + 1));
    while (static_cast<int>(c.ibasis.size()) <= maxit) c.ibasis.emplace_back(new DevMem());
    std::vector<void*> bp(maxit + 1);
    for (int i = 0; i <= maxit; ++i) {
      c.ibasis[i]->ensure(sizeof(cd) * ld * c.incap);
      bp[i] = c.ibasis[i]->p;
    }
    CK(cudaMemcpyAsync(c.ibasis_ptrs.p, bp.data(), sizeof(void*) * bp.size(), cudaMemcpyHostToDevice, c.st));
    CK(cudaStreamSynchronize(c.st));
    c.imaxit_cap = maxit;
  }
}

// inner shifts / folded coefficients of problem k (0: solve, 1: adjoint)
void hybrid_setup(zolo_ctx& c) {
  const double* poles = c.design.data() + ZOLO_DESIGN_HEAD;
  const std::complex<double> sp(poles[2 * c.hy_pole], poles[2 * c.hy_pole + 1]);
  for (int k = 0; k < 2; ++k) {
    std::vector<cd> sh, cf;
    for (int j = 0; j < c.r; ++j) {
      if (j == c.hy_pole) continue;
      std::complex<double> d = std::complex<double>(poles[2 * j], poles[2 * j + 1]) - sp;
      std::complex<double> w = c.eff_w[j];
      if (k == 1) {
        d = std::conj(d);
        w = std::conj(w);
      }
      const std::complex<double> s = -1.0 / d, co = w * (-1.0 / d);
      sh.push_back(mk(s.real(), s.imag()));
      cf.push_back(mk(co.real(), co.imag()));
    }
    if (sh.empty()) sh.push_back(mk(0.0, 0.0)), cf.push_back(mk(0.0, 0.0));
    upload(c.hy_shifts[k], sh, c.st);
    upload(c.hy_ccoef[k], cf, c.st);
  }
  const std::complex<double> w0 = c.eff_w[c.hy_pole];
  upload(c.hy_weights, std::vector<cd>{mk(w0.real(), w0.imag()), mk(1.0, 0.0)}, c.st);
}

GmresDev inner_view(zolo_ctx& c, int k, int nv, int q, int maxit) {
  GmresDev g;
  g.maxit = maxit;
  g.q = q;
  g.nv = nv;
  g.H = c.iH.p;
  g.R = c.iR.as<cd>();
  g.G = c.iG.as<cd>();
  g.ROT = c.iROT.as<cd>();
  g.Y = c.iY.as<cd>();
  g.Z = c.iZ.as<cd>();
  g.res = c.ires.as<double>();
  g.frozen = c.ifrozen.as<int>();
  g.mlen = c.imlen.as<int>();
  g.beta = c.ibeta.as<double>();
  g.mcol = c.imcol.as<int>();
  g.happy = c.ihappy.as<int>();
  g.done = c.idone.as<int>();
  g.wnorm = c.iwnorm.as<double>();
  g.shifts = c.hy_shifts[k].as<cd>();
  g.coef = nullptr;
  g.ccoef = c.hy_ccoef[k].as<cd>();
  return g;
}

// y[:, 0:na] = sum_j ccoef_j (M_k + s_j I)^{-1} x0[:, 0:na] (compacted columns), M_0 = K_p^{-1} B,
// M_1 = K_p^{-H} B; the operator is applied through chain k of the factored pole.
void inner_gmres(zolo_ctx& c, int k, int na) {
  const int64_t ld = c.geom.npad, n = ld;
  const int q = c.r - 1, maxit = c.hy_max;
  GmresDev g = inner_view(c, k, na, q, maxit);
  const cd* x0 = c.hy_x0[k].as<cd>();
  cd* const* basis = c.ibasis_ptrs.as<cd*>();
  Krylov<cd>::col_norms(c.st, x0, ld, ld, na, g.beta);
  Krylov<cd>::scale_cols(c.st, x0, c.ibasis[0]->as<cd>(), n, ld, na, g.beta);
  gmres_init(c.st, g);
  std::vector<double> beta(na);
  CK(cudaMemcpyAsync(beta.data(), g.beta, sizeof(double) * na, cudaMemcpyDeviceToHost, c.st));
  CK(cudaStreamSynchronize(c.st));
  std::vector<int> active, done(na);
  for (int a = 0; a < na; ++a)
    if (beta[a] != 0.0) active.push_back(a);
  const int nchunk = static_cast<int>((ld + CHUNK - 1) / CHUNK);
  for (int it = 0; it < maxit && !active.empty(); ++it) {
    const int nai = static_cast<int>(active.size());
    std::memcpy(c.act_in_h, active.data(), sizeof(int) * nai);
    CK(cudaMemcpyAsync(c.act_in_d.p, c.act_in_h, sizeof(int) * nai, cudaMemcpyHostToDevice, c.st));
    const int* act = c.act_in_d.as<int>();
    // w = M V_it: B, then the sweeps of chain k, scattered back to the columns
    Krylov<cd>::apply_b(c.st, n, ld, c.b_identity ? nullptr : c.brp_d.as<int>(), c.bci_d.as<int>(),
                        c.cx ? c.bv_d.as<cd>() : c.bvc_d.as<cd>(), c.ibasis[it]->as<cd>(), act, nai,
                        c.bbuf.as<cd>());
    sweep_sparse(c, k, 1, nai);
    Krylov<cd>::scatter_cols(c.st, ld, c.xbuf[k]->as<cd>(), act, nai, c.hy_w.as<cd>());
    c.inner_solves += nai;
    c.hy_inner_its += nai;
    Krylov<cd>::arnoldi(c.st, 0, ld, ld, basis, it, c.hy_w.as<cd>(), act, nai, g, c.ipartial.as<double>(),
                        c.ihsave.as<cd>());
    Krylov<cd>::least_squares(c.st, act, nai, it, g, c.ipartial.as<double>(), nchunk, c.hy_tol);
    if (it + 1 < maxit) Krylov<cd>::next_basis(c.st, n, ld, c.hy_w.as<cd>(), c.ibasis[it + 1]->as<cd>(), act, nai, g);
    CK(cudaGetLastError());
    int spin_err[2] = {0, 0};
    CK(cudaMemcpyAsync(done.data(), g.done, sizeof(int) * na, cudaMemcpyDeviceToHost, c.st));
    CK(cudaMemcpyAsync(spin_err, c.counter.as<int>() + 2, sizeof(int) * 2, cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    if (spin_err[0] || spin_err[1]) throw ZoloError(ZOLO_ERR_CUDA, "triangular solve: dependency wait timed out");
    std::vector<int> next;
    for (int a : active)
      if (!done[a]) next.push_back(a);
    active.swap(next);
  }
  Krylov<cd>::assemble(c.st, n, ld, nullptr, basis, na, g, nullptr, c.hy_y[k].as<cd>());
  // every shift must have reached the inner tolerance (or a happy breakdown)
  std::vector<double> res(static_cast<size_t>(na) * q);
  std::vector<int> happy(na);
  CK(cudaMemcpyAsync(res.data(), g.res, sizeof(double) * res.size(), cudaMemcpyDeviceToHost, c.st));
  CK(cudaMemcpyAsync(happy.data(), g.happy, sizeof(int) * na, cudaMemcpyDeviceToHost, c.st));
  CK(cudaStreamSynchronize(c.st));
  double worst = 0.0;
  for (int a = 0; a < na; ++a)
    if (!happy[a] && beta[a] != 0.0)
      for (int j = 0; j < q; ++j) worst = std::max(worst, res[static_cast<size_t>(a) * q + j]);
  if (worst > 1e3 * c.hy_tol)
    throw ZoloError(ZOLO_ERR_NUMERICAL, "hybrid inner GMRES: relative residual " + std::to_string(worst) +
                                            " after " + std::to_string(maxit) + " iterations");
}

float apply_g_hybrid(zolo_ctx& c, const void* vsrc, int na, void* wdst) {
  const int64_t ld = c.geom.npad, n = ld;
  const int* act = c.act_d.as<int>();
  ensure_inner(c, c.ncap, std::max(c.r - 1, 1), c.hy_max);
  if (c.cx)
    Krylov<cd>::apply_b(c.st, n, ld, c.b_identity ? nullptr : c.brp_d.as<int>(), c.bci_d.as<int>(),
                        c.bv_d.as<cd>(), reinterpret_cast<const cd*>(vsrc), act, na, c.bbuf.as<cd>());
  else
    Krylov<double>::apply_b(c.st, n, ld, c.b_identity ? nullptr : c.brp_d.as<int>(), c.bci_d.as<int>(),
                            c.bv_d.as<double>(), reinterpret_cast<const double*>(vsrc), act, na, c.bbuf.as<cd>());
  CK(cudaEventRecord(c.ev2_use ? c.ev2_use : c.ev2, c.st));
  const int nch = c.nchains();  // 1 (solve) or 2 (solve + adjoint)
  sweep_sparse(c, 0, nch, na);
  for (int k = 0; k < nch; ++k)
    CK(cudaMemcpyAsync(c.hy_x0[k].p, c.xbuf[k]->p, sizeof(cd) * ld * na, cudaMemcpyDeviceToDevice, c.st));
  if (c.r > 1)
    for (int k = 0; k < nch; ++k) inner_gmres(c, k, na);
  else
    for (int k = 0; k < nch; ++k) CK(cudaMemsetAsync(c.hy_y[k].p, 0, sizeof(cd) * ld * na, c.st));
  CK(cudaEventRecord(c.ev3_use ? c.ev3_use : c.ev3, c.st));
  std::vector<cd*> xs;
  xs.push_back(c.hy_x0[0].as<cd>());
  if (c.cx) xs.push_back(c.hy_x0[1].as<cd>());
  xs.push_back(c.hy_y[0].as<cd>());
  if (c.cx) xs.push_back(c.hy_y[1].as<cd>());
  if (c.cx)
    Krylov<cd>::combine(c.st, n, ld, c.constant_term, reinterpret_cast<const cd*>(vsrc), act, na, xs.data(),
                        c.hy_weights.as<cd>(), 2, reinterpret_cast<cd*>(wdst));
  else
    Krylov<double>::combine(c.st, n, ld, c.constant_term, reinterpret_cast<const double*>(vsrc), act, na,
                            xs.data(), c.hy_weights.as<cd>(), 2, reinterpret_cast<double*>(wdst));
  CK(cudaGetLastError());
  return 0.0f;
}

template <class S>
int apply_filter_impl(zolo_ctx& c, const void* d_v, void* d_y, int64_t ncols, double tol, int64_t gmres_max,
                      zolo_report* rep) {
  Nvtx range("zolo::apply_filter");
  require(c.factored, "apply_filter: operator not factorized");
  require(c.shard_size == 1 || c.coll, "apply_filter: a pole-sharded context needs its communicator");
  // (the reference has no cap, gmres.hpp:98-101; the device Krylov kernels hold up to
  // KRYLOV_MAX basis vectors per column, krylov.cuh)
  require(gmres_max >= 1 && gmres_max <= KRYLOV_MAX,
          "apply_filter: gmres_max must be in [1, " + std::to_string(KRYLOV_MAX) + "]");
  const int64_t n = c.n, ld = c.geom.npad;
  const int maxit = static_cast<int>(gmres_max);
  const int q = 2 * c.r;
  if (c.row_shard) c.rb = ((ld + c.shard_size - 1) / c.shard_size + 31) / 32 * 32;
  ensure_workspace(c, ncols);
  ensure_gmres<S>(c, maxit);
  // basis pointers may predate a reallocation: refresh all
  for (int i = 0; i < static_cast<int>(c.basis.size()); ++i) {
    if (c.basis[i]->bytes < c.es() * ld * c.ncap) c.basis[i]->release();
  }
  std::vector<void*> bp;
  for (int i = 0; i <= maxit; ++i) bp.push_back(i < static_cast<int>(c.basis.size()) ? c.basis[i]->p : nullptr);
  CK(cudaMemcpyAsync(c.basis_ptrs.p, bp.data(), sizeof(void*) * bp.size(), cudaMemcpyHostToDevice, c.st));
  CK(cudaStreamSynchronize(c.st));

  c.hy_inner_its = 0;
  CK(cudaEventRecord(c.ev0, c.st));
  S* vin = c.vin.as<S>();
  Krylov<S>::permute_in(c.st, reinterpret_cast<const S*>(d_v), n, vin, ld, ncols, c.perm_d.as<int>());
  GmresDev g = gmres_view(c, maxit);
  g.nv = static_cast<int>(ncols);
  Krylov<S>::col_norms(c.st, vin, ld, ld, ncols, g.beta);
  S* v0 = reinterpret_cast<S*>(basis_block(c, 0));
  Krylov<S>::scale_cols(c.st, vin, v0, n, ld, ncols, g.beta);
  gmres_init(c.st, g);
  std::vector<double> beta(ncols);
  CK(cudaMemcpyAsync(beta.data(), g.beta, sizeof(double) * ncols, cudaMemcpyDeviceToHost, c.st));
  CK(cudaStreamSynchronize(c.st));
  std::vector<int> active;
  for (int64_t k = 0; k < ncols; ++k)
    if (beta[k] != 0.0) active.push_back(static_cast<int>(k));

  float trsm_ms = 0.0f, busy_ms = 0.0f;
  int trsm_launches = 0;
  int64_t launches = 4;
  int its = 0;
  // Lagged control: iterations are enqueued up to `lag` ahead of the convergence flags the host
  // has read -- the active list of iteration it+1 is the one known from iteration it-lag+... i.e.
  // filtered by the flags of iteration it+1-lag-1. Columns that converged in between are skipped
  // on the device (done flags: the Arnoldi / least-squares kernels return, the sweeps skip fully
  // converged column groups, an all-converged sweep exits at once), so the GPU does not wait for
  // host round trips and a short host stall is absorbed by the queued iterations. The hybrid
  // solve keeps the synchronous loop (its inner GMRES must not see finished columns).
  static const int lag_env = std::min(std::max(env_int("ZOLO_GMRES_LAG", 2), 0), 3);
  // refined solves: synchronous control, so that every G application can be judged on the
  // residuals of the iteration before (a host round trip is nothing beside a refined application)
  const int lag = (c.hybrid || c.refine) ? 0 : lag_env;
  const int nslot = lag + 1;
  struct LagGuard {
    zolo_ctx& c;
    ~LagGuard() {
      c.lag_done = nullptr;
      c.ev2_use = c.ev3_use = nullptr;
      c.in_filter = false;
      c.refine_skip = false;
    }
  } lag_guard{c};
  c.in_filter = true;
  c.lag_done = lag ? g.done : nullptr;
  cudaEvent_t ev_done[4], ev_t[4][2], ev_b[4][2];
  for (int p = 0; p < 4; ++p) {
    ev_done[p] = c.lag_ev[p];
    for (int q = 0; q < 2; ++q) ev_t[p][q] = c.lag_ev[4 + 2 * p + q], ev_b[p][q] = c.lag_ev[12 + 2 * p + q];
  }
  auto collect = [&](int p) {  // timings of a finished iteration in slot p
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, ev_t[p][0], ev_t[p][1]));
    trsm_ms += ms;
    CK(cudaEventElapsedTime(&ms, ev_b[p][0], ev_b[p][1]));
    busy_ms += ms;
  };
  auto check_spin = [&] {
    int spin_err[2] = {0, 0};
    CK(cudaMemcpyAsync(spin_err, c.counter.as<int>() + 2, sizeof(int) * 2, cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    if (spin_err[0] || spin_err[1]) throw ZoloError(ZOLO_ERR_CUDA, "triangular solve: dependency wait timed out");
  };
  auto filter_active = [&](const int* dn) {
    std::vector<int> next;
    for (int col : active)
      if (!dn[col]) next.push_back(col);
    active.swap(next);
  };
  std::vector<double> res_h;
  const int q2 = 2 * c.r;
  int nskipped = 0;  // G applications that ran unrefined under the relaxed-refinement rule
  c.refine_skip = false;
  c.refine_skipped = 0;
  int pend[4], npend = 0;  // slots enqueued whose flags are not yet read, oldest first
  for (int it = 0; it < maxit && !active.empty(); ++it) {
    its = it + 1;
    const int p = it % nslot;  // its previous user (iteration it - nslot) has been read
    const int na = static_cast<int>(active.size());
    std::memcpy(c.act_hq[p], active.data(), sizeof(int) * na);
    CK(cudaMemcpyAsync(c.act_d.p, c.act_hq[p], sizeof(int) * na, cudaMemcpyHostToDevice, c.st));
    S* vm = reinterpret_cast<S*>(basis_block(c, it));
    CK(cudaEventRecord(ev_b[p][0], c.st));
    c.ev2_use = ev_t[p][0];
    c.ev3_use = ev_t[p][1];
    apply_g_device(c, vm, na, c.w.p);
    trsm_launches += 2;
    launches += 8 + (it + 1 < maxit ? 1 : 0);
    nvtxRangePushA("zolo::arnoldi");
    const int nls = Krylov<S>::arnoldi(c.st, row_lo(c), row_hi(c), ld, c.basis_ptrs.as<S*>(), it, c.w.as<S>(),
                                       c.act_d.as<int>(), na, g, c.partial.as<double>(), c.hsave.as<S>(),
                                       c.row_shard ? c.coll : nullptr);
    Krylov<S>::least_squares(c.st, c.act_d.as<int>(), na, it, g, c.partial.as<double>(), nls, tol);
    nvtxRangePop();
    if (it + 1 < maxit) {
      S* vn = reinterpret_cast<S*>(basis_block(c, it + 1));
      Krylov<S>::next_basis(c.st, n, ld, c.w.as<S>(), vn, c.act_d.as<int>(), na, g);
      if (c.row_shard) {  // every rank's poles need all rows of the next basis vector
        const int64_t r0 = row_lo(c), rows = row_hi(c) - r0, rb = c.rb;
        c.vpack.ensure(c.es() * rb * std::max(na, 1));
        c.vgath.ensure(c.es() * rb * c.shard_size * std::max(na, 1));
        CK(cudaMemsetAsync(c.vpack.p, 0, c.es() * rb * na, c.st));  // the last block's padding rows
        Krylov<S>::pack_rows(c.st, vn, ld, r0, rows, rb, c.act_d.as<int>(), na, c.vpack.as<S>());
        c.coll->allgather(c.vpack.as<double>(), c.vgath.as<double>(), static_cast<size_t>(rb) * na * (c.es() / 8),
                          c.st);
        Krylov<S>::unpack_blocks(c.st, c.vgath.as<S>(), rb, c.shard_size, c.act_d.as<int>(), na, vn, ld);
      }
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(ev_b[p][1], c.st));
    CK(cudaMemcpyAsync(c.done_hq[p], g.done, sizeof(int) * ncols, cudaMemcpyDeviceToHost, c.st));
    CK(cudaEventRecord(ev_done[p], c.st));
    pend[npend++] = p;
    if (npend > lag) {  // the oldest pending iteration's flags: filter the next active list
      const int q = pend[0];
      for (int k = 1; k < npend; ++k) pend[k - 1] = pend[k];
      --npend;
      CK(cudaEventSynchronize(ev_done[q]));
      if (!lag) check_spin();
      collect(q);
      filter_active(c.done_hq[q]);
      if (c.refine && !active.empty()) {
        // Relaxed refinement (inexact Krylov: the later a G application, the less exact it must
        // be): with relative GMRES residuals rho after this iteration, an unrefined application
        // perturbs the solutions by ~rho x (residual of the unrefined solves) -- skip the
        // correction once that is a tenth of the GMRES tolerance.
        res_h.resize(static_cast<size_t>(ncols) * q2);
        CK(cudaMemcpyAsync(res_h.data(), g.res, sizeof(double) * res_h.size(), cudaMemcpyDeviceToHost, c.st));
        CK(cudaStreamSynchronize(c.st));
        double rho = 0.0;
        for (int col : active)
          for (int k = 0; k < q2; ++k) rho = std::max(rho, res_h[static_cast<size_t>(col) * q2 + k]);
        c.refine_skip = c.refine_relax && c.unrefined_res >= 0.0 && std::isfinite(rho) &&
                        10.0 * rho * c.unrefined_res <= tol;
        nskipped += c.refine_skip ? 1 : 0;
        c.refine_skipped = nskipped;
      }
    }
  }
  c.refine_skip = false;
  for (int k = 0; k < npend; ++k) {
    CK(cudaEventSynchronize(ev_done[pend[k]]));
    collect(pend[k]);
  }
  check_spin();
  c.ev2_use = nullptr;
  c.ev3_use = nullptr;
  c.iters_seen = std::max(c.iters_seen, its);
  S* yp = c.vout.as<S>();
  Krylov<S>::assemble(c.st, n, ld, v0, c.basis_ptrs.as<S*>(), static_cast<int>(ncols), g, vin, yp);
  Krylov<S>::permute_out(c.st, yp, ld, reinterpret_cast<S*>(d_y), n, ncols, c.perm_d.as<int>());
  CK(cudaEventRecord(c.ev1, c.st));
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c.st));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, c.ev0, c.ev1));
  c.last_ms[0] = ms;
  c.last_ms[2] = trsm_ms;
  c.last_ms[3] = trsm_launches;
  c.last_ms[4] = static_cast<double>(launches + 2);
  c.last_ms[6] = static_cast<double>(c.hy_inner_its);  // hybrid: inner K_p applications (column-steps)
  c.last_ms[7] = busy_ms;  // device time of the GMRES iterations (the rest of [0]: prologue, epilogue, host gaps)

  // report (gmres.hpp:31-43 merged as filter_engine.hpp:127-133)
  std::vector<double> res(ncols * q);
  std::vector<int> mcol(ncols), happy(ncols);
  // (on the context stream: the legacy default stream does not order with it)
  CK(cudaMemcpyAsync(res.data(), g.res, sizeof(double) * ncols * q, cudaMemcpyDeviceToHost, c.st));
  CK(cudaMemcpyAsync(mcol.data(), g.mcol, sizeof(int) * ncols, cudaMemcpyDeviceToHost, c.st));
  CK(cudaMemcpyAsync(happy.data(), g.happy, sizeof(int) * ncols, cudaMemcpyDeviceToHost, c.st));
  CK(cudaStreamSynchronize(c.st));
  bool all_conv = true;
  if (rep) {
    rep->iterations = 0;
    rep->operator_applications = 0;
    rep->n_shifts = q;
    for (int k = 0; k < q; ++k) {
      rep->residuals[k] = 0.0;
      rep->converged[k] = 1;
    }
  }
  int64_t opapps = 0;  // G applications = sum of the columns' Krylov dimensions (gmres.hpp:31-43)
  for (int64_t col = 0; col < ncols; ++col) opapps += mcol[col];
  c.g_apps += opapps;
  c.inner_solves += static_cast<int64_t>(c.nchains()) * opapps;
  c.last_ms[5] = static_cast<double>(opapps);
  for (int64_t col = 0; col < ncols; ++col) {
    for (int k = 0; k < q; ++k) {
      const double rk = res[col * q + k];
      if (rep) rep->residuals[k] = std::max(rep->residuals[k], rk);
      if (!(rk <= tol) && !happy[col] && beta[col] != 0.0) {
        all_conv = false;
        if (rep) rep->converged[k] = 0;
      }
    }
    if (rep) {
      rep->iterations = std::max<int64_t>(rep->iterations, mcol[col]);
      rep->operator_applications += mcol[col];
      if (rep->column_iterations) rep->column_iterations[col] = mcol[col];
    }
  }
  if (rep) rep->all_converged = all_conv ? 1 : 0;
  if (!all_conv) {
    c.err = "multishift_gmres: not converged within " + std::to_string(maxit) + " iterations";
    return ZOLO_ERR_GMRES;
  }
  return ZOLO_OK;
}

template <class S>
void apply_g_impl(zolo_ctx& c, const double* v, double* gv, int64_t k) {
  require(c.factored, "apply_g: operator not factorized");
  const int64_t n = c.n, ld = c.geom.npad;
  ensure_workspace(c, k);
  CK(cudaMemcpyAsync(c.vin_orig.p, v, c.es() * n * k, cudaMemcpyHostToDevice, c.st));
  Krylov<S>::permute_in(c.st, c.vin_orig.as<S>(), n, c.vin.as<S>(), ld, k, c.perm_d.as<int>());
  for (int64_t i = 0; i < k; ++i) c.act_h[i] = static_cast<int>(i);
  CK(cudaMemcpyAsync(c.act_d.p, c.act_h, sizeof(int) * k, cudaMemcpyHostToDevice, c.st));
  apply_g_device(c, c.vin.p, static_cast<int>(k), c.w.p);
  Krylov<S>::permute_out(c.st, c.w.as<S>(), ld, c.vin_orig.as<S>(), n, k, c.perm_d.as<int>());
  CK(cudaMemcpyAsync(gv, c.vin_orig.p, c.es() * n * k, cudaMemcpyDeviceToHost, c.st));
  CK(cudaStreamSynchronize(c.st));
  if (!c.hybrid) {  // sweep time of this application (last_timings trsm_ms)
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, c.ev2, c.ev3));
    c.last_ms[2] = ms;
  }
  // filter_engine.hpp:58,70,79: one application per call, r or 2r solves
  c.g_apps += 1;
  c.inner_solves += c.nchains();
}

template <class S>
void rr_impl(zolo_ctx& c, const double* y, int64_t k, double* at, double* bt) {
  Nvtx range("zolo::rr_project");
  ensure_perm_csr(c);
  const int64_t n = c.n, ld = c.geom.npad;
  const size_t es = sizeof(S);
  DevMem yo, yp, ay;
  yo.ensure(es * n * k);
  yp.ensure(es * ld * k);
  ay.ensure(es * ld * k);
  const int64_t nchunk = (ld + CHUNK - 1) / CHUNK;
  c.rr_partial.ensure(es * nchunk * k * k + 64);
  c.rr_out.ensure(es * k * k);
  CK(cudaMemcpyAsync(yo.p, y, es * n * k, cudaMemcpyHostToDevice, c.st));
  Krylov<S>::permute_in(c.st, yo.as<S>(), n, yp.as<S>(), ld, k, c.perm_d.as<int>());
  device_spmm<S>(c, 0, yp.as<S>(), k, ay.as<S>());
  Krylov<S>::gram(c.st, ld, ld, yp.as<S>(), k, ay.as<S>(), k, c.rr_out.as<S>(), c.rr_partial.as<double>());
  CK(cudaMemcpyAsync(at, c.rr_out.p, es * k * k, cudaMemcpyDeviceToHost, c.st));
  CK(cudaStreamSynchronize(c.st));
  if (c.b_identity) {
    Krylov<S>::gram(c.st, ld, ld, yp.as<S>(), k, yp.as<S>(), k, c.rr_out.as<S>(), c.rr_partial.as<double>());
  } else {
    device_spmm<S>(c, 1, yp.as<S>(), k, ay.as<S>());
    Krylov<S>::gram(c.st, ld, ld, yp.as<S>(), k, ay.as<S>(), k, c.rr_out.as<S>(), c.rr_partial.as<double>());
  }
  CK(cudaMemcpyAsync(bt, c.rr_out.p, es * k * k, cudaMemcpyDeviceToHost, c.st));
  CK(cudaStreamSynchronize(c.st));
  CK(cudaGetLastError());
}

template <class S>
void block_update_impl(zolo_ctx& c, const double* y, int64_t k, const double* q, int64_t kk, double* out) {
  const int64_t n = c.n;
  const size_t es = sizeof(S);
  DevMem yd, qd, od;
  yd.ensure(es * n * k);
  qd.ensure(es * k * kk);
  od.ensure(es * n * kk);
  CK(cudaMemcpyAsync(yd.p, y, es * n * k, cudaMemcpyHostToDevice, c.st));
  CK(cudaMemcpyAsync(qd.p, q, es * k * kk, cudaMemcpyHostToDevice, c.st));
  Krylov<S>::block_gemm(c.st, n, n, yd.as<S>(), k, qd.as<S>(), kk, od.as<S>());
  CK(cudaMemcpyAsync(out, od.p, es * n * kk, cudaMemcpyDeviceToHost, c.st));
  CK(cudaStreamSynchronize(c.st));
  CK(cudaGetLastError());
}

// ---- device-block helpers for the host driver (original ordering, ld = n) ----
template <class S>
void spmm_dev_impl(zolo_ctx& c, int which, const void* x, void* out, int64_t k) {
  ensure_perm_csr(c);
  const int64_t n = c.n, ld = c.geom.npad;
  const size_t es = sizeof(S);
  if (which == 1 && c.b_identity) {
    CK(cudaMemcpyAsync(out, x, es * n * k, cudaMemcpyDeviceToDevice, c.st));
  } else {
    c.tmp1.ensure(es * ld * k);
    c.tmp2.ensure(es * ld * k);
    Krylov<S>::permute_in(c.st, reinterpret_cast<const S*>(x), n, c.tmp1.as<S>(), ld, k, c.perm_d.as<int>());
    device_spmm<S>(c, which, c.tmp1.as<S>(), k, c.tmp2.as<S>());
    Krylov<S>::permute_out(c.st, c.tmp2.as<S>(), ld, reinterpret_cast<S*>(out), n, k, c.perm_d.as<int>());
  }
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c.st));  // like its siblings: d_out is complete when the call returns
}

template <class S>
void gram_dev_impl(zolo_ctx& c, const void* y, const void* z, int64_t k, int64_t kk, double* out) {
  Nvtx range("zolo::gram");
  const int64_t n = c.n;
  const int64_t nchunk = (n + CHUNK - 1) / CHUNK;
  c.rr_partial.ensure(sizeof(S) * nchunk * k * kk + 64);
  c.rr_out.ensure(sizeof(S) * k * kk);
  Krylov<S>::gram(c.st, n, n, reinterpret_cast<const S*>(y), k, reinterpret_cast<const S*>(z), kk, c.rr_out.as<S>(),
                  c.rr_partial.as<double>());
  CK(cudaMemcpyAsync(out, c.rr_out.p, sizeof(S) * k * kk, cudaMemcpyDeviceToHost, c.st));
  CK(cudaStreamSynchronize(c.st));
  CK(cudaGetLastError());
}

template <class S>
void gemm_dev_impl(zolo_ctx& c, const void* y, int64_t k, const double* q, int64_t kk, void* out) {
  c.tmp3.ensure(sizeof(S) * k * kk);
  CK(cudaMemcpyAsync(c.tmp3.p, q, sizeof(S) * k * kk, cudaMemcpyHostToDevice, c.st));
  Krylov<S>::block_gemm(c.st, c.n, c.n, reinterpret_cast<const S*>(y), k, c.tmp3.as<S>(), kk,
                        reinterpret_cast<S*>(out));
  CK(cudaStreamSynchronize(c.st));
  CK(cudaGetLastError());
}

template <class S>
void resid_dev_impl(zolo_ctx& c, const void* ax, const void* bx, int64_t k, const double* lam, double* num,
                    double* den) {
  c.tmp3.ensure(sizeof(double) * 3 * k + 64);
  double* d = c.tmp3.as<double>();
  CK(cudaMemcpyAsync(d, lam, sizeof(double) * k, cudaMemcpyHostToDevice, c.st));
  Krylov<S>::residuals(c.st, c.n, reinterpret_cast<const S*>(ax), reinterpret_cast<const S*>(bx), d, k, d + k,
                       d + 2 * k);
  CK(cudaMemcpyAsync(num, d + k, sizeof(double) * k, cudaMemcpyDeviceToHost, c.st));
  CK(cudaMemcpyAsync(den, d + 2 * k, sizeof(double) * k, cudaMemcpyDeviceToHost, c.st));
  CK(cudaStreamSynchronize(c.st));
  CK(cudaGetLastError());
}

}  // namespace

namespace zolo {
cudaStream_t ctx_stream(const zolo_ctx* c) { return c ? c->st : nullptr; }
}  // namespace zolo

extern "C" {

const char* zolo_version(void) { return "zolo-b200 0.1.0 (sm_100a)"; }

int zolo_spmm_device(zolo_ctx* c, int which, const void* d_x, void* d_out, int64_t k) {
  return guarded(c, [&] {
    require(c->have_pencil, "spmm: no pencil");
    require(which == 0 || which == 1, "spmm: which must be 0 (A) or 1 (B)");
    if (k <= 0) return;
    if (c->cx)
      spmm_dev_impl<cd>(*c, which, d_x, d_out, k);
    else
      spmm_dev_impl<double>(*c, which, d_x, d_out, k);
  });
}

int zolo_gram_device(zolo_ctx* c, const void* d_y, const void* d_z, int64_t k, int64_t kk, double* out) {
  return guarded(c, [&] {
    require(c->have_pencil, "gram: no pencil");
    if (k <= 0 || kk <= 0) return;
    if (c->cx)
      gram_dev_impl<cd>(*c, d_y, d_z, k, kk, out);
    else
      gram_dev_impl<double>(*c, d_y, d_z, k, kk, out);
  });
}

int zolo_block_gemm_device(zolo_ctx* c, const void* d_y, int64_t k, const double* q, int64_t kk, void* d_out) {
  return guarded(c, [&] {
    require(c->have_pencil, "block_gemm: no pencil");
    if (kk <= 0) return;
    if (c->cx)
      gemm_dev_impl<cd>(*c, d_y, k, q, kk, d_out);
    else
      gemm_dev_impl<double>(*c, d_y, k, q, kk, d_out);
  });
}

int zolo_residual_norms_device(zolo_ctx* c, const void* d_ax, const void* d_bx, int64_t k, const double* lambdas,
                               double* num, double* den) {
  return guarded(c, [&] {
    require(c->have_pencil, "residuals: no pencil");
    if (k <= 0) return;
    if (c->cx)
      resid_dev_impl<cd>(*c, d_ax, d_bx, k, lambdas, num, den);
    else
      resid_dev_impl<double>(*c, d_ax, d_bx, k, lambdas, num, den);
  });
}

int zolo_ctx_create(int device, zolo_ctx** out) {
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    g_create_err = std::string("no CUDA device: ") + cudaGetErrorString(e);
    return ZOLO_ERR_CUDA;
  }
  if (device < 0 || device >= ndev) {
    g_create_err = "device index out of range";
    return ZOLO_ERR_DOMAIN;
  }
  auto* c = new zolo_ctx();
  c->device = device;
  const int st = guarded(c, [&] {
    CK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    CK(cudaEventCreate(&c->ev0));
    CK(cudaEventCreate(&c->ev1));
    CK(cudaEventCreate(&c->ev2));
    CK(cudaEventCreate(&c->ev3));
    CK(cudaEventCreate(&c->ev4));
    CK(cudaEventCreate(&c->ev5));
    for (auto& e : c->lag_ev) CK(cudaEventCreate(&e));  // 4 slots x (done copy, sweep pair, busy pair)
  });
  if (st != ZOLO_OK) {
    g_create_err = c->err;
    delete c;
    return st;
  }
  *out = c;
  return ZOLO_OK;
}

int zolo_ctx_destroy(zolo_ctx* c) {
  if (!c) return ZOLO_OK;
  DeviceScope scope(c);  // the context's device; the caller's is restored on return
  if (c->st) cudaStreamSynchronize(c->st);
  for (auto s : c->pole_streams) cudaStreamDestroy(s);
  delete c->coll;
  if (c->act_h) cudaFreeHost(c->act_h);
  for (int q = 0; q < 4; ++q) {
    if (c->act_hq[q]) cudaFreeHost(c->act_hq[q]);
    if (c->done_hq[q]) cudaFreeHost(c->done_hq[q]);
  }
  if (c->act_in_h) cudaFreeHost(c->act_in_h);
  if (c->done_h) cudaFreeHost(c->done_h);
  for (cudaEvent_t ev : {c->ev0, c->ev1, c->ev2, c->ev3, c->ev4, c->ev5, c->tev0, c->tev1})
    if (ev) cudaEventDestroy(ev);
  for (cudaEvent_t ev : c->lag_ev)
    if (ev) cudaEventDestroy(ev);
  cudaStream_t st = c->st;
  delete c;
  if (st) cudaStreamDestroy(st);
  return ZOLO_OK;
}

const char* zolo_last_error(const zolo_ctx* c) { return c ? c->err.c_str() : g_create_err.c_str(); }

void zolo_set_error(zolo_ctx* c, const char* msg) {
  if (c)
    c->err = msg;
  else
    g_create_err = msg;
}

int zolo_pencil_upload(zolo_ctx* c, int64_t n, int scalar, const int64_t* a_rp, const int64_t* a_ci,
                       const double* a_v, const int64_t* b_rp, const int64_t* b_ci, const double* b_v) {
  return guarded(c, [&] {
    require(n > 0, "zolo_pencil_upload: n must be positive");
    require(n < (int64_t(1) << 31) - TILE, "zolo_pencil_upload: n exceeds int32 indexing");
    require(scalar == ZOLO_F64 || scalar == ZOLO_C128, "zolo_pencil_upload: bad scalar tag");
    require(a_rp && a_ci && a_v, "zolo_pencil_upload: A missing");
    c->n = n;
    c->cx = scalar;
    const int w = scalar ? 2 : 1;
    c->b_identity = b_rp == nullptr;
    {  // the host copies of the pencil's arrays, side by side (dense-block pencils: hundreds of MB)
      std::exception_ptr cerr[4];
      std::vector<std::thread> cp;
      auto copy_on_thread = [&](int slot, auto&& fn) {
        cp.emplace_back([&cerr, slot, fn] {
          try {
            fn();
          } catch (...) {
            cerr[slot] = std::current_exception();
          }
        });
      };
      copy_on_thread(0, [&] { c->a_ci.assign(a_ci, a_ci + a_rp[n]); });
      copy_on_thread(1, [&] { c->a_v.assign(a_v, a_v + a_rp[n] * w); });
      if (!c->b_identity) {
        copy_on_thread(2, [&] { c->b_ci.assign(b_ci, b_ci + b_rp[n]); });
        copy_on_thread(3, [&] { c->b_v.assign(b_v, b_v + b_rp[n] * w); });
      }
      try {
        c->a_rp.assign(a_rp, a_rp + n + 1);
        if (!c->b_identity) c->b_rp.assign(b_rp, b_rp + n + 1);
      } catch (...) {
        for (auto& t : cp) t.join();
        throw;
      }
      for (auto& t : cp) t.join();
      for (auto& e : cerr)
        if (e) std::rethrow_exception(e);
    }
    if (c->b_identity) {
      c->b_rp.clear();
      c->b_ci.clear();
      c->b_v.clear();
    }
    // (the message strings are built only on failure: this loop visits every entry)
    const auto sorted_in_range = [n](const std::vector<int64_t>& rp, const std::vector<int64_t>& ci, int64_t i) {
      bool ok = true;
      for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
        ok = ok && ci[k] >= 0 && ci[k] < n && (k == rp[i] || ci[k] > ci[k - 1]);
      return ok;
    };
    par_rows(n, [&](int64_t lo, int64_t hi) {
      for (int64_t i = lo; i < hi; ++i) {
        if (c->a_rp[i] > c->a_rp[i + 1]) require(false, "zolo_pencil_upload: A offsets not monotone");
        if (!sorted_in_range(c->a_rp, c->a_ci, i))
          require(false, "zolo_pencil_upload: A column indices must be in range and sorted");
        if (!c->b_identity && !sorted_in_range(c->b_rp, c->b_ci, i))
          require(false, "zolo_pencil_upload: B column indices must be in range and sorted");
      }
    });
    c->have_pencil = true;
    c->have_perm = false;
    c->sym_ready = false;
    c->factored = false;
    c->ncap = 0;
  });
}

int zolo_set_design(zolo_ctx* c, const double* design, int r) {
  return guarded(c, [&] {
    require(r >= 1 && r <= ZOLO_MAX_ORDER, "zolo_set_design: order must be in [1,16]");
    c->design.assign(design, design + ZOLO_DESIGN_LEN(r));
    c->r = r;
    const double m_hat = design[ZOLO_DESIGN_M_HAT];
    const double* wts = design + ZOLO_DESIGN_HEAD + 2 * r;
    const double* opf = design + ZOLO_DESIGN_HEAD + 5 * r;
    const double* oc = design + ZOLO_DESIGN_HEAD + 6 * r + (2 * r - 1);
    const double mo = design[ZOLO_DESIGN_OUTER_M];
    c->eff_w.clear();
    c->shifts.clear();
    c->coef.clear();
    for (int j = 0; j < r; ++j) {
      c->eff_w.push_back(m_hat * std::complex<double>(wts[2 * j], wts[2 * j + 1]));  // filter_engine.hpp:43-44
      const double root = std::sqrt(oc[2 * j]);                                      // filter_engine.hpp:90-96
      c->shifts.emplace_back(0.0, root);
      c->shifts.emplace_back(0.0, -root);
      const double cf = (0.5 * mo) * (0.5 * opf[j]);  // filter_engine.hpp:112-121
      c->coef.push_back(cf);
      c->coef.push_back(cf);
    }
    for (size_t a = 0; a < c->shifts.size(); ++a)
      for (size_t b = a + 1; b < c->shifts.size(); ++b)
        require(c->shifts[a] != c->shifts[b], "multishift_gmres: shifts must be distinct");
    c->constant_term = design[ZOLO_DESIGN_CONSTANT];
    std::vector<cd> s(2 * r);
    for (int k = 0; k < 2 * r; ++k) s[k] = mk(c->shifts[k].real(), c->shifts[k].imag());
    refresh_own(*c);
    upload(c->shifts_d, s, c->st);
    upload(c->coef_d, c->coef, c->st);
    c->have_design = true;
    c->factored = false;
  });
}

int zolo_set_block_size(zolo_ctx* c, int64_t block) {
  return guarded(c, [&] {
    require(block >= 1 && block <= 64, "zolo_set_block_size: block must be in [1, 64]");
    require(!c->have_pencil || c->n % block == 0, "zolo_set_block_size: the order is not a multiple of the block");
    c->bsr = block;
    c->have_perm = false;
    c->sym_ready = false;
    c->factored = false;
  });
}

int zolo_bsr_info(const zolo_ctx* c, int64_t* out) {
  out[0] = c->bsr;
  out[1] = c->bsr_dev ? c->bsr_na : 0;
  return ZOLO_OK;
}

int zolo_set_ordering(zolo_ctx* c, int mode, int64_t nd_leaf) {
  return guarded(c, [&] {
    require(mode == ZOLO_ORDER_ND || mode == ZOLO_ORDER_RCM, "zolo_set_ordering: unknown mode");
    c->order_mode = mode;
    if (nd_leaf > 0) c->nd_leaf = nd_leaf;
    c->factored = false;
  });
}

int zolo_factorize(zolo_ctx* c, const int64_t* perm, zolo_factor_stats* stats) {
  return guarded(c, [&] {
    require(c->have_design, "zolo_factorize: no design set");
    require(c->nloc() >= 1, "zolo_factorize: pole shard owns no pole (need r >= nranks)");
    do_factorize(*c, perm, stats);
  });
}

int zolo_count_below(zolo_ctx* c, double sigma, int64_t* count, double* min_pivot_ratio) {
  return guarded(c, [&] {
    require(c->have_pencil, "zolo_count_below: no pencil uploaded");
    require(c->order_mode == ZOLO_ORDER_ND, "zolo_count_below: needs the ND (block-sparse) ordering");
    require(std::isfinite(sigma), "zolo_count_below: sigma must be finite");
    if (!c->sym_ready) sparse_symbolic(*c, nullptr);
    DevMem store;
    std::vector<FactorTiles> tiles;
    std::vector<cd*> dt;
    std::vector<int> fail;
    std::vector<double> mr;
    sparse_numeric(*c, {std::complex<double>(sigma, 0.0)}, store, nullptr, tiles, dt, fail, mr, nullptr);
    if (min_pivot_ratio) *min_pivot_ratio = mr[0];
    if (fail[0] >= 0)
      throw ZoloError(ZOLO_ERR_FACTORIZATION, "zolo_count_below: pivot " + std::to_string(fail[0]) +
                                                  " below threshold (sigma too close to an eigenvalue)");
    *count = count_negative_pivots(c->st, dt[0], c->sgeom.nb);
  });
}

int zolo_set_solve_mode(zolo_ctx* c, int mode, int pole, double inner_tol, int inner_max) {
  return guarded(c, [&] {
    require(mode == ZOLO_SOLVE_DIRECT || mode == ZOLO_SOLVE_HYBRID, "zolo_set_solve_mode: unknown mode");
    require(c->have_design, "zolo_set_solve_mode: set the design first");
    require(mode == ZOLO_SOLVE_DIRECT || c->refine == 0, "zolo_set_solve_mode: the hybrid solve has no refinement");
    if (mode == ZOLO_SOLVE_HYBRID) {
      require(pole >= 0 && pole < c->r, "zolo_set_solve_mode: factored pole out of range");
      require(c->order_mode == ZOLO_ORDER_ND, "zolo_set_solve_mode: the hybrid solve needs the ND ordering");
      require(c->shard_size == 1, "zolo_set_solve_mode: hybrid solve and pole sharding are exclusive");
      require(inner_tol > 0.0 && inner_max >= 1 && inner_max <= 256, "zolo_set_solve_mode: bad inner limits");
      c->hy_pole = pole;
      c->hy_tol = inner_tol;
      c->hy_max = inner_max;
    }
    c->hybrid = mode == ZOLO_SOLVE_HYBRID;
    refresh_own(*c);
    if (c->hybrid) hybrid_setup(*c);
  });
}

int zolo_set_refinement_relaxation(zolo_ctx* c, int on) {
  if (!c) return ZOLO_ERR_DOMAIN;
  c->refine_relax = on != 0;
  return ZOLO_OK;
}

int zolo_refinement_stats(const zolo_ctx* c, double* out) {
  if (!c || !out) return ZOLO_ERR_DOMAIN;
  out[0] = c->unrefined_res;
  out[1] = static_cast<double>(c->refine_skipped);
  return ZOLO_OK;
}

int zolo_set_refinement(zolo_ctx* c, int steps) {
  return guarded(c, [&] {
    require(steps >= 0 && steps <= 2, "zolo_set_refinement: steps must be in [0, 2]");
    require(steps == 0 || !c->hybrid, "zolo_set_refinement: not available with the hybrid solve");
    if (steps != c->refine) {
      c->unrefined_res = -1.0;
      c->refine = steps;
      c->ncap = 0;  // the workspace (residual blocks, refinement chains) is rebuilt
    }
  });
}

int zolo_pool_trim(int device) {
  int saved = -1;
  cudaGetDevice(&saved);
  if (cudaSetDevice(device) != cudaSuccess) return ZOLO_ERR_CUDA;
  pool_trim(device);
  if (saved >= 0) cudaSetDevice(saved);
  return ZOLO_OK;
}

int zolo_nccl_unique_id(void* out) {
  try {
    nccl_unique_id(out);
    return ZOLO_OK;
  } catch (const std::exception& e) {
    g_create_err = e.what();
    return ZOLO_ERR_CUDA;
  }
}

namespace {
void set_shard(zolo_ctx& c, int rank, int nranks, Collective* coll) {
  require(nranks >= 1 && rank >= 0 && rank < nranks, "zolo_set_pole_shard: need 0 <= rank < nranks");
  require(!c.hybrid || nranks == 1, "zolo_set_pole_shard: hybrid solve and pole sharding are exclusive");
  delete c.coll;
  c.coll = coll;
  c.shard_rank = rank;
  c.shard_size = nranks;
  static const bool rows = env_int("ZOLO_ROW_SHARD", 1) != 0;
  c.row_shard = coll && nranks > 1 && rows;
  c.ncap = 0;
  if (c.have_design) refresh_own(c);
}
}  // namespace

int zolo_set_pole_shard(zolo_ctx* c, int rank, int nranks, const void* unique_id) {
  return guarded(c, [&] {
    // a 1-rank communicator is legal: its all-reduce is the identity, which lets one GPU run the
    // in-library NCCL path end to end
    Collective* coll = nullptr;
    if (unique_id) {
      try {
        coll = nccl_collective(unique_id, nranks, rank);
      } catch (const std::exception& e) {
        throw ZoloError(ZOLO_ERR_CUDA, e.what());
      }
    }
    set_shard(*c, rank, nranks, coll);
  });
}

int zolo_set_pole_shard_host(zolo_ctx* c, int rank, int nranks, zolo_collective_fn fn, void* user) {
  return guarded(c, [&] {
    require(fn != nullptr, "zolo_set_pole_shard_host: callback missing");
    set_shard(*c, rank, nranks, host_collective(fn, user, nranks, rank));
  });
}

int zolo_filter_create(zolo_ctx* c, int64_t n, int scalar, const int64_t* a_rp, const int64_t* a_ci,
                       const double* a_v, const int64_t* b_rp, const int64_t* b_ci, const double* b_v,
                       const double* design, int r, zolo_factor_stats* stats) {
  SetupClock clk;
  int st = zolo_pencil_upload(c, n, scalar, a_rp, a_ci, a_v, b_rp, b_ci, b_v);
  if (st) return st;
  clk.mark("pencil_upload");
  st = zolo_set_design(c, design, r);
  if (st) return st;
  st = zolo_factorize(c, nullptr, stats);
  clk.mark("factorize (total)");
  return st;
}

int zolo_shifted_solve(zolo_ctx* c, int pole, int adjoint, const double* b, double* x, int64_t ncols) {
  return guarded(c, [&] {
    Nvtx range("zolo::shifted_solve");
    require(c->factored, "shifted_solve: operator not factorized");
    require(!c->hybrid, "shifted_solve: the hybrid solve factors one pole only");
    require(ncols >= 1, "shifted_solve: empty block");
    int p = -1;
    for (int q = 0; q < c->nloc(); ++q)
      if (c->own[q] == pole) p = q;
    require(p >= 0, "shifted_solve: pole not factored by this context");
    zolo_ctx& C = *c;
    const int64_t n = C.n, ld = C.geom.npad;
    ensure_workspace(C, ncols);
    // ShiftedFactor::solve / adjoint_solve (band_factor.hpp:53-117): complex n x ncols blocks. For a
    // real pencil K = A - sigma B is complex symmetric, so K^-H b = conj(K^-1 conj(b)).
    const bool conj_trick = adjoint && !C.cx;
    const int ch = C.cx ? 2 * p + (adjoint ? 1 : 0) : p;
    C.tmp1.ensure(sizeof(cd) * n * ncols);  // complex staging (vin_orig holds S = double for real pencils)
    CK(cudaMemcpyAsync(C.tmp1.p, b, sizeof(cd) * n * ncols, cudaMemcpyHostToDevice, C.st));
    if (conj_trick) conj_inplace(C.st, C.tmp1.as<cd>(), n * ncols);
    Krylov<cd>::permute_in(C.st, C.tmp1.as<cd>(), n, C.bbuf.as<cd>(), ld, ncols, C.perm_d.as<int>());
    for (int64_t i = 0; i < ncols; ++i) C.act_h[i] = static_cast<int>(i);
    CK(cudaMemcpyAsync(C.act_d.p, C.act_h, sizeof(int) * ncols, cudaMemcpyHostToDevice, C.st));
    sweep_sparse(C, ch, 1, static_cast<int>(ncols));
    if (C.refine) refine_solves(C, static_cast<int>(ncols), ch, 1);
    Krylov<cd>::permute_out(C.st, C.xbuf[ch]->as<cd>(), ld, C.tmp1.as<cd>(), n, ncols, C.perm_d.as<int>());
    if (conj_trick) conj_inplace(C.st, C.tmp1.as<cd>(), n * ncols);
    CK(cudaMemcpyAsync(x, C.tmp1.p, sizeof(cd) * n * ncols, cudaMemcpyDeviceToHost, C.st));
    CK(cudaStreamSynchronize(C.st));
    CK(cudaGetLastError());
    C.inner_solves += ncols;  // one shifted solve per right-hand side (band_factor.hpp:53-85 per column)
  });
}

int zolo_apply_g(zolo_ctx* c, const double* v, double* gv, int64_t ncols) {
  return guarded(c, [&] {
    require(ncols >= 1, "apply_g: empty block");
    if (c->cx)
      apply_g_impl<cd>(*c, v, gv, ncols);
    else
      apply_g_impl<double>(*c, v, gv, ncols);
  });
}

}  // extern "C"

namespace {

// Device bytes of the per-column workspace (vectors, Krylov basis, GMRES state) of one column.
double bytes_per_column(zolo_ctx& c, int maxit) {
  const double ld = static_cast<double>(c.geom.npad), es = static_cast<double>(c.es());
  const int nch = c.nchains(), q = 2 * c.r;
  const double crows = static_cast<double>(TILE) * std::max(c.sp_nslots, 1);
  const double nchunk = std::ceil(ld / CHUNK);
  double b = c.n * es + ld * (3 * es + 16 + 16.0 * nch + es * (maxit + 2)) + 16.0 * nch * crows;
  b += es * (maxit + 1) * maxit + 16.0 * q * (maxit * maxit + 4.0 * maxit + 1) + 3 * es * nchunk * (maxit + 1);
  if (c.row_shard) b += 3.0 * es * ld;  // blocked partial G, the local block, the gathered basis block
  if (c.hybrid) b += 16.0 * ld * (c.hy_max + 4) + 16.0 * (c.r - 1) * c.hy_max * c.hy_max;
  if (c.refine) b += 16.0 * nch * ld;
  return b;
}

void release_workspace(zolo_ctx& c) {
  for (DevMem* m : {&c.vin_orig, &c.vin, &c.vout, &c.w, &c.bbuf, &c.gH, &c.gR, &c.gG, &c.gROT, &c.gY, &c.gZ,
                    &c.partial, &c.hsave, &c.wc, &c.wloc, &c.vpack, &c.vgath, &c.hy_w, &c.iH, &c.iR, &c.iG, &c.iROT, &c.iY, &c.iZ, &c.ipartial,
                    &c.ihsave})
    m->release();
  for (auto& m : c.xbuf) m->release();
  for (auto& m : c.cbuf) m->release();
  for (auto& m : c.rbuf) m->release();
  for (auto& m : c.basis) m->release();
  for (auto& m : c.ibasis) m->release();
  for (int k = 0; k < 2; ++k) {
    c.hy_x0[k].release();
    c.hy_y[k].release();
  }
  c.ncap = 0;
  c.maxit_cap = 0;
  c.incap = 0;
  c.imaxit_cap = 0;
}

// Columns are independent (one Krylov basis per column, filter_engine.hpp:109-111): when the
// workspace of all columns does not fit beside the factors, filter them in column batches.
// Columns are filtered in batches when their workspace does not fit beside the factors. The
// Krylov basis is allocated on demand, so the budget counts `budget_its` basis vectors per column.
int apply_filter_batched_at(zolo_ctx& c, const void* d_v, void* d_y, int64_t ncols, double tol, int64_t gmres_max,
                            zolo_report* rep, int budget_its) {
  auto run = [&](const void* v, void* y, int64_t k, zolo_report* r) {
    return c.cx ? apply_filter_impl<cd>(c, v, y, k, tol, gmres_max, r)
                : apply_filter_impl<double>(c, v, y, k, tol, gmres_max, r);
  };
  const double per_col = bytes_per_column(c, budget_its);
  static const int64_t forced = env_int("ZOLO_FILTER_BATCH", 0);  // (testing) force a column batch size
  // the workspace of an earlier application fits: no device-memory query (cudaMemGetInfo is a
  // driver round trip that can take milliseconds on a busy host)
  if (forced <= 0 && ncols <= c.ncap) return run(d_v, d_y, ncols, rep);
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  free_b += pool_cached_bytes();
  int64_t batch = forced > 0 ? forced : ncols;
  if (forced <= 0) {
    if (ncols * per_col < 0.85 * free_b) return run(d_v, d_y, ncols, rep);
    release_workspace(c);
    CK(cudaMemGetInfo(&free_b, &total_b));
    free_b += pool_cached_bytes();
    batch = std::max<int64_t>(1, static_cast<int64_t>(0.85 * free_b / per_col));
    constexpr int64_t G = 64;  // whole column groups of the widest sweep tasks
    if (batch >= G) {          // whole column groups, spread evenly over the batches
      const int64_t groups = (ncols + G - 1) / G, per = batch / G;
      const int64_t nbat = (groups + per - 1) / per;
      batch = ((groups + nbat - 1) / nbat) * G;
    }
  }
  if (batch >= ncols) return run(d_v, d_y, ncols, rep);
  const size_t colb = c.es() * c.n;
  int code = ZOLO_OK;
  double ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (rep) {
    rep->iterations = 0;
    rep->operator_applications = 0;
    rep->n_shifts = 2 * c.r;
    rep->all_converged = 1;
    for (int k = 0; k < 2 * c.r; ++k) rep->residuals[k] = 0.0, rep->converged[k] = 1;
  }
  std::string err;
  for (int64_t c0 = 0; c0 < ncols; c0 += batch) {
    const int64_t k = std::min(batch, ncols - c0);
    zolo_report rb;
    rb.column_iterations = rep && rep->column_iterations ? rep->column_iterations + c0 : nullptr;
    const int st = run(static_cast<const char*>(d_v) + colb * c0, static_cast<char*>(d_y) + colb * c0, k, &rb);
    if (st != ZOLO_OK && code == ZOLO_OK) {
      code = st;  // the reference finishes every column before rethrowing (filter_engine.hpp:134-137)
      err = c.err;
    }
    for (int i : {0, 2, 3, 4, 5, 6, 7}) ms[i] += c.last_ms[i];
    if (rep) {
      rep->iterations = std::max(rep->iterations, rb.iterations);
      rep->operator_applications += rb.operator_applications;
      rep->all_converged &= rb.all_converged;
      for (int q = 0; q < rb.n_shifts; ++q) {
        rep->residuals[q] = std::max(rep->residuals[q], rb.residuals[q]);
        rep->converged[q] &= rb.converged[q];
      }
    }
  }
  for (int i : {0, 2, 3, 4, 5, 6, 7}) c.last_ms[i] = ms[i];
  if (code != ZOLO_OK) c.err = err;
  return code;
}

// The first application on a context budgets the full gmres_max basis; later ones budget the
// Krylov dimension seen so far (+4), which keeps the whole block in one batch when the factors
// leave room for it. Should an application need more, the basis allocation fails and it is
// re-run under the full budget (columns are independent and deterministic: same bits).
int apply_filter_batched(zolo_ctx& c, const void* d_v, void* d_y, int64_t ncols, double tol, int64_t gmres_max,
                         zolo_report* rep) {
  const int full = static_cast<int>(gmres_max);
  const int seen = c.iters_seen > 0 ? std::min(full, c.iters_seen + 4) : full;
  if (seen >= full || c.hybrid) return apply_filter_batched_at(c, d_v, d_y, ncols, tol, gmres_max, rep, full);
  const int64_t g0 = c.g_apps, s0 = c.inner_solves;
  int64_t* cols = rep ? rep->column_iterations : nullptr;
  try {
    return apply_filter_batched_at(c, d_v, d_y, ncols, tol, gmres_max, rep, seen);
  } catch (const ZoloError& e) {
    if (e.code != ZOLO_ERR_CUDA || std::string(e.what()).find("cudaMalloc") == std::string::npos) throw;
    cudaGetLastError();  // clear the allocation failure
    c.g_apps = g0;
    c.inner_solves = s0;
    if (rep) rep->column_iterations = cols;
    release_workspace(c);
    return apply_filter_batched_at(c, d_v, d_y, ncols, tol, gmres_max, rep, full);
  }
}

}  // namespace

extern "C" {

int zolo_apply_filter_device(zolo_ctx* c, const void* d_v, void* d_y, int64_t ncols, double gmres_tol,
                             int64_t gmres_max, zolo_report* rep) {
  int code = ZOLO_OK;
  const int st = guarded(c, [&] {
    require(ncols >= 1, "apply_filter: empty block");
    code = apply_filter_batched(*c, d_v, d_y, ncols, gmres_tol, gmres_max, rep);
  });
  return st != ZOLO_OK ? st : code;
}

int zolo_apply_filter(zolo_ctx* c, const double* v, double* y, int64_t ncols, double gmres_tol, int64_t gmres_max,
                      zolo_report* rep) {
  int code = ZOLO_OK;
  const int st = guarded(c, [&] {
    require(ncols >= 1, "apply_filter: empty block");
    require(c->factored, "apply_filter: operator not factorized");
    const size_t bytes = c->es() * c->n * ncols;
    c->host_in.ensure(bytes);  // grow-only staging: no per-call cudaMalloc / cudaFree
    c->host_out.ensure(bytes);
    CK(cudaMemcpyAsync(c->host_in.p, v, bytes, cudaMemcpyHostToDevice, c->st));
    code = apply_filter_batched(*c, c->host_in.p, c->host_out.p, ncols, gmres_tol, gmres_max, rep);
    CK(cudaMemcpyAsync(y, c->host_out.p, bytes, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
  });
  return st != ZOLO_OK ? st : code;
}

int zolo_counters(const zolo_ctx* c, int64_t* inner, int64_t* gapps) {
  if (inner) *inner = c->inner_solves;
  if (gapps) *gapps = c->g_apps;
  return ZOLO_OK;
}

int zolo_rr_project(zolo_ctx* c, const double* y, int64_t k, double* at, double* bt) {
  return guarded(c, [&] {
    require(k >= 1, "rr_project: empty block");
    if (c->cx)
      rr_impl<cd>(*c, y, k, at, bt);
    else
      rr_impl<double>(*c, y, k, at, bt);
  });
}

int zolo_block_update(zolo_ctx* c, const double* y, int64_t k, const double* q, int64_t kk, double* out) {
  return guarded(c, [&] {
    require(c->have_pencil, "block_update: no pencil");
    if (kk == 0) return;
    if (c->cx)
      block_update_impl<cd>(*c, y, k, q, kk, out);
    else
      block_update_impl<double>(*c, y, k, q, kk, out);
  });
}

int zolo_timer(zolo_ctx* c, int op, double* ms) {
  return guarded(c, [&] {
    if (!c->tev0) {
      CK(cudaEventCreate(&c->tev0));
      CK(cudaEventCreate(&c->tev1));
    }
    if (op == 0) {
      CK(cudaEventRecord(c->tev0, c->st));
    } else {
      CK(cudaEventRecord(c->tev1, c->st));
      CK(cudaEventSynchronize(c->tev1));
      float f = 0;
      CK(cudaEventElapsedTime(&f, c->tev0, c->tev1));
      if (ms) *ms = f;
    }
  });
}

int zolo_last_timings(const zolo_ctx* c, double* ms) {
  for (int i = 0; i < 8; ++i) ms[i] = c->last_ms[i];
  return ZOLO_OK;
}

int zolo_sweep_profile(const zolo_ctx* c, int64_t* out) {
  for (int i = 0; i < 8; ++i) out[i] = 0;
  if (!c->factored && !c->sym_ready) return ZOLO_ERR_DOMAIN;
  out[0] = c->geom.nbk;
  out[1] = c->sgeom.ntiles;
  out[2] = c->sched_fwd.ntask;
  out[3] = c->sched_bwd.ntask;
  out[4] = c->sp_nslots;
  out[5] = c->critical_path;
  out[6] = c->work_nnz;
  out[7] = c->work_exec;
  return ZOLO_OK;
}

int zolo_nd_order(int64_t n, const int64_t* rp, const int64_t* ci, int64_t leaf, int64_t* pos, int64_t* npad) {
  try {
    std::vector<std::vector<int64_t>> nodes;
    nd_order(n, rp, ci, leaf, nodes);
    BlockStructure bs;
    block_symbolic(n, rp, ci, nodes, TILE, bs);
    for (int64_t i = 0; i < n; ++i) pos[i] = bs.pos[i];
    if (npad) *npad = bs.npad;
    return ZOLO_OK;
  } catch (const std::exception& e) {
    g_create_err = e.what();
    return ZOLO_ERR_DOMAIN;
  }
}

int zolo_nd_structure(int64_t n, const int64_t* rp, const int64_t* ci, int64_t leaf, int64_t* out) {
  try {
    std::vector<std::vector<int64_t>> nodes;
    nd_order(n, rp, ci, leaf, nodes);
    BlockStructure bs;
    block_symbolic(n, rp, ci, nodes, TILE, bs);
    for (int i = 0; i < 8; ++i) out[i] = 0;
    out[0] = bs.npad;
    out[1] = bs.nb;
    out[2] = bs.ntiles;
    out[3] = bs.critical_path;
    out[4] = bs.nb - trailing_dense_start(bs, 1 << 20);
    out[5] = static_cast<int64_t>(nodes.size());
    int64_t con = 0;  // trailing-update tile products of the factorization: sum over block columns of |col(k)|^2
    for (int64_t k = 0; k < bs.nb; ++k) {
      const int64_t ck = bs.col_ptr[k + 1] - bs.col_ptr[k];
      con += ck * ck;
    }
    out[6] = con;
    return ZOLO_OK;
  } catch (const std::exception& e) {
    g_create_err = e.what();
    return ZOLO_ERR_DOMAIN;
  }
}

int zolo_factor_plan_check(int64_t n, const int64_t* rp, const int64_t* ci, int64_t leaf, int64_t* out) {
  try {
    std::vector<std::vector<int64_t>> nodes;
    nd_order(n, rp, ci, leaf, nodes);
    BlockStructure bs;
    block_symbolic(n, rp, ci, nodes, TILE, bs);
    FactorPlan plan;
    factor_plan(bs, plan);
    const int64_t nb = bs.nb, ntiles = bs.ntiles;
    std::vector<int> tile_row(ntiles), level(nb, -1);
    for (int64_t i = 0; i < nb; ++i)
      for (int64_t e = bs.row_ptr[i]; e < bs.row_ptr[i + 1]; ++e) tile_row[e] = static_cast<int>(i);
    const int nlev = static_cast<int>(plan.lvl_ptr.size()) - 1;
    for (int l = 0; l < nlev; ++l)
      for (int q = plan.lvl_ptr[l]; q < plan.lvl_ptr[l + 1]; ++q) level[plan.cols[q]] = l;
    int64_t bad = 0, expect = 0, split = 0;
    for (int64_t k = 0; k < nb; ++k) {
      const int64_t ck = bs.col_ptr[k + 1] - bs.col_ptr[k];
      expect += ck * ck;  // D: ck, L and U: ck (ck - 1) / 2 each
      if (level[k] < 0) ++bad;  // every block column has a level
    }
    // a contribution list [c0, c1) of target (kind, tile or diagonal id): every entry is
    // (L(a, k), U(k, b)) of the target's (a, b) with one k below, a descendant level, ascending
    // k continuing from `last_k`
    auto check_list = [&](int kind, int id, int c0, int c1, int lvl, int& last_k) {
      const int a = kind == 0 ? id : (kind == 1 ? tile_row[id] : static_cast<int>(bs.row_idx[id]));
      const int b = kind == 0 ? id : (kind == 1 ? static_cast<int>(bs.row_idx[id]) : tile_row[id]);
      const int y = std::min(a, b);  // the block column (row of U) the target belongs to
      if (level[y] != lvl) ++bad;
      for (int q = c0; q < c1; ++q) {
        const int la = plan.con[2 * q], ub = plan.con[2 * q + 1];
        if (la < 0 || la >= ntiles || ub < 0 || ub >= ntiles) {
          ++bad;
          continue;
        }
        const int k = static_cast<int>(bs.row_idx[la]);
        if (tile_row[la] != a || tile_row[ub] != b || bs.row_idx[ub] != k || k >= y || k <= last_k ||
            level[k] >= lvl)
          ++bad;
        last_k = k;
      }
    };
    std::vector<char> seen(3 * std::max<int64_t>(ntiles, nb) + 3, 0);
    auto mark_target = [&](int kind, int id) {
      const int64_t lim = kind == 0 ? nb : ntiles;
      if (id < 0 || id >= lim) {
        ++bad;
        return false;
      }
      char& s = seen[3 * static_cast<int64_t>(id) + kind];
      if (s) ++bad;  // every tile is completed by one target
      s = 1;
      return true;
    };
    for (int l = 0; l < nlev; ++l) {
      // part records of the level by scratch slot
      std::vector<std::pair<int, int>> part(static_cast<size_t>(plan.scratch_slots), {-1, -1});
      for (int t = plan.tgt_ptr[l]; t < plan.tgt_ptr[l + 1]; ++t) {
        const int kind = static_cast<unsigned>(plan.tgt[2 * t]) >> 30, id = plan.tgt[2 * t] & 0x3fffffff;
        const int c0 = plan.tgt[2 * t + 1], c1 = plan.tgt[2 * t + 3];
        if (c0 > c1 || c1 > plan.contributions) {
          ++bad;
          continue;
        }
        if (kind == 3) {
          if (id >= plan.scratch_slots || part[id].first >= 0)
            ++bad;
          else
            part[id] = {c0, c1};
        } else if (mark_target(kind, id)) {
          int last_k = -1;
          check_list(kind, id, c0, c1, l, last_k);
        }
      }
      for (int m = plan.cmb_ptr[l]; m < plan.cmb_ptr[l + 1]; ++m) {
        const int kind = static_cast<unsigned>(plan.cmb[3 * m]) >> 30, id = plan.cmb[3 * m] & 0x3fffffff;
        const int s0 = plan.cmb[3 * m + 1], np = plan.cmb[3 * m + 2];
        ++split;
        if (kind > 2 || np < 2 || s0 < 0 || s0 + np > plan.scratch_slots || !mark_target(kind, id)) {
          ++bad;
          continue;
        }
        int last_k = -1;
        for (int p = 0; p < np; ++p) {  // the parts continue one ascending list
          if (part[s0 + p].first < 0) {
            ++bad;
            continue;
          }
          check_list(kind, id, part[s0 + p].first, part[s0 + p].second, l, last_k);
          part[s0 + p] = {-2, -2};
        }
      }
      for (const auto& pr : part)
        if (pr.first >= 0) ++bad;  // a part no combine entry reads
    }
    if (plan.contributions != expect) ++bad;
    out[0] = bad;
    out[1] = plan.contributions;
    out[2] = plan.tgt_ptr.empty() ? 0 : plan.tgt_ptr.back();
    out[3] = split;
    out[4] = plan.scratch_slots;
    out[5] = nlev;
    return ZOLO_OK;
  } catch (const std::exception& e) {
    g_create_err = e.what();
    return ZOLO_ERR_DOMAIN;
  }
}

int zolo_dag_schedule_check(int64_t n, const int64_t* rp, const int64_t* ci, int64_t leaf, int near, int chunk,
                            int order, int64_t* out) {
  try {
    std::vector<std::vector<int64_t>> nodes;
    nd_order(n, rp, ci, leaf, nodes);
    BlockStructure bs;
    block_symbolic(n, rp, ci, nodes, TILE, bs);
    const int64_t nb = bs.nb;
    int64_t bad = 0, ntask = 0, nslot_all = 0;
    for (int dir = 0; dir < 2; ++dir) {
      const bool fwd = dir == 0;
      const auto& ptr = fwd ? bs.row_ptr : bs.col_ptr;
      const auto& idx = fwd ? bs.row_idx : bs.col_idx;
      std::vector<DagTask> ts;
      const int nslots = dag_schedule(nb, ptr, idx, fwd, chunk, near, order, ts);
      // every row has one row task; every dependency of every row is summed exactly once; a task
      // appears after the tasks it waits on (claim order topological); the partial slots (see
      // DagTask): every write stamps more than the slot held, a chunk that continues a chain reads
      // its own row's previous step, a chunk that takes over a slot waits for the row task that
      // last read it, a row task reads the last step of each of its chains
      std::vector<int64_t> row_at(nb, -1), covered(nb, 0);
      for (size_t t = 0; t < ts.size(); ++t) {
        const DagTask& k = ts[t];
        if (k.out < 0) {
          if (row_at[k.i] >= 0) ++bad;
          row_at[k.i] = static_cast<int64_t>(t);
        }
        covered[k.i] += k.qb - k.qa;
      }
      std::vector<int64_t> stamp(nslots, -1);
      std::vector<int> wrow(nslots, -1), rrow(nslots, -1);  // last writer row / reader row
      auto st_of = [](int gen, int step) { return static_cast<int64_t>(64) * gen + step; };
      for (size_t t = 0; t < ts.size(); ++t) {
        const DagTask& k = ts[t];
        const int64_t e0 = ptr[k.i];
        const int nd = static_cast<int>(ptr[k.i + 1] - e0);
        for (int q = k.qa; q < k.qb; ++q) {
          const int64_t j = fwd ? idx[e0 + q] : idx[e0 + nd - 1 - q];
          if (row_at[j] < 0 || row_at[j] >= static_cast<int64_t>(t)) ++bad;
        }
        if (k.pc > 0 && (k.pa < 0 || k.pa + k.pc > nslots)) {
          ++bad;
          continue;
        }
        if (k.out >= 0) {
          const int c = k.aux & 0xffff, ki = k.aux >> 16, step = c / std::max(ki, 1);
          if (k.out >= nslots || ki < 1 || st_of(k.gen, step) <= stamp[k.out]) ++bad;
          if (step > 0) {  // continues its chain
            if (k.pc != 1 || k.pa != k.out || wrow[k.out] != k.i || stamp[k.out] != st_of(k.gen, step - 1) ||
                k.wait >= 0)
              ++bad;
          } else if (wrow[k.out] >= 0) {  // takes over a slot of another row's unit
            if (k.pc != 0 || k.wait < 0 || k.wait != rrow[k.out] || row_at[k.wait] >= static_cast<int64_t>(t)) ++bad;
          }
          stamp[k.out] = st_of(k.gen, step);
          wrow[k.out] = k.i;
        } else if (k.pc > 0) {
          const int nchunk = k.aux;
          for (int q = 0; q < k.pc; ++q) {
            const int sl = k.pa + q;
            if (wrow[sl] != k.i || stamp[sl] != st_of(k.gen, (nchunk - 1 - q) / k.pc)) ++bad;
            rrow[sl] = k.i;
          }
        }
      }
      for (int64_t i = 0; i < nb; ++i)
        if (row_at[i] < 0 || covered[i] != ptr[i + 1] - ptr[i]) ++bad;
      ntask += static_cast<int64_t>(ts.size());
      nslot_all += nslots;
    }
    out[0] = bad;
    out[1] = ntask;
    out[2] = nslot_all;
    out[3] = nb;
    return ZOLO_OK;
  } catch (const std::exception& e) {
    g_create_err = e.what();
    return ZOLO_ERR_DOMAIN;
  }
}

int zolo_rcm(int64_t n, const int64_t* rp, const int64_t* ci, int64_t* perm, int64_t* bw, int64_t* profile) {
  try {
    rcm_order(n, rp, ci, perm);
    if (bw) *bw = bandwidth_under(n, rp, ci, perm);
    if (profile) *profile = profile_under(n, rp, ci, perm);
    return ZOLO_OK;
  } catch (const std::exception& e) {
    g_create_err = e.what();
    return ZOLO_ERR_NUMERICAL;
  }
}

int zolo_uniform_stream(uint64_t seed, int64_t n, double* out) {
  uniform_stream(seed, n, out);
  return ZOLO_OK;
}

int zolo_random_block(int scalar, int64_t n, int64_t k, uint64_t seed, int orthonormalize, double* out) {
  return random_block(scalar, n, k, seed, orthonormalize != 0, out) ? ZOLO_OK : ZOLO_ERR_NUMERICAL;
}

}  // extern "C"

// Collectives of the pole-sharded filter: the inner operator
// is a sum over poles (filter_engine.hpp:63-69, 73-78), so rank g factors the
// poles j = g, g + nranks, ... and every G application ends with a reduction
// of the ranks' partial sums over NVLink / NVSwitch (capi.cu combine_g: a
// reduce-scatter over row blocks when the Arnoldi step is row-sharded, an
// all-reduce when it is replicated). NCCL is opened with dlopen when a
// communicator is built, so single-GPU use has no NCCL dependency; the
// library resolves to the libnccl.so.2 already loaded by torch when there is
// one. The host-staged variant runs the same control flow through a caller
// callback (tests: several ranks as threads of one process on one GPU, where
// no kernel of one rank waits on another's).
#include <dlfcn.h>
#include <nccl.h>

#include <stdexcept>
#include <string>

#include "shard.hpp"

namespace zolo {

namespace {
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*reduce_scatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                 cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  if (a.h) return a;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* nm : names) {
    a.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (a.h) break;
  }
  if (!a.h) throw std::runtime_error(std::string("pole sharding: cannot load libnccl.so.2: ") + dlerror());
  auto sym = [&](const char* s) {
    void* p = dlsym(a.h, s);
    if (!p) throw std::runtime_error(std::string("pole sharding: NCCL symbol missing: ") + s);
    return p;
  };
  a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(sym("ncclGetUniqueId"));
  a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(sym("ncclCommInitRank"));
  a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(sym("ncclAllReduce"));
  a.reduce_scatter = reinterpret_cast<decltype(a.reduce_scatter)>(sym("ncclReduceScatter"));
  a.all_gather = reinterpret_cast<decltype(a.all_gather)>(sym("ncclAllGather"));
  a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(sym("ncclCommDestroy"));
  a.error_string = reinterpret_cast<decltype(a.error_string)>(sym("ncclGetErrorString"));
  return a;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw std::runtime_error(std::string(what) + ": " + api().error_string(r));
}

struct NcclCollective : Collective {
  ncclComm_t comm = nullptr;
  ~NcclCollective() override {
    if (comm) api().comm_destroy(comm);
  }
  void allreduce(double* buf, size_t count, cudaStream_t st) override {
    check(api().all_reduce(buf, buf, count, ncclFloat64, ncclSum, comm, st), "ncclAllReduce");
  }
  void reduce_scatter(const double* in, double* out, size_t per_rank, cudaStream_t st) override {
    check(api().reduce_scatter(in, out, per_rank, ncclFloat64, ncclSum, comm, st), "ncclReduceScatter");
  }
  void allgather(const double* in, double* out, size_t per_rank, cudaStream_t st) override {
    check(api().all_gather(in, out, per_rank, ncclFloat64, comm, st), "ncclAllGather");
  }
};

struct HostCollective : Collective {
  HostCollectiveFn fn = nullptr;
  void* user = nullptr;
  std::vector<double> buf;
  void call(int op, int64_t count) {
    if (fn(op, buf.data(), count, user) != 0) throw std::runtime_error("pole sharding: host collective failed");
  }
  void sync(cudaStream_t st) {
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) throw std::runtime_error(std::string("host collective: ") + cudaGetErrorString(e));
  }
  void allreduce(double* d, size_t count, cudaStream_t st) override {
    buf.resize(count);
    cudaMemcpyAsync(buf.data(), d, count * 8, cudaMemcpyDeviceToHost, st);
    sync(st);
    call(0, static_cast<int64_t>(count));
    cudaMemcpyAsync(d, buf.data(), count * 8, cudaMemcpyHostToDevice, st);
    sync(st);
  }
  void reduce_scatter(const double* in, double* out, size_t per_rank, cudaStream_t st) override {
    buf.resize(per_rank * nranks);
    cudaMemcpyAsync(buf.data(), in, per_rank * nranks * 8, cudaMemcpyDeviceToHost, st);
    sync(st);
    call(1, static_cast<int64_t>(per_rank));
    cudaMemcpyAsync(out, buf.data(), per_rank * 8, cudaMemcpyHostToDevice, st);
    sync(st);
  }
  void allgather(const double* in, double* out, size_t per_rank, cudaStream_t st) override {
    buf.resize(per_rank * nranks);
    cudaMemcpyAsync(buf.data() + per_rank * rank, in, per_rank * 8, cudaMemcpyDeviceToHost, st);
    sync(st);
    call(2, static_cast<int64_t>(per_rank));
    cudaMemcpyAsync(out, buf.data(), per_rank * nranks * 8, cudaMemcpyHostToDevice, st);
    sync(st);
  }
};
}  // namespace

static_assert(sizeof(ncclUniqueId) == ZOLO_NCCL_ID_BYTES, "ncclUniqueId size");

void nccl_unique_id(void* out) {
  ncclUniqueId id;
  check(api().get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
}

Collective* nccl_collective(const void* unique_id, int nranks, int rank) {
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  auto* c = new NcclCollective();
  c->rank = rank;
  c->nranks = nranks;
  const ncclResult_t r = api().comm_init_rank(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    c->comm = nullptr;
    delete c;
    check(r, "ncclCommInitRank");
  }
  return c;
}

Collective* host_collective(HostCollectiveFn fn, void* user, int nranks, int rank) {
  auto* c = new HostCollective();
  c->fn = fn;
  c->user = user;
  c->nranks = nranks;
  c->rank = rank;
  return c;
}

}  // namespace zolo

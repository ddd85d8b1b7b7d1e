// Pole sharding over NCCL: the inner operator is a sum over
// poles (filter_engine.hpp:63-69, 73-78), so rank g factors the poles
// j = g, g + nranks, ... and every G application ends with one in-place
// ncclAllReduce(sum) of the ranks' partial sums on the library stream. NCCL is
// opened with dlopen at zolo_set_pole_shard time, so single-GPU use has no
// NCCL dependency; the library resolves to the libnccl.so.2 already loaded by
// torch when there is one.
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
  a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(sym("ncclCommDestroy"));
  a.error_string = reinterpret_cast<decltype(a.error_string)>(sym("ncclGetErrorString"));
  return a;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw std::runtime_error(std::string(what) + ": " + api().error_string(r));
}
}  // namespace

struct NcclComm {
  ncclComm_t comm = nullptr;
};

static_assert(sizeof(ncclUniqueId) == ZOLO_NCCL_ID_BYTES, "ncclUniqueId size");

void nccl_unique_id(void* out) {
  ncclUniqueId id;
  check(api().get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
}

NcclComm* nccl_open(const void* unique_id, int nranks, int rank) {
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  auto* c = new NcclComm();
  const ncclResult_t r = api().comm_init_rank(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    check(r, "ncclCommInitRank");
  }
  return c;
}

void nccl_allreduce_sum(NcclComm* c, double* buf, size_t count, cudaStream_t st) {
  check(api().all_reduce(buf, buf, count, ncclFloat64, ncclSum, c->comm, st), "ncclAllReduce");
}

void nccl_close(NcclComm* c) {
  if (!c) return;
  if (c->comm) api().comm_destroy(c->comm);
  delete c;
}

}  // namespace zolo

#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <cstring>
#include <vector>

#define ZOLO_NCCL_ID_BYTES 128

namespace zolo {
// The collective operations of a pole-shard group, on device buffers of
// doubles, stream-ordered on `st`:
//   allreduce       in place, sum over the ranks
//   reduce_scatter  in: nranks x per_rank doubles (rank-major blocks); out: this rank's block summed
//   allgather       in: this rank's per_rank doubles; out: nranks x per_rank (rank-major)
struct Collective {
  int rank = 0, nranks = 1;
  virtual ~Collective() {}
  virtual void allreduce(double* buf, size_t count, cudaStream_t st) = 0;
  virtual void reduce_scatter(const double* in, double* out, size_t per_rank, cudaStream_t st) = 0;
  virtual void allgather(const double* in, double* out, size_t per_rank, cudaStream_t st) = 0;
};
void nccl_unique_id(void* out);  // ZOLO_NCCL_ID_BYTES
// NCCL over NVLink / NVSwitch (dlopen'ed libnccl.so.2); collective over the ranks
Collective* nccl_collective(const void* unique_id, int nranks, int rank);
// host-staged collective through a caller callback (zolo_set_pole_shard_host): device -> host,
// callback(op, buffer, count, user), host -> device
typedef int (*HostCollectiveFn)(int op, double* buf, int64_t count, void* user);
Collective* host_collective(HostCollectiveFn fn, void* user, int nranks, int rank);
// poles owned by `rank` of `nranks`: j = rank, rank + nranks, ... (< r)
inline int shard_pole_count(int r, int rank, int nranks) { return rank < r ? (r - 1 - rank) / nranks + 1 : 0; }
}  // namespace zolo

#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstring>

#define ZOLO_NCCL_ID_BYTES 128

namespace zolo {
struct NcclComm;
void nccl_unique_id(void* out);                                // ZOLO_NCCL_ID_BYTES
NcclComm* nccl_open(const void* unique_id, int nranks, int rank);  // collective over the ranks
void nccl_allreduce_sum(NcclComm* c, double* buf, size_t count, cudaStream_t st);
void nccl_close(NcclComm* c);
// poles owned by `rank` of `nranks`: j = rank, rank + nranks, ... (< r)
inline int shard_pole_count(int r, int rank, int nranks) { return rank < r ? (r - 1 - rank) / nranks + 1 : 0; }
}  // namespace zolo

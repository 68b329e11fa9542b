// mrq_comm.cuh -- multi-GPU list sharding and the decision-T exchanges
// (DESIGN.md §6).
#pragma once
#include <vector>
#include "mrq_internal.cuh"

void mrq_shard_lists(const std::vector<uint32_t> &sizes, int world, std::vector<uint32_t> &owner);
// Sets up the exchange of a world > 1 index: NCCL communicator from the unique
// id, else the host all-gather callback.
int mrq_comm_init(mrq_index *ix, const mrq_dist_cfg *dist);
void mrq_comm_free(mrq_index *ix);
// All-gather of `bytes` per rank from device `send` into device `recv`
// (world * bytes, rank-major) on stream st.  world == 1: a device copy.
int mrq_allgather(mrq_index *ix, const void *send, void *recv, size_t bytes, cudaStream_t st);
// Grouped all-gathers (one NCCL group; in place when send = recv + rank * bytes).
int mrq_allgather_group(mrq_index *ix, int n, const void *const *send, void *const *recv, const size_t *bytes,
                        cudaStream_t st);
// Abort the communicator after a failed collective (later exchanges return MRQ_ENCCL).
void mrq_comm_fail(mrq_index *ix);

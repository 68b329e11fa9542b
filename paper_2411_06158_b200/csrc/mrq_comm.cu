// mrq_comm.cu -- list sharding across ranks and NCCL exchanges.
#include <algorithm>
#include <numeric>

#include "mrq_comm.cuh"

// Greedy longest-processing-time assignment of lists to ranks: lists by size
// descending (ties by id), each to the currently least-loaded rank (ties by
// rank).  Deterministic, so every rank computes the same map.
void mrq_shard_lists(const std::vector<uint32_t> &sizes, int world, std::vector<uint32_t> &owner)
{
    const int k = (int)sizes.size();
    std::vector<int> order(k);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return sizes[a] > sizes[b]; });
    std::vector<uint64_t> load(world, 0);
    owner.assign(k, 0);
    for (int c : order) {
        int best = 0;
        for (int r = 1; r < world; r++)
            if (load[r] < load[best]) best = r;
        owner[c] = (uint32_t)best;
        load[best] += sizes[c];
    }
}

int mrq_comm_init(mrq_index *, const void *)
{
    mrq_set_error("multi-GPU (NCCL) path not built in this library");
    return MRQ_ENCCL;
}
void mrq_comm_free(mrq_index *) {}
int mrq_comm_seeds(mrq_index *, int64_t, int, int, uint32_t *, uint32_t *, double *, double *, cudaStream_t)
{
    return MRQ_ENCCL;
}
int mrq_comm_tau1(mrq_index *, int64_t, int, int, const uint32_t *, const uint32_t *, const double *,
                  const uint32_t *, const uint32_t *, const double *, double *, cudaStream_t)
{
    return MRQ_ENCCL;
}
int mrq_comm_merge(mrq_index *, int64_t, int, int64_t *, float *, cudaStream_t) { return MRQ_ENCCL; }

// mrq_comm.cuh -- multi-GPU list sharding and the NCCL exchanges.
#pragma once
#include <vector>
#include "mrq_internal.cuh"

void mrq_shard_lists(const std::vector<uint32_t> &sizes, int world, std::vector<uint32_t> &owner);
int mrq_comm_init(mrq_index *ix, const void *unique_id);
void mrq_comm_free(mrq_index *ix);
int mrq_comm_seeds(mrq_index *ix, int64_t nq, int K, int Kp, uint32_t *s0_cnt, uint32_t *s0_pos, double *s0_exact,
                   double *tau0, cudaStream_t st);
int mrq_comm_tau1(mrq_index *ix, int64_t nq, int K, int Kp, const uint32_t *s0_cnt, const uint32_t *s0_pos,
                  const double *s0_exact, const uint32_t *s1_cnt, const uint32_t *s1_pos, const double *s1_exact,
                  double *tau1, cudaStream_t st);
int mrq_comm_merge(mrq_index *ix, int64_t nq, int K, int64_t *d_ids, float *d_dist, cudaStream_t st);

// mrq_probe_tc.cuh -- tcgen05 tensor-core screen of the probe (Alg.2 L7).
#pragma once
#include "mrq_internal.cuh"

int mrq_probe_tc_init(mrq_index *ix);
void mrq_probe_tc_free(mrq_index *ix);
bool mrq_probe_tc_enabled(const mrq_index *ix);
double mrq_probe_tc_kappa(const mrq_index *ix);
int mrq_probe_tc_run(mrq_index *ix, const float *qd32, int64_t nq, float *approx, cudaStream_t st);

// mrq_probe_tc.cuh -- tcgen05 tensor-core screen of the probe (Alg.2 L7).
#pragma once
#include "mrq_internal.cuh"

int mrq_probe_tc_init(mrq_index *ix);
void mrq_probe_tc_free(mrq_index *ix);
bool mrq_probe_tc_enabled(const mrq_index *ix);
double mrq_probe_tc_kappa(const mrq_index *ix);
int mrq_probe_tc_run(mrq_index *ix, const float *qd32, int64_t nq, float *approx, cudaStream_t st);
// Fused screen + running top-np (np <= 16), the row's columns split into P
// parts (mrq_probe_tc_parts): per-(row, part) candidate buffers
// cbuf[nq][P][capp] of (screen value bits, centroid), counts ccnt[nq][P] and
// the part's 16 smallest screen values kvbuf[nq][P][16]; finished by
// launch_probe_finish_w.
bool mrq_probe_tc_fusable(const mrq_index *ix, int np);
int mrq_probe_tc_parts(const mrq_index *ix, int64_t nq);
int mrq_probe_tc_run_fused(mrq_index *ix, const float *qd32, int64_t nq, int np, const double *qnorm, double kappa,
                           uint2 *cbuf, int capp, uint32_t *ccnt, float *kvbuf, cudaStream_t st);

// mrq_probe_tc.cuh -- tcgen05 tensor-core screen of the probe (Alg.2 L7).
#pragma once
#include "mrq_internal.cuh"

int mrq_probe_tc_init(mrq_index *ix);
void mrq_probe_tc_free(mrq_index *ix);
bool mrq_probe_tc_enabled(const mrq_index *ix);
double mrq_probe_tc_kappa(const mrq_index *ix);
int mrq_probe_tc_run(mrq_index *ix, const float *qd32, int64_t nq, float *approx, cudaStream_t st);
// Fused screen + running top-np (np <= 64), the row's columns split into P
// parts (mrq_probe_tc_parts): per-(row, part) candidate buffers
// cbuf[nq][P][capp] of (screen value bits, centroid), counts ccnt[nq][P] and
// the part's np smallest screen values kvbuf[nq][P][np]; gkey[nq] (scratch,
// or NULL) carries the bound the parts of a row share; finished by
// launch_probe_finish_w.
bool mrq_probe_tc_fusable(const mrq_index *ix, int np);
int mrq_probe_tc_capp(const mrq_index *ix, int np);
int mrq_probe_tc_parts(const mrq_index *ix, int64_t nq);
int mrq_probe_tc_grid(const mrq_index *ix, int64_t nq);

// Balanced schedule of the probe GEMM: the mblocks x ntiles (128-query block,
// 256-centroid tile) units, flattened block-major, are split into G
// contiguous ranges, one per CTA (G = the SM count), so one wave does all the
// work.  CTA i owns units [u0(i), u0(i+1)), u0(i) = floor(i U / G).  A query
// block's tiles span a few consecutive CTAs; its "part" in a CTA is that
// CTA's rank among them (x 2 epilogue halves).
#define TC_BM 128
#define TC_BN 256
__host__ __device__ __forceinline__ int64_t tc_u0(int64_t i, int64_t U, int64_t G) { return i * U / G; }
__host__ __device__ __forceinline__ int64_t tc_owner(int64_t u, int64_t U, int64_t G)
{
    int64_t i = u * G / U;
    while (i + 1 < G && tc_u0(i + 1, U, G) <= u) i++;
    while (i > 0 && tc_u0(i, U, G) > u) i--;
    return i;
}
// parts actually written for query block mb
__host__ __device__ __forceinline__ int tc_parts_of(int64_t mb, int64_t nq, int k, int G)
{
    const int64_t ntiles = (k + TC_BN - 1) / TC_BN, U = ((nq + TC_BM - 1) / TC_BM) * ntiles;
    return (int)(2 * (tc_owner((mb + 1) * ntiles - 1, U, G) - tc_owner(mb * ntiles, U, G) + 1));
}
int mrq_probe_tc_run_fused(mrq_index *ix, const float *qd32, int64_t nq, int np, const double *qnorm, double kappa,
                           uint2 *cbuf, int capp, uint32_t *ccnt, float *kvbuf, uint32_t *gkey, cudaStream_t st);

// mrq_kernels.cuh -- kernel declarations and launch argument packs.
#pragma once
#include "mrq_internal.cuh"

void launch_rowmat_f32(const float *X, int64_t nrows, int ldx, int Din, const double *mu, const double *MT, int Dout,
                       double *out, int ldo, cudaStream_t st);
void launch_rowmat_f64(const double *X, int64_t nrows, int ldx, int Din, const double *mu, const double *MT,
                       int Dout, double *out, int ldo, cudaStream_t st);
__global__ void k_encode_finish(const double *xp, int64_t n0, int64_t cnt, int D, int d, int W,
                                const uint32_t *assign, const uint32_t *slot_of, const double *C, const double *RT,
                                int64_t npad, float *heads, float *tails, float *xr2o, uint32_t *codes, float *f1,
                                float *f2, float *f3, uint8_t *hq, float4 *hs, int dq);
__global__ void k_rc(const double *C, const double *RT, int k, int d, int W, double *Rc);
__global__ void k_qtail(const double *qp, int64_t nq, int D, int d, int W, const double *lam, const double *RT,
                        double rscale, double m, double *qr2o, double *eps_r, double *r0, float *qd32,
                        double *qnorm, uint16_t *qkey, float *qa3);
__global__ void k_probe_approx(const float *qd32, int64_t nq, int d, int k, const float *C32T, float *approx);
void launch_fill_f64(double *p, int64_t n, double v, cudaStream_t st);
void launch_qorder(const uint16_t *qkey, int64_t nq, uint32_t *order, cudaStream_t st);
void launch_quant(const uint32_t *probe, const double *probe_qn2, int64_t nq, int np, int d, int W,
                  const double *r0, const double *Rc, const double *qr2, double eps0, uint32_t *planes,
                  double *qconst, uint8_t *qsk_b, double *qsk_c, int dq, const double *qnorm, double cmax,
                  cudaStream_t st);
__global__ void k_cand_count(const uint32_t *probe, int64_t nq, int np, const uint32_t *list_size, uint64_t *cnt,
                             const uint16_t *list_key, uint16_t *qkey);
__global__ void k_offsets_order(const uint64_t *cnt, int64_t nq, uint64_t *off, const uint16_t *qkey,
                                uint32_t *order);
__global__ void k_exclusive_scan(const uint64_t *in, int64_t n, uint64_t *out);
struct StageArgs {
    int64_t nq;
    int np, K, Kp, D, d, mode, tight, aligned, seed_lists, aligned_tails;
    int store_f1;             // k_head_b also writes f1_head/f1_diso/f1_id when F2 is fused (debug dumps)
    int sketch;               // the scan dropped F1 entries with the head sketch (LOOSE): f1_pos holds
    uint32_t *surv_cnt;       // surv_cnt[q] survivors per query
    int64_t npad;
    double isd;
    const uint32_t *probe, *list_off, *list_size, *ids, *codes, *planes;
    const float *f1, *f2, *f3, *heads, *tails, *xr2;
    const double *qconst, *qp, *qr2, *eps_r;
    const uint32_t *list_size_g;
    uint32_t *s0_cnt, *s0_pos, *s1_cnt, *s1_pos, *f1_cnt, *f1_pos, *f2_cnt, *f2_pos, *exact_cnt;
    uint32_t *s0_id, *s1_id;
    XItem *xout;   // sharded exchange send buffer (NULL = single-rank fast path)
    double *s0_exact, *s1_exact, *tau0, *tau1, *f1_head, *f1_diso, *f2_head, *f2_exact;
    uint32_t *f1_id;
    const uint64_t *f1_off;
    int64_t *out_ids;
    float *out_dist;
    const uint32_t *qorder;   // processing order of the queries (NULL: 0..nq-1)
    int fuse_topk;            // allow k_head_topk (stage 2 + re-rank + top-K in one kernel)
};

// the fused head-sketch test of the scan (FULL with tau1 = tau0, i.e. LOOSE;
// no debug dumps): k_head_b then gathers only the survivors
inline bool mrq_sketch_used(const StageArgs &a)
{
    return a.sketch && a.mode == 0 && !a.tight && !a.store_f1 && a.surv_cnt;
}
int launch_seed_w(int W, const StageArgs &a, cudaStream_t st);
int launch_stage2_w(const StageArgs &a, cudaStream_t st, cudaEvent_t after_gather = nullptr);
int launch_topk_w(const StageArgs &a, cudaStream_t st);
bool mrq_head_topk_used(const StageArgs &a);
int launch_head_topk(const StageArgs &a, cudaStream_t st);
int launch_nocorr_w(int W, const StageArgs &a, cudaStream_t st);
int launch_exact_count(const StageArgs &a, cudaStream_t st);
int launch_f2_w(const StageArgs &a, cudaStream_t st);
int launch_xmerge(int kind, const StageArgs &a, int world, int rank, const XItem *recv, cudaStream_t st);

struct LaunchScan {
    int64_t nq;
    size_t smem;
    const uint32_t *probe;
    int np;
    int64_t npad;
    const uint32_t *list_off, *list_size, *codes;
    const float *f1, *f2, *f3;
    const uint32_t *planes;
    const double *qconst, *eps_r, *tau0;
    double isd;
    const uint64_t *f1_off;
    uint32_t *f1_cnt, *f1_pos;
    const uint32_t *qorder;   // processing order of the queries (NULL: 0..nq-1)
    // fused head-sketch test (surv_cnt != NULL): see ScanSketch in mrq_kernels.cu
    const uint8_t *hq, *qsk_b;
    const float4 *hs;
    const double *qsk_c, *qr2;
    int dq;
    uint32_t *surv_cnt;
    // list-major scan (lm != 0): the (query, probed list) pairs
    // grouped by list (mrq_lm_build); the work units are (list, 128-slot tile,
    // chunk of <= qg of the list's pairs), handed out by an atomic counter
    int lm, k, qg;
    const uint32_t *pairs, *loff, *upre, *unit_list;
    uint32_t *unit_ctr;
};

// scratch of the list-major scan's pair grouping (all device, k + 1 / nq np entries)
struct LmScratch {
    uint32_t *lcnt, *lfill, *loff, *upre, *pairs, *unit_ctr;
    uint32_t *unit_list;   // [units]: the list of each work unit
};
// pairs of list c: pairs[loff[c] .. loff[c + 1]) (pair = q np + p); units of
// list c: upre[c] .. upre[c + 1) = ceil(size_c / 128) ceil(count_c / qg)
int mrq_lm_build(const uint32_t *probe, int64_t nq, int np, int k, const uint32_t *list_size, int qg,
                 const LmScratch &s, cudaStream_t st);

// dynamic shared memory of k_scan: per probed list 5 constants, 4 W plane words, tile prefix / start / end
inline size_t mrq_scan_smem(int np, int W)
{
    return (size_t)np * 5 * 8 + (size_t)np * MRQ_BQ * W * 4 + (size_t)(3 * np + 1) * 4;
}
// ... plus, with the fused head-sketch test, the per-list sketch constants and rows
inline size_t mrq_scan_smem_sk(int np, int W, int dq) { return mrq_scan_smem(np, W) + (size_t)np * 24 + 16 + (size_t)np * (dq + 16); }
// The fused sketch's queue entry packs (probe index, slot) into 32 bits: the probe index takes
// ceil(log2 np) high bits, the slot the rest (np = 16: up to 2^28 slots per GPU; np = 64: 2^26).
// A search that does not fit runs without the sketch (same results).
inline int mrq_scan_pshift(int np)
{
    int b = 0;
    while ((1 << b) < np) b++;
    return 32 - b;
}
inline bool mrq_scan_sketch_fits(int np, int64_t npad) { return npad <= ((int64_t)1 << mrq_scan_pshift(np)); }
int launch_scan(int W, const LaunchScan &a, cudaStream_t st);
bool supported_W(int W);
void launch_f1_all(const uint32_t *probe, int64_t nq, int np, const uint32_t *list_off, const uint32_t *list_size,
                   const uint64_t *f1_off, uint32_t *f1_cnt, uint32_t *f1_pos, cudaStream_t st);
void launch_scan_dbg(int W, const LaunchScan &a, double *dis, double *lb1, cudaStream_t st);
int launch_probe_finish_w(int64_t nq, int k, int d, int np, const double *qp, int D, const double *C,
                          const double *qnorm, double cmax, double kappa, const uint2 *cbuf, int P, int capp,
                          int G, const uint32_t *ccnt, const float *kvbuf, uint32_t *cand, uint32_t *probe,
                          double *probe_qn2, uint32_t *ncand, cudaStream_t st);
int launch_probe_select_w(const float *approx, int64_t nq, int k, int d, int np, const double *qp, int D,
                          const double *C, const double *qnorm, double cmax, double kappa, uint32_t *cand,
                          uint32_t *probe, double *probe_qn2, uint32_t *ncand, cudaStream_t st);

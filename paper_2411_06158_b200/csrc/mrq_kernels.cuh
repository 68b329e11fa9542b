// mrq_kernels.cuh -- kernel declarations and launch argument packs.
#pragma once
#include "mrq_internal.cuh"

__global__ void k_project(const float *X, int64_t nrows, int D, const double *mu, const double *PT, double *out);
__global__ void k_encode_finish(const double *xp, int64_t n0, int64_t cnt, int D, int d, int W,
                                const uint32_t *assign, const uint32_t *slot_of, const double *C, const double *RT,
                                int64_t npad, float *heads, float *tails, float *xr2o, uint32_t *codes, float *f1,
                                float *f2, float *f3);
__global__ void k_rc(const double *C, const double *RT, int k, int d, int W, double *Rc);
__global__ void k_qtail(const double *qp, int64_t nq, int D, int d, int W, const double *lam, const double *RT,
                        double rscale, double m, double *qr2o, double *eps_r, double *r0, float *qd32,
                        double *qnorm);
__global__ void k_probe_approx(const float *qd32, int64_t nq, int d, int k, const float *C32T, float *approx);
__global__ void k_probe_select(const float *approx, int64_t nq, int k, int d, int np, const double *qp, int D,
                               const double *C, const double *qnorm, double cmax, double kappa, int cap, int S,
                               uint32_t *probe, double *probe_qn2, uint32_t *fallback_cnt);
__global__ void k_quant(const uint32_t *probe, const double *probe_qn2, int64_t nq, int np, int d, int W,
                        const double *r0, const double *Rc, const double *qr2, double eps0, uint32_t *planes,
                        double *qconst);
__global__ void k_cand_count(const uint32_t *probe, int64_t nq, int np, const uint32_t *list_size, uint64_t *cnt);
__global__ void k_exclusive_scan(const uint64_t *in, int64_t n, uint64_t *out);
__global__ void k_stage2(int mode, int tight, int K, int Kp, int D, int d, const uint32_t *ids, const float *heads,
                         const float *tails, const float *xr2, const double *qp, const double *qr2_arr,
                         const double *eps_r_arr, const double *tau0_arr, const uint64_t *f1_off,
                         const uint32_t *f1_cnt, const uint32_t *f1_pos, double *f1_head, double *f1_diso,
                         const uint32_t *s0_cnt, const uint32_t *s0_pos, const double *s0_exact, uint32_t *s1_cnt,
                         uint32_t *s1_pos, double *s1_exact, int S, double *tau1_arr, uint32_t *f2_cnt,
                         uint32_t *f2_pos, double *f2_head);
__global__ void k_rerank(int D, int d, const float *tails, const double *qp, const uint64_t *f1_off,
                         const uint32_t *f2_cnt, const uint32_t *f2_pos, const double *f2_head, double *f2_exact);
__global__ void k_topk(int K, int Kp, const uint32_t *ids, const uint32_t *s0_cnt, const uint32_t *s0_pos,
                       const double *s0_exact, const uint32_t *s1_cnt, const uint32_t *s1_pos,
                       const double *s1_exact, const uint64_t *f1_off, const uint32_t *f2_cnt,
                       const uint32_t *f2_pos, const double *f2_exact, int S, int64_t *out_ids, float *out_dist,
                       uint32_t *exact_cnt);

struct LaunchSeed {
    int64_t nq;
    size_t smem;
    const uint32_t *probe;
    int np, K, Kp, D, d;
    int64_t npad;
    const uint32_t *list_off, *list_size, *ids, *codes;
    const float *f1, *f2, *f3, *heads, *tails;
    const uint32_t *planes;
    const double *qconst, *qp, *eps_r;
    double isd;
    int pool_cap, S;
    SelItem *pool;
    uint32_t *s0_cnt, *s0_pos;
    double *s0_exact, *tau0;
};

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
};

void launch_seed(int W, const LaunchSeed &a, cudaStream_t st);
void launch_scan(int W, const LaunchScan &a, cudaStream_t st);
bool supported_W(int W);
void launch_scan_dbg(int W, const LaunchScan &a, double *dis, double *lb1, cudaStream_t st);

// mrq_stages.cu -- seeds (a4), stage 2 (a6), exact re-rank (a7) and top-K
// (a8): one warp per query.  The selections keep a warp-private sorted top-L
// list in shared memory (WarpTop), so a query's candidates stream through the
// warp once; rows are gathered through a 32x33 shared tile so global loads
// stay 128-byte coalesced and each lane sums its own row left to right (the
// canonical order of DESIGN.md).
#include "mrq_internal.cuh"
#include "mrq_kernels.cuh"

// ----------------------------------------------------------------------- a4
// Seeds S0 and tau0 (decision T; replaces "tau <- threshold of the
// result queue", Alg.2 L9 P:311): the probed lists in probe order until they
// hold >= K' candidates form the pool; S0 = the K' smallest (dis', id) of the
// pool; exact distances ||x_p - q_p||^2 (Alg.2 L14 P:316) of S0; tau0 = K-th
// smallest exact over S0 (+inf if |S0| < K).
template <int W>
__global__ void __launch_bounds__(256) k_seed_w(
    int64_t nq, int aligned, const uint32_t *__restrict__ probe, int np, int K, int Kp, int D, int d, int64_t npad,
    const uint32_t *__restrict__ list_off, const uint32_t *__restrict__ list_size, const uint32_t *__restrict__ ids,
    const uint32_t *__restrict__ codes, const float *__restrict__ f1, const float *__restrict__ f2,
    const float *__restrict__ f3, const float *__restrict__ heads, const float *__restrict__ tails,
    const uint32_t *__restrict__ planes, const double *__restrict__ qconst, const double *__restrict__ qp,
    const double *__restrict__ eps_r_arr, double isd, uint32_t *__restrict__ s0_cnt, uint32_t *__restrict__ s0_pos,
    double *__restrict__ s0_exact, double *__restrict__ tau0)
{
    extern __shared__ unsigned char wsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    const int64_t q = (int64_t)blockIdx.x * wpb + warp;
    if (q >= nq) return;
    float *tile = (float *)wsm + warp * MRQ_RG_FLOATS;
    SelItem *lst = (SelItem *)((float *)wsm + wpb * MRQ_RG_FLOATS) + (size_t)warp * Kp;
    WarpTop top;
    top.init(lst, Kp);
    const double eps_r = eps_r_arr[q];
    const double *qrow = qp + q * D;
    int npool = 0;
    for (int p = 0; p < np && npool < Kp; p++) {
        const uint32_t c = probe[q * np + p];
        if (c == 0xFFFFFFFFu) continue;
        const uint32_t off = list_off[c], sz = list_size[c];
        const uint32_t *pl = planes + (q * np + p) * (MRQ_BQ * W);
        const double *qc = qconst + (q * np + p) * 8;
        for (uint32_t e0 = 0; e0 < sz; e0 += 32) {
            const uint32_t e = e0 + lane;
            const bool v = e < sz;
            SelItem it = sel_inf();
            if (v) {
                const uint32_t slot = off + e;
                uint32_t code[W];
#pragma unroll
                for (int w = 0; w < W; w++) code[w] = codes[(int64_t)w * npad + slot];
                double dis;
                mrq_lb1<W>(code, pl, qc, isd, eps_r, f1[slot], f2[slot], f3[slot], &dis);
                it.key = dis;
                it.id = ids[slot];
                it.pay = slot;
            }
            top.offer(it, v);
        }
        npool += sz;
    }
    const int ns0 = npool < Kp ? npool : Kp;
    // exact distances of S0: HEAD over the head rows, then continued over the tail rows
    warp_rows(aligned, heads, d, 0, d, qrow, ns0, tile, [&](int e) { return lst[e].pay; },
              [&](int) { return 0.0; }, [&](int e, bool v, double acc) {
                  if (v) {
                      s0_pos[q * Kp + e] = lst[e].pay;
                      s0_exact[q * Kp + e] = acc;
                  }
              });
    __syncwarp();
    if (D > d)
        warp_rows(aligned, tails, D - d, 0, D - d, qrow + d, ns0, tile, [&](int e) { return s0_pos[q * Kp + e]; },
                  [&](int e) { return s0_exact[q * Kp + e]; }, [&](int e, bool v, double acc) {
                      if (v) s0_exact[q * Kp + e] = acc;
                  });
    __syncwarp();
    // tau0 = K-th smallest exact over S0
    top.init(lst, K);
    for (int g = 0; g < ns0; g += 32) {
        const int e = g + lane;
        const bool v = e < ns0;
        SelItem it = sel_inf();
        if (v) {
            it.key = s0_exact[q * Kp + e];
            it.id = ids[s0_pos[q * Kp + e]];
            it.pay = e;
        }
        top.offer(it, v);
    }
    if (lane == 0) {
        s0_cnt[q] = ns0;
        tau0[q] = lst[K - 1].key;    // +inf while fewer than K distinct seeds
    }
}

// ----------------------------------------------------------------------- a6
// Stage 2 (Alg.2 L13 P:315; "Optimization" P:327, reading A-7): for every F1
// entry HEAD = ||x_d - q_d||^2 (left to right over i < d) and
// dis_o' = (HEAD + ||x_r||^2) + ||q_r||^2.  TIGHT: S1 = the K' smallest
// (dis_o', id) of F1, their exact distances (HEAD continued over the tail),
// tau1 = K-th smallest distinct exact over S0 u S1; LOOSE: tau1 = tau0.
// F2 = {e in F1 : dis_o' - eps_r < tau1} (FULL), F1 (STAGE1_ONLY / EXACT).
__global__ void __launch_bounds__(256) k_stage2_w(
    int64_t nq, int aligned, int mode, int tight, int K, int Kp, int D, int d, const uint32_t *__restrict__ ids,
    const float *__restrict__ heads, const float *__restrict__ tails, const float *__restrict__ xr2,
    const double *__restrict__ qp, const double *__restrict__ qr2_arr, const double *__restrict__ eps_r_arr,
    const double *__restrict__ tau0_arr, const uint64_t *__restrict__ f1_off, const uint32_t *__restrict__ f1_cnt,
    const uint32_t *__restrict__ f1_pos, double *__restrict__ f1_head, double *__restrict__ f1_diso,
    const uint32_t *__restrict__ s0_cnt, const uint32_t *__restrict__ s0_pos, const double *__restrict__ s0_exact,
    uint32_t *__restrict__ s1_cnt, uint32_t *__restrict__ s1_pos, double *__restrict__ s1_exact,
    double *__restrict__ tau1_arr, uint32_t *__restrict__ f2_cnt, uint32_t *__restrict__ f2_pos,
    double *__restrict__ f2_head)
{
    extern __shared__ unsigned char wsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    const int64_t q = (int64_t)blockIdx.x * wpb + warp;
    if (q >= nq) return;
    float *tile = (float *)wsm + warp * MRQ_RG_FLOATS;
    SelItem *lst = (SelItem *)((float *)wsm + wpb * MRQ_RG_FLOATS) + (size_t)warp * Kp;
    const bool sel1 = mode == 0 && tight;
    WarpTop top;
    top.init(lst, Kp);
    const uint64_t base = f1_off[q];
    const int n1 = (int)f1_cnt[q];
    const double qr2 = qr2_arr[q], eps_r = eps_r_arr[q];
    const double *qrow = qp + q * D;
    warp_rows(aligned, heads, d, 0, d, qrow, n1, tile, [&](int e) { return f1_pos[base + e]; },
              [&](int) { return 0.0; }, [&](int e, bool v, double head) {
                  SelItem it = sel_inf();
                  if (v) {
                      const uint32_t slot = f1_pos[base + e];
                      const double diso = (head + (double)xr2[slot]) + qr2;
                      f1_head[base + e] = head;
                      f1_diso[base + e] = diso;
                      it.key = diso;
                      it.id = ids[slot];
                      it.pay = (uint32_t)e;
                  }
                  if (sel1) top.offer(it, v);
              });
    __syncwarp();
    double tau1 = tau0_arr[q];
    if (sel1) {
        const int ns1 = n1 < Kp ? n1 : Kp;
        for (int e = lane; e < ns1; e += 32) s1_pos[q * Kp + e] = f1_pos[base + lst[e].pay];
        __syncwarp();
        auto s1_init = [&](int e) { return f1_head[base + lst[e].pay]; };
        auto s1_done = [&](int e, bool v, double acc) {
            if (v) s1_exact[q * Kp + e] = acc;
        };
        if (D > d)
            warp_rows(aligned, tails, D - d, 0, D - d, qrow + d, ns1, tile, [&](int e) { return s1_pos[q * Kp + e]; },
                      s1_init, s1_done);
        else
            for (int e = lane; e < ns1; e += 32) s1_exact[q * Kp + e] = s1_init(e);
        __syncwarp();
        // tau1 = K-th smallest distinct exact over S0 u S1 (duplicates dropped by WarpTop)
        top.init(lst, K);
        const int ns0 = (int)s0_cnt[q];
        for (int g = 0; g < ns0 + ns1; g += 32) {
            const int e = g + lane;
            const bool v = e < ns0 + ns1;
            SelItem it = sel_inf();
            if (v) {
                const bool a0 = e < ns0;
                const uint32_t slot = a0 ? s0_pos[q * Kp + e] : s1_pos[q * Kp + (e - ns0)];
                it.key = a0 ? s0_exact[q * Kp + e] : s1_exact[q * Kp + (e - ns0)];
                it.id = ids[slot];
                it.pay = slot;
            }
            top.offer(it, v);
        }
        tau1 = lst[K - 1].key;
        if (lane == 0) s1_cnt[q] = ns1;
    } else if (lane == 0) {
        s1_cnt[q] = 0;
    }
    if (lane == 0) tau1_arr[q] = tau1;
    // F2: ordered compaction (warp-local, no atomics)
    uint32_t at = 0;
    for (int g = 0; g < n1; g += 32) {
        const int e = g + lane;
        bool pass = false;
        if (e < n1) pass = (mode != 0) || (f1_diso[base + e] - eps_r < tau1);
        const unsigned bal = __ballot_sync(0xffffffffu, pass);
        if (pass) {
            const uint32_t o = at + __popc(bal & ((1u << lane) - 1u));
            f2_pos[base + o] = f1_pos[base + e];
            f2_head[base + o] = f1_head[base + e];
        }
        at += __popc(bal);
    }
    if (lane == 0) f2_cnt[q] = at;
}

// ----------------------------------------------------------------------- a7
// Exact re-rank of F2 (Alg.2 L14 P:316): exact = HEAD continued over the
// tail = ||x_p - q_p||^2 left to right over i = 0..D-1 (A-8).
__global__ void __launch_bounds__(256) k_rerank_w(int64_t nq, int aligned, int D, int d, const float *__restrict__ tails,
                                                  const double *__restrict__ qp, const uint64_t *__restrict__ f1_off,
                                                  const uint32_t *__restrict__ f2_cnt,
                                                  const uint32_t *__restrict__ f2_pos,
                                                  const double *__restrict__ f2_head, double *__restrict__ f2_exact)
{
    extern __shared__ unsigned char wsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    const int64_t q = (int64_t)blockIdx.x * wpb + warp;
    if (q >= nq) return;
    float *tile = (float *)wsm + warp * MRQ_RG_FLOATS;
    const uint64_t base = f1_off[q];
    const int n2 = (int)f2_cnt[q];
    const double *qt = qp + q * D + d;
    if (D > d)
        warp_rows(aligned, tails, D - d, 0, D - d, qt, n2, tile, [&](int e) { return f2_pos[base + e]; },
                  [&](int e) { return f2_head[base + e]; }, [&](int e, bool v, double acc) {
                      if (v) f2_exact[base + e] = acc;
                  });
    else
        for (int e = lane; e < n2; e += 32) f2_exact[base + e] = f2_head[base + e];
}

// ----------------------------------------------------------------------- a8
// Per-query top-K (Alg.2 L15-L16): the K smallest (exact, id) over
// the distinct union S0 u S1 u F2 (a candidate in several sets has the same
// exact value in each, so WarpTop drops the copies); ids returned as the
// original int64 index, distances rounded to fp32; padding id -1 / +inf.
__global__ void __launch_bounds__(256) k_topk_w(
    int64_t nq, int K, int Kp, const uint32_t *__restrict__ ids, const uint32_t *__restrict__ s0_cnt,
    const uint32_t *__restrict__ s0_pos, const double *__restrict__ s0_exact, const uint32_t *__restrict__ s1_cnt,
    const uint32_t *__restrict__ s1_pos, const double *__restrict__ s1_exact, const uint64_t *__restrict__ f1_off,
    const uint32_t *__restrict__ f2_cnt, const uint32_t *__restrict__ f2_pos, const double *__restrict__ f2_exact,
    int64_t *__restrict__ out_ids, float *__restrict__ out_dist, uint32_t *__restrict__ exact_cnt)
{
    extern __shared__ unsigned char wsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    const int64_t q = (int64_t)blockIdx.x * wpb + warp;
    if (q >= nq) return;
    SelItem *lst = (SelItem *)wsm + (size_t)warp * K;
    WarpTop top;
    top.init(lst, K);
    const int ns0 = (int)s0_cnt[q], ns1 = (int)s1_cnt[q], n2 = (int)f2_cnt[q];
    const uint64_t base = f1_off[q];
    const int n = ns0 + ns1 + n2;
    for (int g = 0; g < n; g += 32) {
        const int e = g + lane;
        const bool v = e < n;
        SelItem it = sel_inf();
        if (v) {
            uint32_t slot;
            if (e < ns0) {
                slot = s0_pos[q * Kp + e];
                it.key = s0_exact[q * Kp + e];
            } else if (e < ns0 + ns1) {
                slot = s1_pos[q * Kp + (e - ns0)];
                it.key = s1_exact[q * Kp + (e - ns0)];
            } else {
                slot = f2_pos[base + (e - ns0 - ns1)];
                it.key = f2_exact[base + (e - ns0 - ns1)];
            }
            it.id = ids[slot];
            it.pay = slot;
        }
        top.offer(it, v);
    }
    for (int i = lane; i < K; i += 32) {
        const bool ok = lst[i].id != 0xFFFFFFFFu;
        out_ids[q * K + i] = ok ? (int64_t)lst[i].id : (int64_t)-1;
        out_dist[q * K + i] = ok ? (float)lst[i].key : __int_as_float(0x7f800000);
    }
    // distinct exact computations = |S0 u S1 u F2| (S1 and F2 are subsets of F1; S0 may overlap both)
    if (lane == 0) exact_cnt[q] = 0;
    __syncwarp();
    uint32_t dup = 0;
    for (int g = ns0; g < n; g += 32) {
        const int e = g + lane;
        if (e < n) {
            const uint32_t slot = e < ns0 + ns1 ? s1_pos[q * Kp + (e - ns0)] : f2_pos[base + (e - ns0 - ns1)];
            bool d0 = false;
            for (int t = 0; t < ns0; t++) d0 |= s0_pos[q * Kp + t] == slot;
            bool d1 = false;
            if (e >= ns0 + ns1)
                for (int t = 0; t < ns1; t++) d1 |= s1_pos[q * Kp + t] == slot;
            dup += (d0 || d1) ? 1u : 0u;
        }
    }
    for (int o = 16; o > 0; o >>= 1) dup += __shfl_xor_sync(0xffffffffu, dup, o);
    if (lane == 0) exact_cnt[q] = (uint32_t)n - dup;
}

// ---------------------------------------------------------------- launchers
static int warps_for(size_t per_warp)
{
    int w = 4;
    while (w > 1 && per_warp * w > 100 * 1024) w >>= 1;
    return w;
}

static int set_attr(const void *fn, size_t smem)
{
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) {
            mrq_set_error("cudaFuncSetAttribute: %s", cudaGetErrorString(e));
            return MRQ_ECUDA;
        }
    }
    return MRQ_OK;
}

int launch_seed_w(int W, const StageArgs &a, cudaStream_t st)
{
    const size_t per = MRQ_RG_FLOATS * 4 + (size_t)a.Kp * sizeof(SelItem);
    const int wpb = warps_for(per);
    const size_t smem = per * wpb;
    const unsigned grid = (unsigned)((a.nq + wpb - 1) / wpb);
#define MRQ_SEED(WW)                                                                                                \
    do {                                                                                                            \
        int rc = set_attr((const void *)k_seed_w<WW>, smem);                                                        \
        if (rc) return rc;                                                                                          \
        k_seed_w<WW><<<grid, wpb * 32, smem, st>>>(a.nq, a.aligned, a.probe, a.np, a.K, a.Kp, a.D, a.d, a.npad, a.list_off,   \
                                                   a.list_size, a.ids, a.codes, a.f1, a.f2, a.f3, a.heads, a.tails, \
                                                   a.planes, a.qconst, a.qp, a.eps_r, a.isd, a.s0_cnt, a.s0_pos,    \
                                                   a.s0_exact, a.tau0);                                             \
    } while (0)
    switch (W) {
    case 1: MRQ_SEED(1); break;
    case 2: MRQ_SEED(2); break;
    case 3: MRQ_SEED(3); break;
    case 4: MRQ_SEED(4); break;
    case 8: MRQ_SEED(8); break;
    case 16: MRQ_SEED(16); break;
    default: mrq_set_error("unsupported W"); return MRQ_EINVAL;
    }
#undef MRQ_SEED
    return MRQ_OK;
}

int launch_stage2_w(const StageArgs &a, cudaStream_t st)
{
    const size_t per = MRQ_RG_FLOATS * 4 + (size_t)a.Kp * sizeof(SelItem);
    const int wpb = warps_for(per);
    const size_t smem = per * wpb;
    int rc = set_attr((const void *)k_stage2_w, smem);
    if (rc) return rc;
    k_stage2_w<<<(unsigned)((a.nq + wpb - 1) / wpb), wpb * 32, smem, st>>>(
        a.nq, a.aligned, a.mode, a.tight, a.K, a.Kp, a.D, a.d, a.ids, a.heads, a.tails, a.xr2, a.qp, a.qr2, a.eps_r, a.tau0,
        a.f1_off, a.f1_cnt, a.f1_pos, a.f1_head, a.f1_diso, a.s0_cnt, a.s0_pos, a.s0_exact, a.s1_cnt, a.s1_pos,
        a.s1_exact, a.tau1, a.f2_cnt, a.f2_pos, a.f2_head);
    return MRQ_OK;
}

int launch_rerank_w(const StageArgs &a, cudaStream_t st)
{
    const int wpb = 4;
    const size_t smem = (size_t)wpb * MRQ_RG_FLOATS * 4;
    int rc = set_attr((const void *)k_rerank_w, smem);
    if (rc) return rc;
    k_rerank_w<<<(unsigned)((a.nq + wpb - 1) / wpb), wpb * 32, smem, st>>>(a.nq, a.aligned, a.D, a.d, a.tails, a.qp, a.f1_off,
                                                                         a.f2_cnt, a.f2_pos, a.f2_head, a.f2_exact);
    return MRQ_OK;
}

int launch_topk_w(const StageArgs &a, cudaStream_t st)
{
    const size_t per = (size_t)a.K * sizeof(SelItem);
    const int wpb = warps_for(per);
    const size_t smem = per * wpb;
    int rc = set_attr((const void *)k_topk_w, smem);
    if (rc) return rc;
    k_topk_w<<<(unsigned)((a.nq + wpb - 1) / wpb), wpb * 32, smem, st>>>(
        a.nq, a.K, a.Kp, a.ids, a.s0_cnt, a.s0_pos, a.s0_exact, a.s1_cnt, a.s1_pos, a.s1_exact, a.f1_off, a.f2_cnt,
        a.f2_pos, a.f2_exact, a.out_ids, a.out_dist, a.exact_cnt);
    return MRQ_OK;
}

// ----------------------------------------------------------------------- a2
// Exact top-nprobe from a screened distance row (Alg.2 L7), warp per
// query.  Every screen value a_c is within delta_q of an exact-order key
// (||q_d - c||^2 for the CUDA-core screen, ||q_d - c||^2 - ||q_d||^2 for the
// tensor-core screen; the shift is the same for every c), so every member of
// the exact top-np has a_c <= a_(np) + 2 delta_q with a_(np) the np-th
// smallest screen value.  Pass 1 finds a_(np)
// (WarpTop over the row), pass 2 collects {c : a_c <= a_(np) + 2 delta_q},
// pass 3 rescores them in fp64 left to right over i and keeps the np
// smallest (qn2, c).
__global__ void __launch_bounds__(128) k_probe_select_w(
    const float *__restrict__ approx, int64_t nq, int k, int d, int np, const double *__restrict__ qp, int D,
    const double *__restrict__ C, const double *__restrict__ qnorm, double cmax, double kappa,
    uint32_t *__restrict__ cand, uint32_t *__restrict__ probe, double *__restrict__ probe_qn2,
    uint32_t *__restrict__ ncand_out)
{
    extern __shared__ unsigned char wsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    const int64_t q = (int64_t)blockIdx.x * wpb + warp;
    if (q >= nq) return;
    SelItem *lst = (SelItem *)wsm + (size_t)warp * np;
    const float *row = approx + q * k;
    WarpTop top;
    top.init(lst, np);
    for (int c0 = 0; c0 < k; c0 += 32) {
        const int c = c0 + lane;
        SelItem it = sel_inf();
        if (c < k) {
            it.key = (double)row[c];
            it.id = (uint32_t)c;
            it.pay = (uint32_t)c;
        }
        top.offer(it, c < k);
    }
    const double g = qnorm[q] + cmax;
    const double thr = lst[np - 1].key + 2.0 * (kappa * (g * g));
    uint32_t *cq = cand + q * k;
    uint32_t nc = 0;
    for (int c0 = 0; c0 < k; c0 += 32) {
        const int c = c0 + lane;
        const bool in = c < k && (double)row[c] <= thr;
        const unsigned bal = __ballot_sync(0xffffffffu, in);
        if (in) cq[nc + __popc(bal & ((1u << lane) - 1u))] = (uint32_t)c;
        nc += __popc(bal);
    }
    __syncwarp();
    const double *qd = qp + q * D;
    top.init(lst, np);
    for (uint32_t e0 = 0; e0 < nc; e0 += 32) {
        const uint32_t e = e0 + lane;
        SelItem it = sel_inf();
        if (e < nc) {
            const uint32_t c = cq[e];
            const double *cr = C + (int64_t)c * d;
            double acc = 0.0;
            for (int j = 0; j < d; j++) {
                const double t = qd[j] - cr[j];
                acc = acc + t * t;
            }
            it.key = acc;
            it.id = c;
            it.pay = c;
        }
        top.offer(it, e < nc);
    }
    for (int p = lane; p < np; p += 32) {
        const bool ok = lst[p].id != 0xFFFFFFFFu;
        probe[q * np + p] = ok ? lst[p].id : 0xFFFFFFFFu;
        probe_qn2[q * np + p] = ok ? lst[p].key : __longlong_as_double(0x7ff0000000000000ll);
    }
    if (lane == 0) ncand_out[q] = nc;
}

int launch_probe_select_w(const float *approx, int64_t nq, int k, int d, int np, const double *qp, int D,
                          const double *C, const double *qnorm, double cmax, double kappa, uint32_t *cand,
                          uint32_t *probe, double *probe_qn2, uint32_t *ncand, cudaStream_t st)
{
    const int wpb = 4;
    const size_t smem = (size_t)wpb * np * sizeof(SelItem);
    int rc = set_attr((const void *)k_probe_select_w, smem);
    if (rc) return rc;
    k_probe_select_w<<<(unsigned)((nq + wpb - 1) / wpb), wpb * 32, smem, st>>>(
        approx, nq, k, d, np, qp, D, C, qnorm, cmax, kappa, cand, probe, probe_qn2, ncand);
    return MRQ_OK;
}

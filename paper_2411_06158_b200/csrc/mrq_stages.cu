// mrq_stages.cu -- seeds (a4), stage 2 (a6), exact re-rank (a7) and top-K
// (a8): one warp per query.  The selections keep a warp-private sorted top-L
// list in shared memory (WarpTop), so a query's candidates stream through the
// warp once; rows are gathered through per-warp shared-memory stages
// (warp_gather_rows) and each lane sums its own row left to right (the
// canonical order of DESIGN.md).
#include <stdlib.h>

#include <algorithm>

#include "mrq_internal.cuh"
#include "mrq_kernels.cuh"
#include "mrq_probe_tc.cuh"

// ----------------------------------------------------------------------- a4
// Seeds S0 and tau0 (decision T; replaces "tau <- threshold of the
// result queue", Alg.2 L9 P:311): the probed lists in probe order until they
// hold >= K' candidates and number >= seed_lists form the pool; S0 = the K' smallest (dis', id) of the
// pool; exact distances ||x_p - q_p||^2 (Alg.2 L14 P:316) of S0; tau0 = K-th
// smallest exact over S0 (+inf if |S0| < K).
// Short rows (D <= MRQ_SEED_REG_D): the S0 rows (<= K' <= a few dozen) go
// through the register-staged gather (warp_rows_sqdist, a 32 x 33 tile)
// rather than the double-buffered cp.async stages: a third of the shared
// memory per warp, so more one-warp blocks fit on an SM (the kernel is
// latency-bound; shared memory limited it to 18; Deep-shaped 0.251 -> 0.206
// ms).  Long rows keep the cp.async pipeline (GIST-shaped, D = 960: 0.069 vs
// 0.126 ms).
#ifndef MRQ_SEED_REG_D
#define MRQ_SEED_REG_D 256
#endif
#ifndef MRQ_SEED_MINB
#define MRQ_SEED_MINB 32  // one-warp blocks, 32 resident per SM: <= 64 registers (seed 0.134 -> 0.126 ms); 0: plain bounds
#endif
#if MRQ_SEED_MINB > 0   // (short codes only: W > 2 would spill at 64 registers)
#define MRQ_SEED_LB __launch_bounds__(W <= 2 ? 32 : 256, W <= 2 ? MRQ_SEED_MINB : 0)
#else
#define MRQ_SEED_LB __launch_bounds__(256)
#endif
template <int W, bool MG>
__global__ void MRQ_SEED_LB k_seed_w(
    int64_t nq, int aligned, const uint32_t *__restrict__ probe, int np, int K, int Kp, int D, int d, int64_t npad,
    const uint32_t *__restrict__ list_off, const uint32_t *__restrict__ list_size, const uint32_t *__restrict__ ids,
    const uint32_t *__restrict__ codes, const float *__restrict__ f1, const float *__restrict__ f2,
    const float *__restrict__ f3, const float *__restrict__ heads, const float *__restrict__ tails,
    const uint32_t *__restrict__ planes, const double *__restrict__ qconst, const double *__restrict__ qp,
    const double *__restrict__ eps_r_arr, double isd, uint32_t *__restrict__ s0_cnt, uint32_t *__restrict__ s0_pos,
    double *__restrict__ s0_exact, double *__restrict__ tau0, const uint32_t *__restrict__ list_size_g,
    uint32_t *__restrict__ s0_id, XItem *__restrict__ xout, int seed_lists, int aligned_t,
    const uint32_t *__restrict__ qorder)
{
    extern __shared__ unsigned char wsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    const int64_t qi = (int64_t)blockIdx.x * wpb + warp;
    if (qi >= nq) return;
    const int64_t q = qorder ? (int64_t)qorder[qi] : qi;
    // shared memory: [query rows (MRQ_QS(D) doubles per warp)][gather tiles][selection lists]
    double *qs = (double *)wsm + (size_t)warp * MRQ_QS(D);
    const int tilef = D <= MRQ_SEED_REG_D ? 32 * 33 : MRQ_RG_FLOATS;   // per-warp gather tile (floats)
    float *tile = (float *)((double *)wsm + (size_t)wpb * MRQ_QS(D)) + warp * tilef;
    SelItem *lst = (SelItem *)((float *)((double *)wsm + (size_t)wpb * MRQ_QS(D)) + wpb * tilef) +
                   (size_t)warp * MRQ_SELREG(Kp);
    SelItem *queue = lst + Kp;
    if (D <= MRQ_SEED_REG_D) aligned = aligned_t = 0;   // the register-staged gather (warp_rows_sqdist)
    for (int i = lane; i < D; i += 32) qs[i] = qp[q * D + i];   // the query row, read by every gathered row
    __syncwarp();
    const double eps_r = eps_r_arr[q];
    const double *qrow = qs;
    // the pool is defined on GLOBAL list sizes (decision T); a rank scans only
    // the lists it owns (list_size = 0 for the others).  each(it, valid) sees
    // every pool item (dis', id, slot) of this rank, 32 at a time.
    int nloc = 0;
    auto scan_pool = [&](auto each) {
        int64_t npool = 0;
        nloc = 0;
        for (int p = 0; p < np && (npool < Kp || p < seed_lists); p++) {
            const uint32_t c = probe[q * np + p];
            if (c == 0xFFFFFFFFu) continue;
            npool += list_size_g[c];
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
                each(it, v);
            }
            nloc += (int)sz;
        }
    };
    WarpSelT<MG> top;
    top.init(lst, Kp);
    // one pass: items below the running K'-th smallest are queued and merged
    // 32 at a time (bitonic) for K' <= 32; the shared-memory list otherwise
    top.init(lst, Kp, true, queue);
    scan_pool([&](const SelItem &it, bool v) { top.offer(it, v); });
    top.finish();
    const int ns0 = nloc < Kp ? nloc : Kp;
    // exact distances of S0: HEAD over the head rows, then continued over the tail rows
    warp_rows(aligned, heads, d, 0, d, qrow, ns0, tile, [&](int e) { return lst[e].pay; },
              [&](int, uint32_t) { return 0.0; }, [&](int e, bool v, double acc) {
                  if (v) {
                      s0_pos[q * Kp + e] = lst[e].pay;
                      s0_id[q * Kp + e] = lst[e].id;
                      s0_exact[q * Kp + e] = acc;
                  }
              });
    __syncwarp();
    if (D > d)
        warp_rows(aligned_t, tails, D - d, 0, D - d, qrow + d, ns0, tile, [&](int e) { return s0_pos[q * Kp + e]; },
                  [&](int e, uint32_t) { return s0_exact[q * Kp + e]; }, [&](int e, bool v, double acc) {
                      if (v) s0_exact[q * Kp + e] = acc;
                  });
    __syncwarp();
    if (xout) {   // sharded: this rank's part of S0 goes to the exchange (k_xmerge makes S0, tau0)
        for (int e = lane; e < Kp; e += 32) {
            XItem x;
            x.key = e < ns0 ? lst[e].key : __longlong_as_double(0x7ff0000000000000ll);
            x.exact = e < ns0 ? s0_exact[q * Kp + e] : x.key;
            x.id = e < ns0 ? lst[e].id : MRQ_PAD_ID;
            x.slot = e < ns0 ? lst[e].pay : MRQ_PAD_ID;
            xout[q * Kp + e] = x;
        }
        return;
    }
    // tau0 = K-th smallest exact over S0 (distinct items)
    top.init(lst, K, true, queue);
    for (int g = 0; g < ns0; g += 32) {
        const int e = g + lane;
        const bool v = e < ns0;
        SelItem it = sel_inf();
        if (v) {
            it.key = s0_exact[q * Kp + e];
            it.id = s0_id[q * Kp + e];
            it.pay = e;
        }
        top.offer(it, v);
    }
    top.finish();
    if (lane == 0) {
        s0_cnt[q] = ns0;
        tau0[q] = lst[K - 1].key;    // +inf while fewer than K distinct seeds
    }
}

// ------------------------------------------------------------- NOCORR mode
// mode 3: no error-bound correction and no re-rank
// -- the K smallest (dis', id) over every probed candidate, dis' the Eq.4
// estimate (reading R-1) reported as the distance.  Warp per query
// (one-warp blocks); the same epilogue (mrq_lb1) as the scan.  Sharded
// (xout != NULL): the local top-K goes to the exchange (key = exact = dis').
template <int W, bool MG>
__global__ void __launch_bounds__(32) k_nocorr_w(
    int64_t nq, const uint32_t *__restrict__ probe, int np, int K, int64_t npad,
    const uint32_t *__restrict__ list_off, const uint32_t *__restrict__ list_size, const uint32_t *__restrict__ ids,
    const uint32_t *__restrict__ codes, const float *__restrict__ f1, const float *__restrict__ f2,
    const float *__restrict__ f3, const uint32_t *__restrict__ planes, const double *__restrict__ qconst,
    const double *__restrict__ eps_r_arr, double isd, int64_t *__restrict__ out_ids, float *__restrict__ out_dist,
    XItem *__restrict__ xout)
{
    extern __shared__ unsigned char wsm[];
    const int lane = threadIdx.x & 31;
    const int64_t q = blockIdx.x;
    if (q >= nq) return;
    SelItem *lst = (SelItem *)wsm;
    SelItem *queue = lst + K;
    const double eps_r = eps_r_arr[q];
    WarpSelT<MG> top;
    top.init(lst, K, true, queue);
    for (int p = 0; p < np; p++) {
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
    }
    top.finish();
    for (int i = lane; i < K; i += 32) {
        const bool ok = lst[i].id != MRQ_PAD_ID;
        if (xout) {
            XItem x;
            x.key = lst[i].key;
            x.exact = lst[i].key;
            x.id = ok ? lst[i].id : MRQ_PAD_ID;
            x.slot = ok ? lst[i].pay : MRQ_PAD_ID;
            xout[q * K + i] = x;
        } else {
            out_ids[q * K + i] = ok ? (int64_t)lst[i].id : (int64_t)-1;
            out_dist[q * K + i] = ok ? (float)lst[i].key : __int_as_float(0x7f800000);
        }
    }
}

// ----------------------------------------------------------------------- a6
// F2 = {e in F1 : dis_o' - eps_r < tau1} (FULL), all of F1 otherwise:
// ordered warp compaction (no atomics) of the query's F1 segment.
__device__ __forceinline__ void f2_compact(int64_t q, int mode, int n1, uint64_t base, double eps_r, double tau1,
                                           const uint32_t *__restrict__ f1_pos, const double *__restrict__ f1_head,
                                           const double *__restrict__ f1_diso, uint32_t *__restrict__ f2_cnt,
                                           uint32_t *__restrict__ f2_pos, double *__restrict__ f2_head)
{
    const int lane = threadIdx.x & 31;
    uint32_t at = 0;
    for (int g0 = 0; g0 < n1; g0 += 128) {
        double dv[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int e = g0 + 32 * j + lane;
            dv[j] = e < n1 ? f1_diso[base + e] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int e = g0 + 32 * j + lane;
            bool pass = false;
            if (e < n1) pass = (mode != 0) || (dv[j] - eps_r < tau1);
            const unsigned bal = __ballot_sync(0xffffffffu, pass);
            if (pass) {
                const uint32_t o = at + __popc(bal & ((1u << lane) - 1u));
                f2_pos[base + o] = f1_pos[base + e];
                f2_head[base + o] = f1_head[base + e];
            }
            at += __popc(bal);
        }
    }
    if (lane == 0) f2_cnt[q] = at;
}

// With the head sketch (sketch != 0, LOOSE) the scan has already dropped the
// F1 entries whose sketch bound fails the F2 test (k_scan<W, true>): f1_pos
// then holds only the surv_cnt[q] survivors, which are gathered here.
__global__ void __launch_bounds__(128) k_head_b(
    int aligned, int D, int d, const uint32_t *__restrict__ ids, const float *__restrict__ heads,
    const float *__restrict__ xr2, const double *__restrict__ qp, const double *__restrict__ qr2_arr,
    const uint64_t *__restrict__ f1_off, const uint32_t *__restrict__ f1_cnt, const uint32_t *__restrict__ f1_pos,
    double *__restrict__ f1_head, double *__restrict__ f1_diso, uint32_t *__restrict__ f1_id,
    const uint32_t *__restrict__ qorder, int fuse_f2, int mode, const double *__restrict__ eps_r_arr,
    const double *__restrict__ tau0_arr, uint32_t *__restrict__ f2_cnt, uint32_t *__restrict__ f2_pos,
    double *__restrict__ f2_head, uint32_t *__restrict__ s1_cnt, double *__restrict__ tau1_arr, int store_f1,
    int sketch, const uint32_t *__restrict__ surv_cnt)
{
    extern __shared__ unsigned char wsm[];
    __shared__ uint32_t f2n;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    const int64_t q = qorder ? (int64_t)qorder[blockIdx.x] : (int64_t)blockIdx.x;
    float *tile = (float *)wsm + warp * MRQ_RG_FLOATS;
    double *qs = (double *)((float *)wsm + wpb * MRQ_RG_FLOATS);   // q_d staged once per block
    for (int i = threadIdx.x; i < d; i += blockDim.x) qs[i] = qp[q * D + i];
    if (threadIdx.x == 0) f2n = 0;
    __syncthreads();
    const uint64_t base = f1_off[q];
    const int n1 = (int)f1_cnt[q];
    const double qr2 = qr2_arr[q];
    // fused F2 (every schedule but FULL/TIGHT: tau1 = tau0, no S1): the test
    // of f2_compact on the dis_o' just formed, appended unordered (F2 is a set)
    const double eps_r = fuse_f2 ? eps_r_arr[q] : 0.0, tau1 = fuse_f2 ? tau0_arr[q] : 0.0;
    const uint32_t *rows = f1_pos + base;   // the entries whose fp32 head rows are gathered
    int n = n1;
    if (sketch) n = (int)surv_cnt[q];   // the scan kept only the sketch survivors in f1_pos
    float xr2v = 0.f;   // ||x_r||^2, id and slot of the lane's row, loaded while the row is in flight
    uint32_t idv = 0, slotv = 0;
    warp_rows(aligned, heads, d, 0, d, qs, n, tile, [&](int e) { return rows[e]; },
              [&](int, uint32_t slot) {
                  xr2v = xr2[slot];
                  if (store_f1) idv = ids[slot];
                  slotv = slot;
                  return 0.0;
              },
              [&](int e, bool v, double head) {
                  double diso = 0.0;
                  if (v) {
                      diso = (head + (double)xr2v) + qr2;
                      if (store_f1) {   // read only by the S1 selection / F2 compaction of k_stage2_w
                          f1_head[base + e] = head;
                          f1_diso[base + e] = diso;
                          f1_id[base + e] = idv;
                      }
                  }
                  if (fuse_f2) {
                      const bool pass = v && ((mode != 0) || (diso - eps_r < tau1));
                      const unsigned bal = __ballot_sync(0xffffffffu, pass);
                      if (bal) {
                          uint32_t o = 0;
                          if (lane == 0) o = atomicAdd(&f2n, (uint32_t)__popc(bal));
                          o = __shfl_sync(0xffffffffu, o, 0) + __popc(bal & ((1u << lane) - 1u));
                          if (pass) {
                              MRQ_ASSERT(o < (uint32_t)n1);
                              f2_pos[base + o] = slotv;
                              f2_head[base + o] = head;
                          }
                      }
                  }
              },
              warp, wpb);
    if (fuse_f2) {
        __syncthreads();
        if (threadIdx.x == 0) {
            f2_cnt[q] = f2n;
            s1_cnt[q] = 0;
            tau1_arr[q] = tau1;
        }
    }
}

// Stage 2 + exact re-rank + top-K in one block per query (every schedule
// without S1 -- LOOSE, STAGE1_ONLY, EXACT -- and K <= 32): the F2 test of
// k_head_b on the gathered head rows (phase 1), then the block's warps split
// the F2 tail rows (Alg.2 L14 P:316: exact = HEAD continued over the tail,
// left to right, R-8) and each offers its exact distances to a warp top-K
// (phase 2); warp 0 merges the warps' lists with S0 (de-duplicated) into the
// K smallest (exact, id) (Alg.2 L15-L16 P:317-321).  Same sets and values as
// k_head_b + k_topk_w (the F2 exact distances are stored too, f2_exact).  Sharded (xout != NULL): the local top-K goes to the
// exchange.
__global__ void __launch_bounds__(128) k_head_topk(
    int aligned, int aligned_t, int D, int d, int K, int Kp, const uint32_t *__restrict__ ids,
    const float *__restrict__ heads, const float *__restrict__ tails, const float *__restrict__ xr2,
    const double *__restrict__ qp, const double *__restrict__ qr2_arr, const uint64_t *__restrict__ f1_off,
    const uint32_t *__restrict__ f1_cnt, const uint32_t *__restrict__ f1_pos, const uint32_t *__restrict__ qorder,
    int mode, const double *__restrict__ eps_r_arr, const double *__restrict__ tau0_arr,
    uint32_t *__restrict__ f2_cnt, uint32_t *__restrict__ f2_pos, double *__restrict__ f2_head,
    double *__restrict__ f2_exact, uint32_t *__restrict__ s1_cnt, double *__restrict__ tau1_arr, int sketch,
    const uint32_t *__restrict__ surv_cnt,
    const uint32_t *__restrict__ s0_cnt, const uint32_t *__restrict__ s0_pos, const uint32_t *__restrict__ s0_id,
    const double *__restrict__ s0_exact, int64_t *__restrict__ out_ids, float *__restrict__ out_dist,
    XItem *__restrict__ xout)
{
    extern __shared__ unsigned char wsm[];
    __shared__ uint32_t f2n;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    const int64_t q = qorder ? (int64_t)qorder[blockIdx.x] : (int64_t)blockIdx.x;
    // shared memory: [query row][gather tiles][per-warp selection lists + queues][merge list + queue]
    double *qs = (double *)wsm;
    float *tile = (float *)(qs + MRQ_QS(D)) + warp * MRQ_RG_FLOATS;
    SelItem *sel = (SelItem *)((float *)(qs + MRQ_QS(D)) + wpb * MRQ_RG_FLOATS);
    SelItem *lst = sel + (size_t)warp * MRQ_SELREG(K);
    for (int i = threadIdx.x; i < D; i += blockDim.x) qs[i] = qp[q * D + i];
    if (threadIdx.x == 0) f2n = 0;
    __syncthreads();
    const uint64_t base = f1_off[q];
    const int n1 = (int)f1_cnt[q];
    const double qr2 = qr2_arr[q], eps_r = eps_r_arr[q], tau1 = tau0_arr[q];
    // ---- phase 1: HEAD and dis_o' of the (sketch-surviving) F1 rows; the F2 test (Alg.2 L13)
    const uint32_t *rows = f1_pos + base;
    const int n = sketch ? (int)surv_cnt[q] : n1;
    float xr2v = 0.f;
    uint32_t slotv = 0;
    warp_rows(aligned, heads, d, 0, d, qs, n, tile, [&](int e) { return rows[e]; },
              [&](int, uint32_t slot) {
                  xr2v = xr2[slot];
                  slotv = slot;
                  return 0.0;
              },
              [&](int, bool v, double head) {
                  const double diso = (head + (double)xr2v) + qr2;
                  const bool pass = v && ((mode != 0) || (diso - eps_r < tau1));
                  const unsigned bal = __ballot_sync(0xffffffffu, pass);
                  if (bal) {
                      uint32_t o = 0;
                      if (lane == 0) o = atomicAdd(&f2n, (uint32_t)__popc(bal));
                      o = __shfl_sync(0xffffffffu, o, 0) + __popc(bal & ((1u << lane) - 1u));
                      if (pass) {
                          MRQ_ASSERT(o < (uint32_t)n1);
                          f2_pos[base + o] = slotv;
                          f2_head[base + o] = head;
                      }
                  }
              },
              warp, wpb);
    __syncthreads();
    const int n2 = (int)f2n;
    if (threadIdx.x == 0) {
        f2_cnt[q] = n2;
        s1_cnt[q] = 0;
        tau1_arr[q] = tau1;
    }
    // ---- phase 2: exact distances of F2 (the warps split the tail rows), per-warp top-K
    WarpSel top;
    top.init(lst, K, true, lst + K);   // F2 entries are distinct
    uint32_t idv = 0;
    if (D > d) {
        warp_rows(aligned_t, tails, D - d, 0, D - d, qs + d, n2, tile, [&](int e) { return f2_pos[base + e]; },
                  [&](int e, uint32_t slot) {
                      slotv = slot;
                      idv = ids[slot];
                      return f2_head[base + e];
                  },
                  [&](int e, bool v, double ex) {
                      if (v) f2_exact[base + e] = ex;
                      SelItem it;
                      it.key = ex;
                      it.id = idv;
                      it.pay = slotv;
                      top.offer(it, v);
                  },
                  warp, wpb);
    } else {
        for (int g = warp * 32; g < n2; g += wpb * 32) {
            const int e = g + lane;
            SelItem it = sel_inf();
            if (e < n2) {
                it.pay = f2_pos[base + e];
                it.id = ids[it.pay];
                it.key = f2_head[base + e];
                f2_exact[base + e] = it.key;
            }
            top.offer(it, e < n2);
        }
    }
    top.finish();
    __syncthreads();
    if (warp != 0) return;
    // ---- merge: S0 u (the warps' lists), de-duplicated, the K smallest (exact, id)
    SelItem *fl = sel + (size_t)wpb * MRQ_SELREG(K);
    WarpSel fin;
    fin.init(fl, K, false, fl + K);
    const int ns0 = (int)s0_cnt[q];
    for (int g = 0; g < ns0; g += 32) {
        const int e = g + lane;
        SelItem it = sel_inf();
        if (e < ns0) {
            it.key = s0_exact[q * Kp + e];
            it.id = s0_id[q * Kp + e];
            it.pay = s0_pos[q * Kp + e];
        }
        fin.offer(it, e < ns0 && it.pay != MRQ_PAD_ID);
    }
    for (int w = 0; w < wpb; w++) {
        const SelItem *wl = sel + (size_t)w * MRQ_SELREG(K);
        SelItem it = sel_inf();
        if (lane < K) it = wl[lane];
        fin.offer(it, lane < K && it.id != MRQ_PAD_ID);
    }
    fin.finish();
    for (int i = lane; i < K; i += 32) {
        const SelItem x = fl[i];
        if (xout) {
            XItem o;
            o.key = x.key;
            o.exact = x.key;
            o.id = x.id;
            o.slot = x.pay;
            xout[q * K + i] = o;
        } else {
            const bool ok = x.id != 0xFFFFFFFFu;
            out_ids[q * K + i] = ok ? (int64_t)x.id : (int64_t)-1;
            out_dist[q * K + i] = ok ? (float)x.key : __int_as_float(0x7f800000);
        }
    }
}

// Stage 2, decision half, warp per query.  TIGHT: S1 = the K' smallest
// (dis_o', id) of F1, their exact distances (HEAD continued over the tail),
// tau1 = K-th smallest distinct exact over S0 u S1; LOOSE: tau1 = tau0.
// F2 as in f2_compact.  Sharded TIGHT (xout != NULL): the local S1 goes to
// the exchange and k_xmerge / k_f2_w finish tau1 and F2.
template <bool MG>
__global__ void __launch_bounds__(256) k_stage2_w(
    int64_t nq, int aligned, int mode, int tight, int K, int Kp, int D, int d, const float *__restrict__ tails,
    const double *__restrict__ qp, const double *__restrict__ eps_r_arr, const double *__restrict__ tau0_arr,
    const uint64_t *__restrict__ f1_off, const uint32_t *__restrict__ f1_cnt, const uint32_t *__restrict__ f1_pos,
    const double *__restrict__ f1_head, const double *__restrict__ f1_diso, const uint32_t *__restrict__ f1_id,
    const uint32_t *__restrict__ s0_cnt, const uint32_t *__restrict__ s0_id, const double *__restrict__ s0_exact,
    uint32_t *__restrict__ s1_cnt, uint32_t *__restrict__ s1_pos, uint32_t *__restrict__ s1_id,
    double *__restrict__ s1_exact, double *__restrict__ tau1_arr, uint32_t *__restrict__ f2_cnt,
    uint32_t *__restrict__ f2_pos, double *__restrict__ f2_head, XItem *__restrict__ xout,
    const uint32_t *__restrict__ qorder)
{
    extern __shared__ unsigned char wsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    const int64_t qi = (int64_t)blockIdx.x * wpb + warp;
    if (qi >= nq) return;
    const int64_t q = qorder ? (int64_t)qorder[qi] : qi;
    // shared memory: [query rows (MRQ_QS(D) doubles per warp)][gather tiles][selection lists]
    double *qs = (double *)wsm + (size_t)warp * MRQ_QS(D);
    float *tile = (float *)((double *)wsm + (size_t)wpb * MRQ_QS(D)) + warp * MRQ_RG_FLOATS;
    SelItem *lst = (SelItem *)((float *)((double *)wsm + (size_t)wpb * MRQ_QS(D)) + wpb * MRQ_RG_FLOATS) +
                   (size_t)warp * MRQ_SELREG(Kp);
    SelItem *queue = lst + Kp;
    for (int i = lane; i < D; i += 32) qs[i] = qp[q * D + i];   // the query row, read by every gathered row
    __syncwarp();
    const bool sel1 = mode == 0 && tight;
    const uint64_t base = f1_off[q];
    const int n1 = (int)f1_cnt[q];
    const double eps_r = eps_r_arr[q];
    const double *qrow = qs;
    double tau1 = tau0_arr[q];
    if (sel1) {
        WarpSelT<MG> top;
        top.init(lst, Kp);
        // each(it, valid) over F1: (dis_o', id, entry), 128 entries per round
        auto scan_f1 = [&](auto each) {
            for (int g0 = 0; g0 < n1; g0 += 128) {
                double kv[4];
                uint32_t iv[4];
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const int e = g0 + 32 * j + lane;
                    kv[j] = e < n1 ? f1_diso[base + e] : 0.0;
                    iv[j] = e < n1 ? f1_id[base + e] : 0u;
                }
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const int e = g0 + 32 * j + lane;
                    SelItem it;
                    it.key = kv[j];
                    it.id = iv[j];
                    it.pay = (uint32_t)e;
                    each(it, e < n1);
                }
            }
        };
        if (Kp <= 32) {
            // two passes: U = Kp-th smallest lane minimum bounds the Kp-th
            // smallest dis_o' from above, so only items <= U can enter S1
            double mn = __longlong_as_double(0x7ff0000000000000ll);
            scan_f1([&](const SelItem &it, bool v) {
                if (v) mn = fmin(mn, it.key);
            });
            const double U = warp_kth_smallest(mn, Kp);
            top.init(lst, Kp, true, queue);
            scan_f1([&](const SelItem &it, bool v) { top.offer(it, v && it.key <= U); });
        } else {
            top.init(lst, Kp, true, queue);
            scan_f1([&](const SelItem &it, bool v) { top.offer(it, v); });
        }
        top.finish();
        const int ns1 = n1 < Kp ? n1 : Kp;
        for (int e = lane; e < ns1; e += 32) {
            s1_pos[q * Kp + e] = f1_pos[base + lst[e].pay];
            s1_id[q * Kp + e] = lst[e].id;
        }
        __syncwarp();
        auto s1_init = [&](int e, uint32_t) { return f1_head[base + lst[e].pay]; };
        auto s1_done = [&](int e, bool v, double acc) {
            if (v) s1_exact[q * Kp + e] = acc;
        };
        if (D > d)
            warp_rows(aligned, tails, D - d, 0, D - d, qrow + d, ns1, tile, [&](int e) { return s1_pos[q * Kp + e]; },
                      s1_init, s1_done);
        else
            for (int e = lane; e < ns1; e += 32) s1_exact[q * Kp + e] = s1_init(e, 0u);
        __syncwarp();
        if (xout) {   // sharded TIGHT: exchange the local S1
            for (int e = lane; e < Kp; e += 32) {
                XItem x;
                x.key = e < ns1 ? lst[e].key : __longlong_as_double(0x7ff0000000000000ll);
                x.exact = e < ns1 ? s1_exact[q * Kp + e] : x.key;
                x.id = e < ns1 ? lst[e].id : MRQ_PAD_ID;
                x.slot = e < ns1 ? s1_pos[q * Kp + e] : MRQ_PAD_ID;
                xout[q * Kp + e] = x;
            }
            return;
        }
        // tau1 = K-th smallest distinct exact over S0 u S1 (duplicates dropped by the selection)
        top.init(lst, K, false, queue);
        const int ns0 = (int)s0_cnt[q];
        for (int g = 0; g < ns0 + ns1; g += 32) {
            const int e = g + lane;
            const bool v = e < ns0 + ns1;
            SelItem it = sel_inf();
            if (v) {
                const bool a0 = e < ns0;
                it.key = a0 ? s0_exact[q * Kp + e] : s1_exact[q * Kp + (e - ns0)];
                it.id = a0 ? s0_id[q * Kp + e] : s1_id[q * Kp + (e - ns0)];
                it.pay = (uint32_t)e;
            }
            top.offer(it, v);
        }
        top.finish();
        tau1 = lst[K - 1].key;
        if (lane == 0) s1_cnt[q] = ns1;
    } else if (lane == 0) {
        s1_cnt[q] = 0;
    }
    if (lane == 0) tau1_arr[q] = tau1;
    f2_compact(q, mode, n1, base, eps_r, tau1, f1_pos, f1_head, f1_diso, f2_cnt, f2_pos, f2_head);
}

// F2 after a sharded tau1 exchange (warp per query).
__global__ void __launch_bounds__(256) k_f2_w(int64_t nq, int mode, const double *__restrict__ eps_r_arr,
                                              const double *__restrict__ tau1_arr, const uint64_t *__restrict__ f1_off,
                                              const uint32_t *__restrict__ f1_cnt, const uint32_t *__restrict__ f1_pos,
                                              const double *__restrict__ f1_head, const double *__restrict__ f1_diso,
                                              uint32_t *__restrict__ f2_cnt, uint32_t *__restrict__ f2_pos,
                                              double *__restrict__ f2_head)
{
    const int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (q >= nq) return;
    f2_compact(q, mode, (int)f1_cnt[q], f1_off[q], eps_r_arr[q], tau1_arr[q], f1_pos, f1_head, f1_diso, f2_cnt,
               f2_pos, f2_head);
}

// ----------------------------------------------------------------------- a8
// Exact re-rank of F2 (a7) and per-query top-K (Alg.2 L15-L16),
// block per query: F2's tails are gathered first (f2_exact), then the K
// smallest (exact, id) over
// the distinct union S0 u S1 u F2 restricted to this rank's slots (a
// candidate in several sets has the same exact value in each, so WarpTop
// drops the copies; members of the global S0/S1 owned by another rank carry
// slot PAD and are skipped).  ids are returned as the original int64 index,
// distances rounded to fp32, padding id -1 / +inf.  Sharded (xout != NULL):
// the local top-K (exact fp64, id) goes to the exchange and k_xmerge writes
// the outputs.
// Block per query (MRQ_TOPK_WPB warps split the F2 re-rank rows, warp 0
// selects; 1 measured best once the query row is staged in shared memory).
template <bool MG>
__global__ void __launch_bounds__(64) k_topk_w(
    int64_t nq, int K, int Kp, const uint32_t *__restrict__ ids, const uint32_t *__restrict__ s0_cnt,
    const uint32_t *__restrict__ s0_pos, const uint32_t *__restrict__ s0_id, const double *__restrict__ s0_exact,
    const uint32_t *__restrict__ s1_cnt, const uint32_t *__restrict__ s1_pos, const uint32_t *__restrict__ s1_id,
    const double *__restrict__ s1_exact, const uint64_t *__restrict__ f1_off, const uint32_t *__restrict__ f2_cnt,
    const uint32_t *__restrict__ f2_pos, double *__restrict__ f2_exact, int64_t *__restrict__ out_ids,
    float *__restrict__ out_dist, XItem *__restrict__ xout, int aligned, int D,
    int d, const float *__restrict__ tails, const double *__restrict__ qp, const double *__restrict__ f2_head,
    const uint32_t *__restrict__ qorder)
{
    extern __shared__ unsigned char wsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    const int64_t q = qorder ? (int64_t)qorder[blockIdx.x] : (int64_t)blockIdx.x;
    // shared memory: [query tail][gather tiles][selection list]
    double *qs = (double *)wsm;
    float *tile = (float *)(qs + MRQ_QS(D)) + warp * MRQ_RG_FLOATS;
    SelItem *lst = (SelItem *)((float *)(qs + MRQ_QS(D)) + wpb * MRQ_RG_FLOATS);
    SelItem *queue = lst + K;
    for (int i = d + threadIdx.x; i < D; i += blockDim.x) qs[i] = qp[q * D + i];
    __syncthreads();
    const int ns0 = (int)s0_cnt[q], ns1 = (int)s1_cnt[q], n2 = (int)f2_cnt[q];
    const uint64_t base = f1_off[q];
    // a7 exact re-rank of F2 (Alg.2 L14 P:316): exact = HEAD continued over
    // the tail = ||x_p - q_p||^2 left to right over i = 0..D-1 (R-8)
    // (the block's warps split the F2 rows; warp 0 then selects)
    if (D > d)
        warp_rows(aligned, tails, D - d, 0, D - d, qs + d, n2, tile, [&](int e) { return f2_pos[base + e]; },
                  [&](int e, uint32_t) { return f2_head[base + e]; }, [&](int e, bool v, double acc) {
                      if (v) f2_exact[base + e] = acc;
                  }, warp, wpb);
    else
        for (int e = threadIdx.x; e < n2; e += blockDim.x) f2_exact[base + e] = f2_head[base + e];
    __syncthreads();
    if (warp != 0) return;
    WarpSelT<MG> top;
    top.init(lst, K, false, queue);
    const int n = ns0 + ns1 + n2;
    for (int g = 0; g < n; g += 32) {
        const int e = g + lane;
        bool v = e < n;
        SelItem it = sel_inf();
        if (v) {
            uint32_t slot;
            if (e < ns0) {
                slot = s0_pos[q * Kp + e];
                it.key = s0_exact[q * Kp + e];
                it.id = s0_id[q * Kp + e];
            } else if (e < ns0 + ns1) {
                slot = s1_pos[q * Kp + (e - ns0)];
                it.key = s1_exact[q * Kp + (e - ns0)];
                it.id = s1_id[q * Kp + (e - ns0)];
            } else {
                slot = f2_pos[base + (e - ns0 - ns1)];
                it.key = f2_exact[base + (e - ns0 - ns1)];
                it.id = ids[slot];
            }
            it.pay = slot;
            v = slot != MRQ_PAD_ID;
            if (!v) it = sel_inf();
        }
        top.offer(it, v);
    }
    top.finish();
    if (xout) {
        for (int i = lane; i < K; i += 32) {
            XItem x;
            x.key = lst[i].key;
            x.exact = lst[i].key;
            x.id = lst[i].id;
            x.slot = lst[i].pay;
            xout[q * K + i] = x;
        }
    } else {
        for (int i = lane; i < K; i += 32) {
            const bool ok = lst[i].id != 0xFFFFFFFFu;
            out_ids[q * K + i] = ok ? (int64_t)lst[i].id : (int64_t)-1;
            out_dist[q * K + i] = ok ? (float)lst[i].key : __int_as_float(0x7f800000);
        }
    }
}

// Statistic (stats requested only, after the timed stages): distinct exact
// computations on this rank = |(S0 u S1 u F2) n owned| (S1 and F2 are
// subsets of F1; S0 may overlap both).  Warp per query.
__global__ void __launch_bounds__(256) k_exact_count_w(int64_t nq, int Kp, const uint32_t *__restrict__ s0_cnt,
                                                       const uint32_t *__restrict__ s0_pos,
                                                       const uint32_t *__restrict__ s1_cnt,
                                                       const uint32_t *__restrict__ s1_pos,
                                                       const uint64_t *__restrict__ f1_off,
                                                       const uint32_t *__restrict__ f2_cnt,
                                                       const uint32_t *__restrict__ f2_pos, uint32_t *__restrict__ exact_cnt)
{
    const int lane = threadIdx.x & 31;
    const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (q >= nq) return;
    const int ns0 = (int)s0_cnt[q], ns1 = (int)s1_cnt[q], n2 = (int)f2_cnt[q];
    const uint64_t base = f1_off[q];
    const int n = ns0 + ns1 + n2;
    uint32_t cnt = 0;
    for (int g = 0; g < n; g += 32) {
        const int e = g + lane;
        if (e < n) {
            const uint32_t slot = e < ns0 ? s0_pos[q * Kp + e]
                                  : e < ns0 + ns1 ? s1_pos[q * Kp + (e - ns0)] : f2_pos[base + (e - ns0 - ns1)];
            bool dup = slot == MRQ_PAD_ID;
            if (e >= ns0)
                for (int t = 0; t < ns0 && !dup; t++) dup = s0_pos[q * Kp + t] == slot;
            if (e >= ns0 + ns1)
                for (int t = 0; t < ns1 && !dup; t++) dup = s1_pos[q * Kp + t] == slot;
            cnt += dup ? 0u : 1u;
        }
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) exact_cnt[q] = cnt;
}

// ----------------------------------------------------------------------- a9
// Merge of an all-gather, warp per query.  recv holds, rank
// major, every rank's L items of every query: recv[(r * nq + q) * L + j].
// The L smallest (key, id) of the union are kept (ids are distinct across
// ranks: each vector lives on one rank).
//   kind 0 (seeds):  global S0 (key = dis') and tau0 = K-th smallest exact
//   kind 1 (S1):     global S1 (key = dis_o') and tau1 = K-th smallest
//                    distinct exact over S0 u S1
//   kind 2 (final):  top-K (key = exact) -> out_ids / out_dist
// Slots of items that came from another rank become PAD.
template <bool MG>
__global__ void __launch_bounds__(128) k_xmerge(int kind, int64_t nq, int world, int rank, int L, int K, int Kp,
                                                const XItem *__restrict__ recv, uint32_t *__restrict__ s_cnt,
                                                uint32_t *__restrict__ s_pos, uint32_t *__restrict__ s_id,
                                                double *__restrict__ s_exact, double *__restrict__ tau,
                                                const uint32_t *__restrict__ s0_cnt, const uint32_t *__restrict__ s0_id,
                                                const double *__restrict__ s0_exact, int64_t *__restrict__ out_ids,
                                                float *__restrict__ out_dist)
{
    extern __shared__ unsigned char wsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    const int64_t q = (int64_t)blockIdx.x * wpb + warp;
    if (q >= nq) return;
    SelItem *lst = (SelItem *)wsm + (size_t)warp * MRQ_SELREG(L);
    SelItem *queue = lst + L;
    WarpSelT<MG> top;
    top.init(lst, L, true, queue);
    for (int r = 0; r < world; r++) {
        const XItem *src = recv + ((int64_t)r * nq + q) * L;
        for (int j0 = 0; j0 < L; j0 += 32) {
            const int j = j0 + lane;
            SelItem it = sel_inf();
            bool v = false;
            if (j < L) {
                const XItem x = src[j];
                v = x.id != MRQ_PAD_ID;
                if (v) {
                    it.key = x.key;
                    it.id = x.id;
                    it.pay = (uint32_t)(r * L + j);
                }
            }
            top.offer(it, v);
        }
    }
    top.finish();
    if (kind == 2) {
        for (int i = lane; i < K; i += 32) {
            const bool ok = lst[i].id != MRQ_PAD_ID;
            double ex = 0.0;
            if (ok) {
                const uint32_t pay = lst[i].pay;
                ex = recv[((int64_t)(pay / L) * nq + q) * L + pay % L].exact;
            }
            out_ids[q * K + i] = ok ? (int64_t)lst[i].id : (int64_t)-1;
            out_dist[q * K + i] = ok ? (float)ex : __int_as_float(0x7f800000);
        }
        return;
    }
    int n = 0;
    for (int j0 = 0; j0 < L; j0 += 32) n += __popc(__ballot_sync(0xffffffffu, j0 + lane < L && lst[j0 + lane].id != MRQ_PAD_ID));
    for (int e = lane; e < n; e += 32) {
        const uint32_t pay = lst[e].pay;
        const int r = (int)(pay / L);
        const XItem x = recv[((int64_t)r * nq + q) * L + pay % L];
        s_exact[q * Kp + e] = x.exact;
        s_id[q * Kp + e] = x.id;
        s_pos[q * Kp + e] = r == rank ? x.slot : MRQ_PAD_ID;
    }
    __syncwarp();
    // tau = K-th smallest distinct exact over S0 (kind 0) or S0 u S1 (kind 1)
    top.init(lst, K, false, queue);
    const int n0 = kind == 1 ? (int)s0_cnt[q] : 0;
    for (int g = 0; g < n0 + n; g += 32) {
        const int e = g + lane;
        const bool v = e < n0 + n;
        SelItem it = sel_inf();
        if (v) {
            const bool a0 = e < n0;
            it.key = a0 ? s0_exact[q * Kp + e] : s_exact[q * Kp + (e - n0)];
            it.id = a0 ? s0_id[q * Kp + e] : s_id[q * Kp + (e - n0)];
            it.pay = (uint32_t)e;
        }
        top.offer(it, v);
    }
    top.finish();
    if (lane == 0) {
        s_cnt[q] = (uint32_t)n;
        tau[q] = lst[K - 1].key;
    }
}

// ---------------------------------------------------------------- launchers
#ifndef MRQ_WPB_MAX
#define MRQ_WPB_MAX 1   // one warp (query) per block measured best of 1/2/4/8 for seed / stage 2 / merge
#endif
static int warps_for(size_t per_warp)
{
    int w = MRQ_WPB_MAX;
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
    const size_t per = (size_t)MRQ_QS(a.D) * 8 + (size_t)(a.D <= MRQ_SEED_REG_D ? 32 * 33 : MRQ_RG_FLOATS) * 4 +
                       (size_t)MRQ_SELREG(a.Kp) * sizeof(SelItem);
    const int wpb = warps_for(per);
    const size_t smem = per * wpb;
    const unsigned grid = (unsigned)((a.nq + wpb - 1) / wpb);
    const bool mg = a.Kp > MRQ_MERGE_MIN;
#define MRQ_SEED(WW)                                                                                                \
    do {                                                                                                            \
        auto fn = mg ? k_seed_w<WW, true> : k_seed_w<WW, false>;                                                    \
        int rc = set_attr((const void *)fn, smem);                                                                  \
        if (rc) return rc;                                                                                          \
        fn<<<grid, wpb * 32, smem, st>>>(a.nq, a.aligned, a.probe, a.np, a.K, a.Kp, a.D, a.d, a.npad, a.list_off,   \
                                                   a.list_size, a.ids, a.codes, a.f1, a.f2, a.f3, a.heads, a.tails, \
                                                   a.planes, a.qconst, a.qp, a.eps_r, a.isd, a.s0_cnt, a.s0_pos,    \
                                                   a.s0_exact, a.tau0, a.list_size_g, a.s0_id, a.xout,              \
                                                   a.seed_lists, a.aligned_tails, a.qorder);                        \
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

int launch_nocorr_w(int W, const StageArgs &a, cudaStream_t st)
{
    const size_t smem = (size_t)MRQ_SELREG(a.K) * sizeof(SelItem);
    const bool mg = a.K > MRQ_MERGE_MIN;
#define MRQ_NOC(WW)                                                                                              \
    do {                                                                                                         \
        auto fn = mg ? k_nocorr_w<WW, true> : k_nocorr_w<WW, false>;                                             \
        int rc = set_attr((const void *)fn, smem);                                                               \
        if (rc) return rc;                                                                                       \
        fn<<<(unsigned)a.nq, 32, smem, st>>>(a.nq, a.probe, a.np, a.K, a.npad, a.list_off, a.list_size, a.ids,  \
                                             a.codes, a.f1, a.f2, a.f3, a.planes, a.qconst, a.eps_r, a.isd,     \
                                             a.out_ids, a.out_dist, a.xout);                                    \
    } while (0)
    switch (W) {
    case 1: MRQ_NOC(1); break;
    case 2: MRQ_NOC(2); break;
    case 3: MRQ_NOC(3); break;
    case 4: MRQ_NOC(4); break;
    case 8: MRQ_NOC(8); break;
    case 16: MRQ_NOC(16); break;
    default: mrq_set_error("unsupported W"); return MRQ_EINVAL;
    }
#undef MRQ_NOC
    return MRQ_OK;
}

int launch_stage2_w(const StageArgs &a, cudaStream_t st, cudaEvent_t after_gather)
{
    // without an S1 selection (every schedule but FULL/TIGHT) stage 2 is the
    // F2 test alone, done inside the head gather
    const int fuse = !(a.mode == 0 && a.tight);
    {   // gather half: block per query, its 4 warps split the F1 rows (4 measured best of 2/4/8)
#ifndef MRQ_HEAD_WPB
#define MRQ_HEAD_WPB 4   // measured best of 2/4/8 (launch bounds 128)
#endif
        const int wpb = MRQ_HEAD_WPB;
        const bool sk = mrq_sketch_used(a);
        const size_t smem = (size_t)wpb * MRQ_RG_FLOATS * 4 + (size_t)a.d * 8;
        int rc = set_attr((const void *)k_head_b, smem);
        if (rc) return rc;
        k_head_b<<<(unsigned)a.nq, wpb * 32, smem, st>>>(a.aligned, a.D, a.d, a.ids, a.heads, a.xr2, a.qp, a.qr2,
                                                          a.f1_off, a.f1_cnt, a.f1_pos, a.f1_head, a.f1_diso, a.f1_id,
                                                          a.qorder, fuse, a.mode, a.eps_r, a.tau0, a.f2_cnt, a.f2_pos,
                                                          a.f2_head, a.s1_cnt, a.tau1, !fuse || a.store_f1, sk ? 1 : 0,
                                                          a.surv_cnt);
    }
    if (after_gather) MRQ_CUDA_TRY(cudaEventRecord(after_gather, st));
    if (fuse) return MRQ_OK;   // F2 written by the gather kernel
    const size_t per = (size_t)MRQ_QS(a.D) * 8 + MRQ_RG_FLOATS * 4 +
                       (size_t)MRQ_SELREG(std::max(a.Kp, a.K)) * sizeof(SelItem);
    const int wpb = warps_for(per);
    const size_t smem = per * wpb;
    auto fn = std::max(a.Kp, a.K) > MRQ_MERGE_MIN ? k_stage2_w<true> : k_stage2_w<false>;
    int rc = set_attr((const void *)fn, smem);
    if (rc) return rc;
    fn<<<(unsigned)((a.nq + wpb - 1) / wpb), wpb * 32, smem, st>>>(
        a.nq, a.aligned_tails, a.mode, a.tight, a.K, a.Kp, a.D, a.d, a.tails, a.qp, a.eps_r, a.tau0, a.f1_off, a.f1_cnt,
        a.f1_pos, a.f1_head, a.f1_diso, a.f1_id, a.s0_cnt, a.s0_id, a.s0_exact, a.s1_cnt, a.s1_pos, a.s1_id,
        a.s1_exact, a.tau1, a.f2_cnt, a.f2_pos, a.f2_head, a.xout, a.qorder);
    return MRQ_OK;
}

bool mrq_head_topk_used(const StageArgs &a)
{
    return !(a.mode == 0 && a.tight) && a.K <= 32 && !a.store_f1 && a.fuse_topk;
}

int launch_head_topk(const StageArgs &a, cudaStream_t st)
{
    const int wpb = MRQ_HEAD_WPB;
    const size_t smem = (size_t)MRQ_QS(a.D) * 8 + (size_t)wpb * MRQ_RG_FLOATS * 4 +
                        (size_t)(wpb + 1) * MRQ_SELREG(a.K) * sizeof(SelItem);
    int rc = set_attr((const void *)k_head_topk, smem);
    if (rc) return rc;
    const bool sk = mrq_sketch_used(a);
    k_head_topk<<<(unsigned)a.nq, wpb * 32, smem, st>>>(
        a.aligned, a.aligned_tails, a.D, a.d, a.K, a.Kp, a.ids, a.heads, a.tails, a.xr2, a.qp, a.qr2, a.f1_off,
        a.f1_cnt, a.f1_pos, a.qorder, a.mode, a.eps_r, a.tau0, a.f2_cnt, a.f2_pos, a.f2_head, a.f2_exact, a.s1_cnt,
        a.tau1,
        sk ? 1 : 0, a.surv_cnt, a.s0_cnt, a.s0_pos, a.s0_id, a.s0_exact, a.out_ids, a.out_dist, a.xout);
    return MRQ_OK;
}

int launch_f2_w(const StageArgs &a, cudaStream_t st)
{
    k_f2_w<<<(unsigned)((a.nq + 7) / 8), 256, 0, st>>>(a.nq, a.mode, a.eps_r, a.tau1, a.f1_off, a.f1_cnt, a.f1_pos,
                                                       a.f1_head, a.f1_diso, a.f2_cnt, a.f2_pos, a.f2_head);
    return MRQ_OK;
}

int launch_xmerge(int kind, const StageArgs &a, int world, int rank, const XItem *recv, cudaStream_t st)
{
    const int L = kind == 2 ? a.K : a.Kp;
    const size_t per = (size_t)MRQ_SELREG(std::max(L, a.K)) * sizeof(SelItem);
    const int wpb = warps_for(per);
    const size_t smem = per * wpb;
    auto fn = std::max(L, a.K) > MRQ_MERGE_MIN ? k_xmerge<true> : k_xmerge<false>;
    int rc = set_attr((const void *)fn, smem);
    if (rc) return rc;
    uint32_t *cnt = kind == 0 ? a.s0_cnt : a.s1_cnt;
    uint32_t *pos = kind == 0 ? a.s0_pos : a.s1_pos;
    uint32_t *sid = kind == 0 ? a.s0_id : a.s1_id;
    double *ex = kind == 0 ? a.s0_exact : a.s1_exact;
    double *tau = kind == 0 ? a.tau0 : a.tau1;
    fn<<<(unsigned)((a.nq + wpb - 1) / wpb), wpb * 32, smem, st>>>(kind, a.nq, world, rank, L, a.K, a.Kp, recv,
                                                                        cnt, pos, sid, ex, tau, a.s0_cnt, a.s0_id,
                                                                        a.s0_exact, a.out_ids, a.out_dist);
    return MRQ_OK;
}

int launch_exact_count(const StageArgs &a, cudaStream_t st)
{
    k_exact_count_w<<<(unsigned)((a.nq + 7) / 8), 256, 0, st>>>(a.nq, a.Kp, a.s0_cnt, a.s0_pos, a.s1_cnt, a.s1_pos,
                                                                a.f1_off, a.f2_cnt, a.f2_pos, a.exact_cnt);
    return MRQ_OK;
}

int launch_topk_w(const StageArgs &a, cudaStream_t st)
{
#ifndef MRQ_TOPK_WPB
#define MRQ_TOPK_WPB 1   // with the query row in shared memory one warp beats 2 (LOOSE 0.177 -> 0.149 ms)
#endif
    const int wpb = MRQ_TOPK_WPB;
    const size_t smem =
        (size_t)MRQ_QS(a.D) * 8 + (size_t)wpb * MRQ_RG_FLOATS * 4 + (size_t)MRQ_SELREG(a.K) * sizeof(SelItem);
    auto fn = a.K > MRQ_MERGE_MIN ? k_topk_w<true> : k_topk_w<false>;
    int rc = set_attr((const void *)fn, smem);
    if (rc) return rc;
    fn<<<(unsigned)a.nq, wpb * 32, smem, st>>>(
        a.nq, a.K, a.Kp, a.ids, a.s0_cnt, a.s0_pos, a.s0_id, a.s0_exact, a.s1_cnt, a.s1_pos, a.s1_id, a.s1_exact,
        a.f1_off, a.f2_cnt, a.f2_pos, a.f2_exact, a.out_ids, a.out_dist, a.xout, a.aligned_tails, a.D,
        a.d, a.tails, a.qp, a.f2_head, a.qorder);
    return MRQ_OK;
}

// ----------------------------------------------------------------------- a2
// Exact top-nprobe from a screened distance row (Alg.2 L7), warp per
// query.  Every screen value a_c is within delta_q of an exact-order key
// (||q_d - c||^2 for the CUDA-core screen, ||q_d - c||^2 - ||q_d||^2 for the
// tensor-core screen; the shift is the same for every c), so every member of
// the exact top-np has a_c <= a_(np) + 2 delta_q, where a_(np) is the np-th
// smallest screen value.
//   1. Each lane keeps the M = ceil(np/32) smallest of its strided share of
//      the row (registers).  U = the np-th smallest of these 32 M values
//      (radix select on order-preserving u32 keys, ballot counts) is >= a_(np):
//      at least np row values are <= U.
//   2. C = {c : a_c <= U + 2 delta_q} is a superset of the margin set
//      {c : a_c <= a_(np) + 2 delta_q} (ballot compaction into cand[q]).
//   3. C is rescored in fp64 left to right over i; the np smallest (qn2, c) are kept.
template <int M>
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
    SelItem *lst = (SelItem *)wsm + (size_t)warp * MRQ_SELREG(np);
    SelItem *queue = lst + np;
    const float *row = approx + q * k;
    const float FINF = __int_as_float(0x7f800000);
    // 1. lane-local M smallest (sorted ascending in registers)
    float loc[M];
#pragma unroll
    for (int j = 0; j < M; j++) loc[j] = FINF;
    for (int c0 = 0; c0 < k; c0 += 128) {
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int c = c0 + 32 * u + lane;
            v[u] = c < k ? __ldg(row + c) : FINF;
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
            float x = v[u];
            if (x < loc[M - 1]) {
#pragma unroll
                for (int j = 0; j < M; j++) {   // insertion by compare-exchange
                    const float lo = fminf(loc[j], x);
                    x = fmaxf(loc[j], x);
                    loc[j] = lo;
                }
            }
        }
    }
    // np-th smallest key of the 32 M lane-local values
    uint32_t key[M];
#pragma unroll
    for (int j = 0; j < M; j++) key[j] = f2key(loc[j]);
    uint32_t res = 0;
    for (int bit = 31; bit >= 0; bit--) {
        const uint32_t t = res | (1u << bit);
        int cnt = 0;
#pragma unroll
        for (int j = 0; j < M; j++) cnt += __popc(__ballot_sync(0xffffffffu, key[j] < t));
        if (cnt < np) res = t;
    }
    const float U = key2f(res);
    const double g = qnorm[q] + cmax;
    const double margin = 2.0 * (kappa * (g * g));
    // 2. C
    uint32_t *cq = cand + q * k;
    const double t1 = (double)U + margin;
    uint32_t nc = 0;
    for (int c0 = 0; c0 < k; c0 += 32) {
        const int c = c0 + lane;
        const bool in = c < k && (double)__ldg(row + c) <= t1;
        const unsigned bal = __ballot_sync(0xffffffffu, in);
        if (in) cq[nc + __popc(bal & ((1u << lane) - 1u))] = (uint32_t)c;
        nc += __popc(bal);
    }
    __syncwarp();
    WarpSel top;
    // 3. canonical fp64 rescore of C and the np smallest (qn2, c)
    const double *qd = qp + q * D;
    top.init(lst, np, true, queue);
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
    top.finish();
    for (int p = lane; p < np; p += 32) {
        const bool ok = lst[p].id != 0xFFFFFFFFu;
        probe[q * np + p] = ok ? lst[p].id : 0xFFFFFFFFu;
        probe_qn2[q * np + p] = ok ? lst[p].key : __longlong_as_double(0x7ff0000000000000ll);
    }
    if (lane == 0) ncand_out[q] = nc;
}

// sum_{j<d} (q_j - c_j)^2 left to right (canonical), the row's loads issued
// 8 at a time ahead of the dependent sum.
__device__ __forceinline__ double sqdist_rows8(const double *__restrict__ cr, const double *__restrict__ qd, int d)
{
    double acc = 0.0;
    int j = 0;
    for (; j + 16 <= d; j += 16) {
        double cv[16];
#pragma unroll
        for (int u = 0; u < 16; u++) cv[u] = __ldg(cr + j + u);
#pragma unroll
        for (int u = 0; u < 16; u++) {
            const double t = qd[j + u] - cv[u];
            acc = acc + t * t;
        }
    }
    for (; j + 8 <= d; j += 8) {
        double cv[8];
#pragma unroll
        for (int u = 0; u < 8; u++) cv[u] = __ldg(cr + j + u);
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const double t = qd[j + u] - cv[u];
            acc = acc + t * t;
        }
    }
    for (; j < d; j++) {
        const double t = qd[j] - cr[j];
        acc = acc + t * t;
    }
    return acc;
}

// Finish of the fused tensor-core probe (k_probe_tc<true, NPM>), warp per
// query.  a_(np) = np-th smallest of the parts' np smallest screen values
// (their union holds the row's np smallest, np <= 64; radix select on
// order-preserving keys, MK per lane).  The margin set {(a, c) in the parts' candidate
// buffers : a <= a_(np) + 2 delta_q} (every member was appended, see
// mrq_probe_tc.cu) is rescored in fp64 left to right over i and the np
// smallest (qn2, c) are kept.  If a buffer overflowed, all k centroids are
// rescored.
#ifndef MRQ_PF_MINB
#define MRQ_PF_MINB 10   // <= 48 registers: more resident warps (measured)
#endif
template <int MK>
__global__ void __launch_bounds__(128, MK <= 8 ? MRQ_PF_MINB : 6) k_probe_finish_w(int64_t nq, int k, int d, int np, const double *__restrict__ qp,
                                                        int D, const double *__restrict__ C,
                                                        const double *__restrict__ qnorm, double cmax, double kappa,
                                                        const uint2 *__restrict__ cbuf, int P, int capp, int G,
                                                        const uint32_t *__restrict__ ccnt,
                                                        const float *__restrict__ kvbuf, uint32_t *__restrict__ cand,
                                                        int64_t cstride,
                                                        uint32_t *__restrict__ probe, double *__restrict__ probe_qn2,
                                                        uint32_t *__restrict__ ncand_out)
{
    extern __shared__ unsigned char wsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    const int64_t q = (int64_t)blockIdx.x * wpb + warp;
    if (q >= nq) return;
    SelItem *lst = (SelItem *)wsm + (size_t)warp * MRQ_SELREG(np);
    SelItem *queue = lst + np;
    // a_(np): the used parts' 16 smallest, up to 8 per lane (<= 16 parts);
    // buffers are laid out with P parts per row, of which Pq are used
    const int Pq = tc_parts_of(q / TC_BM, nq, k, G);
    const int nv = Pq * np;   // <= 32 MK
    uint32_t key[MK];
    bool all = false;
#pragma unroll
    for (int j = 0; j < MK; j++) {
        const int i = j * 32 + lane;
        key[j] = i < nv ? f2key(kvbuf[q * P * np + i]) : 0xFFFFFFFFu;
    }
    for (int pp = lane; pp < Pq; pp += 32) all |= ccnt[q * P + pp] > (uint32_t)capp;
    all = __any_sync(0xffffffffu, all);
    uint32_t res = 0;
    for (int bit = 31; bit >= 0; bit--) {
        const uint32_t t = res | (1u << bit);
        int cnt = 0;
#pragma unroll
        for (int j = 0; j < MK; j++)
            if (j * 32 < nv) cnt += __popc(__ballot_sync(0xffffffffu, key[j] < t));
        if (cnt < np) res = t;
    }
    const double g = qnorm[q] + cmax;
    const double thr = (double)key2f(res) + 2.0 * (kappa * (g * g));
    uint32_t *cq = cand + q * cstride;   // margin set (<= min(k, P capp) entries)
    uint32_t nc = 0;
    if (all) {
        nc = (uint32_t)k;
    } else {
        // the parts' buffers as one flat index space (lane p holds part p's
        // count and exclusive prefix), 4 batches of loads in flight
        const uint32_t myc = lane < Pq ? ccnt[q * P + lane] : 0u;
        uint32_t pre = myc;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, pre, o);
            if (lane >= o) pre += y;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, pre, 31);
        pre -= myc;   // exclusive
        for (uint32_t e0 = 0; e0 < total; e0 += 128) {
            uint2 x[4];
            bool in[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const uint32_t e = e0 + 32 * u + lane;
                int part = 0;
                uint32_t pbase = 0;
                for (int pp = 1; pp < Pq; pp++) {   // last part whose prefix <= e
                    const uint32_t b = __shfl_sync(0xffffffffu, pre, pp);
                    if (b <= e) {
                        part = pp;
                        pbase = b;
                    }
                }
                x[u] = make_uint2(0u, 0u);
                if (e < total) x[u] = cbuf[(q * P + part) * capp + (e - pbase)];
                in[u] = e < total;
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const bool ok = in[u] && (double)__uint_as_float(x[u].x) <= thr;
                const unsigned bal = __ballot_sync(0xffffffffu, ok);
                if (ok) {
                    MRQ_ASSERT(nc + __popc(bal & ((1u << lane) - 1u)) < (uint32_t)cstride && x[u].y < (uint32_t)k);
                    cq[nc + __popc(bal & ((1u << lane) - 1u))] = x[u].y;
                }
                nc += __popc(bal);
            }
        }
        __syncwarp();
    }
    const double *qd = qp + q * D;
    WarpSel top;
    top.init(lst, np, true, queue);
    for (uint32_t e0 = 0; e0 < nc; e0 += 32) {
        const uint32_t e = e0 + lane;
        SelItem it = sel_inf();
        if (e < nc) {
            const uint32_t c = all ? e : cq[e];
            it.key = sqdist_rows8(C + (int64_t)c * d, qd, d);
            it.id = c;
            it.pay = c;
        }
        top.offer(it, e < nc);
    }
    top.finish();
    for (int p = lane; p < np; p += 32) {
        const bool ok = lst[p].id != 0xFFFFFFFFu;
        probe[q * np + p] = ok ? lst[p].id : 0xFFFFFFFFu;
        probe_qn2[q * np + p] = ok ? lst[p].key : __longlong_as_double(0x7ff0000000000000ll);
    }
    if (lane == 0) ncand_out[q] = nc;
}

int launch_probe_finish_w(int64_t nq, int k, int d, int np, const double *qp, int D, const double *C,
                          const double *qnorm, double cmax, double kappa, const uint2 *cbuf, int P, int capp,
                          int G, const uint32_t *ccnt, const float *kvbuf, uint32_t *cand, uint32_t *probe,
                          double *probe_qn2, uint32_t *ncand, cudaStream_t st)
{
    if (P > 16) {
        mrq_set_error("probe parts %d > 16", P);
        return MRQ_EINVAL;
    }
    const int wpb = 4;
    const size_t smem = (size_t)wpb * MRQ_SELREG(np) * sizeof(SelItem);
    auto fn = P * np <= 256 ? k_probe_finish_w<8> : k_probe_finish_w<32>;
    int rc = set_attr((const void *)fn, smem);
    if (rc) return rc;
    const int64_t cstride = std::min<int64_t>(k, (int64_t)P * capp);
    fn<<<(unsigned)((nq + wpb - 1) / wpb), wpb * 32, smem, st>>>(nq, k, d, np, qp, D, C, qnorm, cmax, kappa, cbuf, P,
                                                                 capp, G, ccnt, kvbuf, cand, cstride, probe, probe_qn2,
                                                                 ncand);
    return MRQ_OK;
}

int launch_probe_select_w(const float *approx, int64_t nq, int k, int d, int np, const double *qp, int D,
                          const double *C, const double *qnorm, double cmax, double kappa, uint32_t *cand,
                          uint32_t *probe, double *probe_qn2, uint32_t *ncand, cudaStream_t st)
{
    const int wpb = 4;
    const size_t smem = (size_t)wpb * MRQ_SELREG(np) * sizeof(SelItem);
    const int m = (np + 31) / 32;
    const unsigned grid = (unsigned)((nq + wpb - 1) / wpb);
#define MRQ_PSEL(MM)                                                                                          \
    do {                                                                                                      \
        int rc = set_attr((const void *)k_probe_select_w<MM>, smem);                                          \
        if (rc) return rc;                                                                                    \
        k_probe_select_w<MM><<<grid, wpb * 32, smem, st>>>(approx, nq, k, d, np, qp, D, C, qnorm, cmax, kappa, \
                                                           cand, probe, probe_qn2, ncand);                    \
    } while (0)
    if (m <= 1) MRQ_PSEL(1);
    else if (m <= 2) MRQ_PSEL(2);
    else if (m <= 4) MRQ_PSEL(4);
    else if (m <= 8) MRQ_PSEL(8);
    else if (m <= 16) MRQ_PSEL(16);
    else MRQ_PSEL(32);
#undef MRQ_PSEL
    return MRQ_OK;
}

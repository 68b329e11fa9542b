// mrq_internal.cuh -- internal declarations of libmrq (B200 / sm_100a).
//
// Everything here is the product path.  It shares nothing with oracle/.
// The numeric contract requires that every
// fp64 expression that decides a code bit, a level, a flag or an ordering is
// evaluated left to right without contraction; the library is compiled with
// --fmad=false and the expressions below spell out their evaluation order.
#pragma once

#include <cuda_runtime.h>
#include <cstdio>
#include <stdint.h>

#include <exception>
#include <map>
#include <new>
#include <string>
#include <vector>

#include "../../include/mrq.h"

#define MRQ_BQ 4                 // query bit-planes (levels 0..15), R-7
#define MRQ_MAX_K 1024
#define MRQ_MAX_NPROBE 1024
#define MRQ_MAX_SEEDS 4096          // seed_mult * K: the seed kernels' per-warp selection region
#define MRQ_SLOT_ALIGN 4         // list starts aligned to 4 slots (16 B) for 128-bit loads
#define MRQ_PAD_ID 0xFFFFFFFFu

// ------------------------------------------------------------------ errors
void mrq_set_error(const char *fmt, ...);

#define MRQ_CUDA_TRY(expr)                                                          \
    do {                                                                            \
        cudaError_t _e = (expr);                                                    \
        if (_e != cudaSuccess) {                                                    \
            mrq_set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),    \
                          __FILE__, __LINE__);                                      \
            return MRQ_ECUDA;                                                       \
        }                                                                           \
    } while (0)

// Entry-point guard: C++ exceptions (std::bad_alloc from a vector resize, ...)
// never cross the extern "C" boundary; they become MRQ_ENOMEM / MRQ_EINVAL.
template <class F>
int mrq_guard(F &&f)
{
    try {
        return f();
    } catch (const std::bad_alloc &) {
        mrq_set_error("host allocation failed (std::bad_alloc)");
        return MRQ_ENOMEM;
    } catch (const std::exception &e) {
        mrq_set_error("internal error: %s", e.what());
        return MRQ_EINVAL;
    } catch (...) {
        mrq_set_error("internal error (unknown exception)");
        return MRQ_EINVAL;
    }
}

// Device-side bounds checks of the MRQ_CHECK build (scripts/variant.sh check
// -DMRQ_CHECK=1; compute-sanitizer is not available on the GPU pool): a
// violated invariant prints its location and traps (the launch fails with an
// error instead of corrupting memory).  Compiled out otherwise.
#if defined(MRQ_CHECK) && MRQ_CHECK
#define MRQ_ASSERT(cond)                                                                                   \
    do {                                                                                                   \
        if (!(cond)) {                                                                                     \
            printf("MRQ_CHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__, __LINE__,       \
                   (int)blockIdx.x, (int)threadIdx.x);                                                     \
            __trap();                                                                                      \
        }                                                                                                  \
    } while (0)
#else
#define MRQ_ASSERT(cond) \
    do {                 \
    } while (0)
#endif

// ------------------------------------------------------------ index object
struct DevArr {
    void *p = nullptr;
    size_t bytes = 0;
};

struct mrq_index {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[13] = {};
    cudaStream_t side = nullptr;      // fork/join stream for the single-block kernels (query order, F1 offsets)
    cudaEvent_t ev_fork[4] = {};
    int64_t N = 0, npad = 0;
    int D = 0, d = 0, k = 0, W = 0;
    int rank = 0, world = 1;
    void *nccl_comm = nullptr;                 // ncclComm_t (NCCL loaded at run time)
    mrq_allgather_fn host_ag = nullptr;        // host exchange (tests / virtual ranks)
    void *host_ctx = nullptr;
    void *xhost = nullptr;                     // pinned staging of the host exchange
    size_t xhost_bytes = 0;
    int force_exchange = 0;                    // mrq_debug_set("force_exchange"): world-1 runs the sharded path
    int front_shard = 1;                       // mrq_debug_set("front_shard"): a1-a3 per query slice + all-gather
    int comm_failed = 0;                       // the NCCL communicator was aborted (mrq_comm_fail)
    void *probe_tc = nullptr;                  // tcgen05 probe state (mrq_probe_tc.cu)
    int force_cuda_core_probe = 0;             // mrq_debug_set("cuda_core_probe"): CUDA-core screen instead
#ifndef MRQ_QORDER_DEFAULT
#define MRQ_QORDER_DEFAULT 2
#endif
    int qorder_on = MRQ_QORDER_DEFAULT;        // mrq_debug_set("qorder"): query processing order (0 as given,
                                               // 1 key from 3 principal coordinates, 2 key of the nearest probed list)
    int force_probe_unfused = 0;               // mrq_debug_set("probe_unfused"): screen to HBM + k_probe_select_w
    int graphs = 1;                            // CUDA-graph replay of repeated searches (mrq_debug_set "graphs")
    int tails_host = 0;                        // MRQ_LOAD_TAILS_HOST: tails in mapped pinned host memory
    void *tails_hbuf = nullptr;                // its host allocation
    void *gexec = nullptr;                     // cudaGraphExec_t of the cached search
    void *g_key = nullptr, *g_pending = nullptr;   // GraphKey of the cached / last uncached search
    int sm_count = 148;
    int sketch_on = 1;                         // mrq_debug_set("sketch"): head-sketch pre-pass of the stage-2 gather
    int probe_capp = 256;                      // mrq_debug_set("probe_capp"): fused-probe candidate buffer per part
    int probe_share = 1;                       // mrq_debug_set("probe_share"): parts of a row share their bound
    int fuse_topk_on = 1;                      // mrq_debug_set("fuse_topk"): k_head_topk where it applies
    int scan_lm = 0;                           // mrq_debug_set("scan_lm"): list-major scan (1 CUDA-core, 2 tensor-core S; d <= 128)
    int lm_qg = 16;                            // mrq_debug_set("scan_lm_qg"): pairs per list-major work unit
    uint64_t cand_budget = (uint64_t)8 << 30;  // mrq_debug_set("cand_budget_mb"): host-bound scratch budget
    int smem_optin = 227 * 1024;               // max dynamic shared memory per block (opt-in)
    uint64_t scratch_gen = 0;                  // bumped whenever a scratch buffer is reallocated (graph key)

    // host mirrors
    std::vector<uint32_t> h_list_off, h_list_size;
    std::vector<uint64_t> h_topsum;   // h_topsum[p] = sum of the p largest local list sizes
    uint32_t max_list = 0;
    double cmax = 0.0;           // max_j ||c_j|| (rounded up), probe error bound

    // device index (HBM layout)
    double *mu = nullptr, *PT = nullptr, *lam = nullptr, *RT = nullptr;   // PT[j][i] = P[i][j], RT[i][j] = R[j][i]
    double *C = nullptr, *Rc = nullptr;                                   // C[k][d], Rc[k][d]
    float *C32T = nullptr;                                                // C32T[i][k] fp32 centroids, transposed
    float *C32 = nullptr;                                                 // C32[k][d] fp32 centroids (GEMM B operand)
    float *cn32 = nullptr;                                                // ||c||^2 fp32 (GEMM epilogue)
    uint32_t *list_off = nullptr, *list_size = nullptr;                   // [k+1], [k] (owned lists; 0 if not owned)
    uint32_t *list_size_g = nullptr;                                      // [k] global list sizes (seed pool, decision T)
    uint32_t *ids = nullptr;                                              // [npad] global id of each slot
    uint16_t *list_key = nullptr;                                         // [k] locality key of each list (< MRQ_QO_KEYS)
    uint32_t *codes = nullptr;                                            // [W][npad]
    float *f1 = nullptr, *f2 = nullptr, *f3 = nullptr, *xr2 = nullptr;    // [npad]
    float *heads = nullptr, *tails = nullptr;                             // [npad][d], [npad][D-d]
    uint8_t *hq = nullptr;                                                // [npad][dq] head sketch (biased int8)
    float4 *hs = nullptr;                                                 // [npad] sketch (s, E, ||x_r||^2, -)
    int dq = 0;                                                           // sketch row bytes: d rounded up to 16

    // per-search scratch (grow only)
    std::map<std::string, DevArr> scratch;
    // shapes of the last search (debug fetch)
    int64_t last_nq = 0;
    int last_np = 0, last_K = 0, last_Kp = 0;
    uint64_t last_total = 0;
    std::vector<void *> owned;   // device allocations of the index
    int dbg_dump_dis = 0;        // mrq_debug_set("dump_dis")
};

// helpers in mrq_api.cu
int mrq_scratch(mrq_index *ix, const char *name, size_t bytes, void **out);

// Item of the multi-rank exchanges: selection key (dis',
// dis_o' or exact), exact distance, global id, local slot (PAD on the
// receiving side when the item belongs to another rank).
struct XItem {
    double key;
    double exact;
    uint32_t id;
    uint32_t slot;
};

// ---------------------------------------------------------- device helpers
struct SelItem {
    double key;
    uint32_t id;     // tie-break key (global vector id or centroid id)
    uint32_t pay;    // payload (slot position, entry index, ...)
};

__device__ __forceinline__ bool sel_less(const SelItem &a, const SelItem &b)
{
    return a.key < b.key || (a.key == b.key && a.id < b.id);
}

__device__ __forceinline__ SelItem sel_inf()
{
    SelItem s;
    s.key = __longlong_as_double(0x7ff0000000000000ll);
    s.id = 0xFFFFFFFFu;
    s.pay = 0xFFFFFFFFu;
    return s;
}

// Ascending bitonic sort of S (power of two) items by (key, id); whole block.
__device__ __forceinline__ void block_bitonic_sort(SelItem *buf, int S)
{
    for (int k = 2; k <= S; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < S; i += blockDim.x) {
                int ixj = i ^ j;
                if (ixj > i) {
                    SelItem a = buf[i], b = buf[ixj];
                    bool up = (i & k) == 0;
                    if (sel_less(b, a) == up) {
                        buf[i] = b;
                        buf[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
}

// Streaming block-wide selection of the L smallest (key, id) among n items
// produced by get(i).  buf holds S items (power of two, S >= L + 32).  On
// return buf[0 .. min(L, n)) are the selected items in ascending order.
template <class Get>
__device__ int block_select(SelItem *buf, int S, int L, int n, Get get)
{
    for (int i = threadIdx.x; i < S; i += blockDim.x) buf[i] = sel_inf();
    __syncthreads();
    const int chunk = S - L;
    for (int base = 0; base < n; base += chunk) {
        for (int i = threadIdx.x; i < chunk; i += blockDim.x) {
            int g = base + i;
            buf[L + i] = g < n ? get(g) : sel_inf();
        }
        __syncthreads();
        block_bitonic_sort(buf, S);
    }
    return n < L ? n : L;
}

// Order-preserving map of a float to uint32 (ascending floats -> ascending keys).
__device__ __forceinline__ uint32_t f2key(float f)
{
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k)
{
    uint32_t u = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
    return __uint_as_float(u);
}

// Warp-cooperative sequential squared distance over row segments.  Each lane
// owns one row (slot_lane, valid): acc += sum_{e=0}^{len-1} ((double)row[off+e]
// - q[e])^2, left to right (the oracle's order).  Rows are staged 32 columns
// at a time through shared memory tile[32][33]: when stride, off and len are
// multiples of 4 floats, each lane issues 8 independent 16-byte loads (8 lanes
// cover one 128-byte row segment, a warp instruction covers 4 rows) before the
// first store, so a warp keeps 8 x 512 B of gathers in flight.
__device__ __forceinline__ double warp_rows_sqdist(const float *__restrict__ base, int64_t stride, int off,
                                                   uint32_t slot_lane, bool valid, int len,
                                                   const double *q, double acc, float *tile)
{
    const int lane = threadIdx.x & 31;
    const bool vec = ((stride | off | len) & 3) == 0;
    const int rs = lane >> 3, cq = lane & 7;
    for (int c0 = 0; c0 < len; c0 += 32) {
        const int cl = min(32, len - c0);
        if (vec) {
            float4 v[8];
#pragma unroll
            for (int it = 0; it < 8; it++) {
                const int r = it * 4 + rs;
                const uint32_t s = __shfl_sync(0xffffffffu, slot_lane, r);
                const int ok = __shfl_sync(0xffffffffu, (int)valid, r);
                const int col = cq * 4;
                v[it] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (ok && col < cl) v[it] = __ldg((const float4 *)(base + (int64_t)s * stride + off + c0 + col));
            }
#pragma unroll
            for (int it = 0; it < 8; it++) {
                float *t = tile + (it * 4 + rs) * 33 + cq * 4;
                t[0] = v[it].x;
                t[1] = v[it].y;
                t[2] = v[it].z;
                t[3] = v[it].w;
            }
        } else {
            for (int r = 0; r < 32; r++) {
                const uint32_t s = __shfl_sync(0xffffffffu, slot_lane, r);
                const int ok = __shfl_sync(0xffffffffu, (int)valid, r);
                if (ok && lane < cl) tile[r * 33 + lane] = __ldg(base + (int64_t)s * stride + off + c0 + lane);
            }
        }
        __syncwarp();
        if (valid) {
            for (int e = 0; e < cl; e++) {
                double t = (double)tile[lane * 33 + e] - q[c0 + e];
                acc = acc + t * t;
            }
        }
        __syncwarp();
    }
    return acc;
}

// Warp-level streaming top-L (L smallest (key, id)) kept sorted in shared
// memory a[0..L).  Every lane offers one item per call; the warp inserts the
// survivors one by one (position = number of smaller entries, found with
// ballots; entries shift up by one).  An item equal to an entry (same key and
// id) is a duplicate and is dropped, so the list holds distinct items.
struct WarpTop {
    SelItem *a;
    int L;

    __device__ __forceinline__ void init(SelItem *buf, int L_)
    {
        a = buf;
        L = L_;
        const int lane = threadIdx.x & 31;
        for (int j = lane; j < L; j += 32) a[j] = sel_inf();
        __syncwarp();
    }

    __device__ __forceinline__ void offer(const SelItem &it, bool valid)
    {
        const int lane = threadIdx.x & 31;
        unsigned m = __ballot_sync(0xffffffffu, valid && sel_less(it, a[L - 1]));
        while (m) {
            const int src = __ffs(m) - 1;
            m &= m - 1;
            SelItem x;
            x.key = __shfl_sync(0xffffffffu, it.key, src);
            x.id = __shfl_sync(0xffffffffu, it.id, src);
            x.pay = __shfl_sync(0xffffffffu, it.pay, src);
            if (!sel_less(x, a[L - 1])) continue;                 // warp-uniform
            int pos = 0;
            bool dup = false;
            for (int j0 = 0; j0 < L; j0 += 32) {
                const int j = j0 + lane;
                const bool in = j < L;
                const SelItem e = in ? a[j] : sel_inf();
                pos += __popc(__ballot_sync(0xffffffffu, in && sel_less(e, x)));
                dup |= __any_sync(0xffffffffu, in && e.key == x.key && e.id == x.id);
            }
            if (dup) continue;                                     // warp-uniform
            for (int j0 = ((L - 1) / 32) * 32; j0 >= 0; j0 -= 32) {
                const int j = j0 + lane;
                const bool mv = j >= pos && j < L - 1;
                SelItem v;
                if (mv) v = a[j];
                __syncwarp();
                if (mv) a[j + 1] = v;
                __syncwarp();
            }
            if (lane == 0) a[pos] = x;
            __syncwarp();
        }
    }
};

// Register-resident variant for L <= 32: lane i holds the i-th smallest
// item; an insertion is one ballot (position) and one shuffle-up (shift).
struct WarpTopReg {
    double key;
    uint32_t id, pay;
    int L;

    __device__ __forceinline__ void init(int L_)
    {
        L = L_;
        const SelItem z = sel_inf();
        key = z.key;
        id = z.id;
        pay = z.pay;
    }

    __device__ __forceinline__ void offer(const SelItem &it, bool valid)
    {
        const int lane = threadIdx.x & 31;
        double tk = __shfl_sync(0xffffffffu, key, L - 1);
        uint32_t ti = __shfl_sync(0xffffffffu, id, L - 1);
        unsigned m = __ballot_sync(0xffffffffu, valid && (it.key < tk || (it.key == tk && it.id < ti)));
        while (m) {
            const int src = __ffs(m) - 1;
            m &= m - 1;
            const double xk = __shfl_sync(0xffffffffu, it.key, src);
            const uint32_t xi = __shfl_sync(0xffffffffu, it.id, src);
            const uint32_t xp = __shfl_sync(0xffffffffu, it.pay, src);
            if (!(xk < tk || (xk == tk && xi < ti))) continue;                      // warp-uniform
            const bool mine = lane < L;
            if (__any_sync(0xffffffffu, mine && key == xk && id == xi)) continue;    // duplicate
            const int pos = __popc(__ballot_sync(0xffffffffu, mine && (key < xk || (key == xk && id < xi))));
            const double uk = __shfl_up_sync(0xffffffffu, key, 1);
            const uint32_t ui = __shfl_up_sync(0xffffffffu, id, 1);
            const uint32_t up = __shfl_up_sync(0xffffffffu, pay, 1);
            if (lane > pos) {
                key = uk;
                id = ui;
                pay = up;
            } else if (lane == pos) {
                key = xk;
                id = xi;
                pay = xp;
            }
            tk = __shfl_sync(0xffffffffu, key, L - 1);
            ti = __shfl_sync(0xffffffffu, id, L - 1);
        }
    }
};

// Register-resident warp select for streams of DISTINCT items, L <= 32
// (bitonic, in the manner of warp-select top-k): the warp keeps its 32
// smallest items sorted across lanes; a batch with any item below the L-th
// smallest is sorted descending (bitonic sort over lanes), merged by an
// elementwise min (a bitonic sequence holding the 32 smallest of both) and
// re-sorted ascending by a bitonic merge -- 20 compare-exchange steps per
// useful batch, independent of how many of its items enter.
struct WarpTopBitonic {
    double key;
    uint32_t id, pay;
    int L;

    __device__ __forceinline__ static bool lt(double ak, uint32_t ai, double bk, uint32_t bi)
    {
        return ak < bk || (ak == bk && ai < bi);
    }
    // compare-exchange with lane ^ j; keep the smaller item iff `keep_min`
    __device__ __forceinline__ static void cx(double &k, uint32_t &i, uint32_t &p, int j, bool keep_min)
    {
        const double ok = __shfl_xor_sync(0xffffffffu, k, j);
        const uint32_t oi = __shfl_xor_sync(0xffffffffu, i, j);
        const uint32_t op = __shfl_xor_sync(0xffffffffu, p, j);
        const bool other_less = lt(ok, oi, k, i);
        if (other_less == keep_min) {
            k = ok;
            i = oi;
            p = op;
        }
    }
    __device__ __forceinline__ void init(int L_)
    {
        L = L_;
        key = __longlong_as_double(0x7ff0000000000000ll);
        id = 0xFFFFFFFFu;
        pay = 0xFFFFFFFFu;
    }
    __device__ __forceinline__ void offer(const SelItem &it, bool valid)
    {
        const int lane = threadIdx.x & 31;
        const double tk = __shfl_sync(0xffffffffu, key, L - 1);
        const uint32_t ti = __shfl_sync(0xffffffffu, id, L - 1);
        const bool pass = valid && lt(it.key, it.id, tk, ti);
        if (!__any_sync(0xffffffffu, pass)) return;
        double xk = pass ? it.key : __longlong_as_double(0x7ff0000000000000ll);
        uint32_t xi = pass ? it.id : 0xFFFFFFFFu, xp = pass ? it.pay : 0xFFFFFFFFu;
        // bitonic sort of the batch, descending across lanes
#pragma unroll
        for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1) {
                const bool up = (lane & k) != 0;           // k = 32: all descending
                const bool lower = (lane & j) == 0;
                cx(xk, xi, xp, j, lower == up);
            }
        }
        // elementwise min with the ascending list: bitonic, holds the 32 smallest
        if (lt(xk, xi, key, id)) {
            key = xk;
            id = xi;
            pay = xp;
        }
        // bitonic merge, ascending
#pragma unroll
        for (int j = 16; j > 0; j >>= 1) cx(key, id, pay, j, (lane & j) == 0);
    }
};

// Query-order key (k_qtail -> k_qorder): Morton interleave of the three
// leading principal coordinates, z_i = q_p[i] / sqrt(lambda_i) in 16 levels
// over [-2, 2) -> 12 bits.
#define MRQ_QO_KEYS 4096
__device__ __forceinline__ uint32_t mrq_qorder_key(const double *row, const double *lam, int D)
{
    uint32_t key = 0;
    const int nd = D < 3 ? D : 3;
    for (int i = 0; i < nd; i++) {
        const double z = lam[i] > 0.0 ? row[i] / sqrt(lam[i]) : 0.0;
        int lv = (int)floor((z + 2.0) * 4.0);
        lv = lv < 0 ? 0 : (lv > 15 ? 15 : lv);
        for (int b = 0; b < 4; b++) key |= (uint32_t)((lv >> b) & 1) << (3 * b + i);
    }
    return key;
}

// x = hi + lo + r with hi = RN_tf32(x), lo = RN_tf32(x - hi), |r| <= 2^-22 |x|
// (the probe's 3xTF32 operands; x - hi is exact in fp32)
__device__ __forceinline__ void tf32_split(float x, float &hi, float &lo)
{
    uint32_t h, l;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
    hi = __uint_as_float(h);
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(x - hi));
    lo = __uint_as_float(l);
}

#define MRQ_SELQ 64   // items of a WarpSel compaction queue
// per-warp selection region for a list of L: list, queue, merge temp
// lists longer than this use the merge selection (shorter: smem insertion)
#define MRQ_MERGE_MIN 64
#define MRQ_SELREG(L) ((L) + MRQ_SELQ + ((L) > MRQ_MERGE_MIN ? (L) + 32 : 0))

// The L-th smallest (L <= 32) of the 32 lane values v (bitonic sort across
// lanes).  Used as a selection pre-threshold: if every lane's v is the
// minimum of its share of a stream, at least L stream items are <= the result.
__device__ __forceinline__ double warp_kth_smallest(double v, int L)
{
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const double o = __shfl_xor_sync(0xffffffffu, v, j);
            const bool up = (lane & k) == 0;
            const bool lower = (lane & j) == 0;
            const bool keep_min = lower == up;
            v = keep_min ? fmin(v, o) : fmax(v, o);
        }
    }
    return __shfl_sync(0xffffffffu, v, L - 1);
}

// Selection of the L smallest distinct (key, id): registers for L <= 32,
// the shared-memory list otherwise.  After finish() the sorted items are in
// buf[0 .. L) either way.
// Merge selection for 32 < L: the sorted list a[0..L) lives in shared
// memory; a batch of up to 32 queued items is sorted across the lanes
// (bitonic), every list item's and batch item's position in the merged order
// is found by binary search (list items first on ties, so a repeated item
// lands next to its first copy), the merge is written to t[0..L+32) and
// compacted back into a[] dropping repeats -- a few hundred instructions per
// 32 items instead of an O(L) insertion per item.
struct WarpTopMerge {
    __device__ __forceinline__ static bool le(const SelItem &x, const SelItem &y) { return !sel_less(y, x); }
    __device__ __forceinline__ static void init(SelItem *a, int L)
    {
        const int lane = threadIdx.x & 31;
        for (int i = lane; i < L; i += 32) a[i] = sel_inf();
        __syncwarp();
    }
    __device__ __forceinline__ static void merge(SelItem *a, SelItem *t, int L, SelItem x, bool valid)
    {
        const int lane = threadIdx.x & 31;
        if (!valid) x = sel_inf();
        // sort the batch ascending across lanes
#pragma unroll
        for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1) {
                const bool up = (lane & k) == 0;
                const bool lower = (lane & j) == 0;
                WarpTopBitonic::cx(x.key, x.id, x.pay, j, lower == up);
            }
        }
        __syncwarp();
        // list items: pos = i + #{batch items < a_i} (warp-uniform trip count:
        // every lane takes part in every shuffle)
        for (int i0 = 0; i0 < L; i0 += 32) {
            const int i = i0 + lane;
            const bool in = i < L;
            const SelItem e = in ? a[i] : sel_inf();
            int lo = 0;   // number of batch items strictly less than e (batch sorted)
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const int probe = lo + step - 1;
                // warp-divergent source lanes: every lane participates in each shuffle
                const double pk = __shfl_sync(0xffffffffu, x.key, probe);
                const uint32_t pi = __shfl_sync(0xffffffffu, x.id, probe);
                SelItem pv;
                pv.key = pk;
                pv.id = pi;
                if (sel_less(pv, e)) lo += step;
            }
            {
                const double pk = __shfl_sync(0xffffffffu, x.key, lo < 32 ? lo : 31);
                const uint32_t pi = __shfl_sync(0xffffffffu, x.id, lo < 32 ? lo : 31);
                SelItem pv;
                pv.key = pk;
                pv.id = pi;
                if (lo < 32 && sel_less(pv, e)) lo++;
            }
            if (in) t[i + lo] = e;
        }
        // batch items: pos = lane + #{list items <= x}
        int lo = 0, hi = L;   // first index with a[idx] > x
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (le(a[mid], x))
                lo = mid + 1;
            else
                hi = mid;
        }
        t[lane + lo] = x;
        __syncwarp();
        // compact t[0..L+32) into a[0..L), dropping repeats of the previous item
        int out = 0;
        for (int i0 = 0; i0 < L + 32 && out < L; i0 += 32) {
            const int i = i0 + lane;
            SelItem v = sel_inf();
            bool keep = false;
            if (i < L + 32) {
                v = t[i];
                keep = v.id != 0xFFFFFFFFu;
                if (keep && i > 0) {
                    const SelItem p = t[i - 1];
                    keep = !(p.key == v.key && p.id == v.id);
                }
            }
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            const int o = out + __popc(bal & ((1u << lane) - 1u));
            __syncwarp();
            if (keep && o < L) a[o] = v;
            out += __popc(bal);
        }
        __syncwarp();
        for (int i = (out < L ? out : L) + lane; i < L; i += 32) a[i] = sel_inf();
        __syncwarp();
    }
};

// MG: the merge selection (mode 3) is compiled in; kernels instantiate it
// only for lists longer than MRQ_MERGE_MIN, so the short-list instances keep
// their register budget.
template <bool MG = false>
struct WarpSelT {
    WarpTop sm;
    WarpTopReg rg;
    WarpTopBitonic bt;
    SelItem *qbuf;   // modes 2, 3: compaction queue of MRQ_SELQ items
    int qn;
    int mode;        // 0 shared-memory list, 1 register insertion (dedup), 2 register bitonic (distinct items),
                     // 3 shared-memory merge (L > 32, dedup)

    // distinct: the caller guarantees no (key, id) is offered twice; then
    // qbuf (MRQ_SELQ items of shared memory) queues the items that pass the
    // current threshold and full batches of 32 go through one bitonic merge.
    // L > MRQ_MERGE_MIN with a queue: merge selection, its temp (L + 32
    // items) right after the queue (the MRQ_SELREG layout).
    __device__ __forceinline__ void init(SelItem *buf, int L, bool distinct = false, SelItem *queue = nullptr)
    {
        mode = L > 32 ? (MG && queue && L > MRQ_MERGE_MIN ? 3 : 0) : (distinct && queue ? 2 : 1);
        sm.a = buf;
        sm.L = L;
        qbuf = queue;
        qn = 0;
        if (mode == 3)
            WarpTopMerge::init(buf, L);
        else if (mode == 2)
            bt.init(L);
        else if (mode == 1)
            rg.init(L);
        else
            sm.init(buf, L);
    }
    __device__ __forceinline__ void flush(int n)
    {
        const int lane = threadIdx.x & 31;
        __syncwarp();
        SelItem x = sel_inf();
        if (lane < n) x = qbuf[lane];
        __syncwarp();
        if (mode == 3)
            WarpTopMerge::merge(sm.a, qbuf + MRQ_SELQ, sm.L, x, lane < n);
        else
            bt.offer(x, lane < n);
    }
    __device__ __forceinline__ void offer(const SelItem &it, bool valid)
    {
        if (mode == 2 || mode == 3) {
            const int lane = threadIdx.x & 31;
            double tk;
            uint32_t ti;
            if (mode == 2) {
                tk = __shfl_sync(0xffffffffu, bt.key, bt.L - 1);
                ti = __shfl_sync(0xffffffffu, bt.id, bt.L - 1);
            } else {
                const SelItem th = sm.a[sm.L - 1];
                tk = th.key;
                ti = th.id;
            }
            const bool pass = valid && WarpTopBitonic::lt(it.key, it.id, tk, ti);
            const unsigned m = __ballot_sync(0xffffffffu, pass);
            if (!m) return;
            if (pass) qbuf[qn + __popc(m & ((1u << lane) - 1u))] = it;
            qn += __popc(m);
            if (qn >= 32) {
                flush(32);
                const int rest = qn - 32;
                SelItem y;
                if (lane < rest) y = qbuf[32 + lane];
                __syncwarp();
                if (lane < rest) qbuf[lane] = y;
                __syncwarp();
                qn = rest;
            }
        } else if (mode == 1) {
            rg.offer(it, valid);
        } else {
            sm.offer(it, valid);
        }
    }
    __device__ __forceinline__ void finish()
    {
        if ((mode == 2 || mode == 3) && qn > 0) {
            flush(qn);
            qn = 0;
        }
        if (mode == 1 || mode == 2) {
            const int lane = threadIdx.x & 31;
            __syncwarp();
            if (lane < sm.L) {
                SelItem x;
                x.key = mode == 2 ? bt.key : rg.key;
                x.id = mode == 2 ? bt.id : rg.id;
                x.pay = mode == 2 ? bt.pay : rg.pay;
                sm.a[lane] = x;
            }
        }
        __syncwarp();
    }
};using WarpSel = WarpSelT<false>;


// ================================================================ a4 / a5
// Weighted population counts with carry-save adders.  words[l] holds the
// words of weight 2^l (counts n[l]); the result is sum_l 2^l sum_i popc(words).
// At each weight the words are reduced with full adders (3 words -> sum at
// this weight + carry at the next: popc(a)+popc(b)+popc(c) = popc(a^b^c) +
// 2 popc(maj(a,b,c))) and half adders (2 -> 1 + carry) until one word is
// left, which is counted with one POPC.  Exact integer identities; fewer
// POPCs (quarter-rate on the SM) for a few more LOP3s: S over 4 planes x W
// words needs 5 POPCs at W = 2 (not 8), 6 at W = 4 (not 16).
template <int NMAX>
struct CsaAcc {
    uint32_t w[NMAX];
    int n = 0;
    __device__ __forceinline__ void push(uint32_t x) { w[n++] = x; }
};

__device__ __forceinline__ uint32_t lop_xor3(uint32_t a, uint32_t b, uint32_t c) { return a ^ b ^ c; }
__device__ __forceinline__ uint32_t lop_maj(uint32_t a, uint32_t b, uint32_t c) { return (a & b) | (c & (a | b)); }

// S = sum_b 2^b sum_w popc(x[b][w]) for NB planes of W words (all indices
// compile-time, so the adder network is fully unrolled into registers).
template <int NB, int W>
__device__ __forceinline__ int csa_weighted_popc(const uint32_t (&x)[NB][W])
{
    int S = 0;
    uint32_t carry[W + 2];
    int nc = 0;
#pragma unroll
    for (int lvl = 0; lvl < NB + 8; lvl++) {
        uint32_t cur[W + 2 + W];
        int n = 0;
#pragma unroll
        for (int i = 0; i < W + 2; i++)
            if (i < nc) cur[n++] = carry[i];
        if (lvl < NB) {
#pragma unroll
            for (int i = 0; i < W; i++) cur[n++] = x[lvl][i];
        }
        nc = 0;
#pragma unroll
        for (int it = 0; it < 2 * W + 2; it++) {
            if (n >= 3) {
                const uint32_t a = cur[n - 1], b = cur[n - 2], c = cur[n - 3];
                cur[n - 3] = lop_xor3(a, b, c);
                carry[nc++] = lop_maj(a, b, c);
                n -= 2;
            } else if (n == 2) {
                const uint32_t a = cur[0], b = cur[1];
                cur[0] = a ^ b;
                carry[nc++] = a & b;
                n = 1;
            }
        }
        if (n == 1) S += __popc(cur[0]) << lvl;
    }
    return S;
}

// The scan epilogue shared by the seed pass and the scan (Eq.4
// with R-1; Eq.5 P:255 with R-2/R-5; Alg.2 L12 P:314):
//   S = sum_b 2^b popc(code & p_b) = sum_{bit_j=1} L_j,  pop = popc(code)
//   ip = ((A pop + Bc S) - C0) / sqrt(d)        = <x_hat, r_bar>
//   dis' = (f1 + g1) - 2 (f2 ip)
//   LB1 = (dis' - eb f3) - eps_r
// Hand-written networks for W = 1 and 2 (the compiler's unrolling of the
// generic one leaves register moves): W = 2 is a half adder at weight 1 and
// full adders at weights 2, 4, 8 -> 5 POPCs for S.
__device__ __forceinline__ int csa_S_w2(uint32_t c0, uint32_t c1, const uint32_t *pl)
{
    const uint32_t a0 = c0 & pl[0], b0 = c1 & pl[1];
    const uint32_t a1 = c0 & pl[2], b1 = c1 & pl[3];
    const uint32_t a2 = c0 & pl[4], b2 = c1 & pl[5];
    const uint32_t a3 = c0 & pl[6], b3 = c1 & pl[7];
    const uint32_t s0 = a0 ^ b0, k1 = a0 & b0;
    const uint32_t s1 = lop_xor3(k1, a1, b1), k2 = lop_maj(k1, a1, b1);
    const uint32_t s2 = lop_xor3(k2, a2, b2), k3 = lop_maj(k2, a2, b2);
    const uint32_t s3 = lop_xor3(k3, a3, b3), k4 = lop_maj(k3, a3, b3);
    return __popc(s0) + (__popc(s1) << 1) + (__popc(s2) << 2) + (__popc(s3) << 3) + (__popc(k4) << 4);
}

// Exact int -> fp64 for 0 <= n < 2^31 as (2^52 + n) - 2^52: one DADD on
// the fp64 pipe instead of an I2F on the XU pipe, which the scan's POPCs and
// F2Fs keep busy (measured: scan -2.7%; moving F2F.F64.F32 to integer ops
// instead, or an fp32 pre-screen of LB1, cost more issue slots than they
// saved -- DESIGN.md performance log).
__device__ __forceinline__ double i2d_exact(int n)
{
    return __hiloint2double(0x43300000, n) - 4503599627370496.0;
}

template <int W>
__device__ __forceinline__ void mrq_pop_S(const uint32_t *code, const uint32_t *pl, int &pop, int &S)
{
    if (W == 1) {
        pop = __popc(code[0]);
        S = __popc(code[0] & pl[0]) + (__popc(code[0] & pl[1]) << 1) + (__popc(code[0] & pl[2]) << 2) +
            (__popc(code[0] & pl[3]) << 3);
    } else if (W == 2) {
        pop = __popc(code[0]) + __popc(code[W - 1]);
        S = csa_S_w2(code[0], code[W - 1], pl);
    } else {
        uint32_t cw[1][W];
#pragma unroll
        for (int w = 0; w < W; w++) cw[0][w] = code[w];
        pop = csa_weighted_popc<1, W>(cw);
        uint32_t x[MRQ_BQ][W];
#pragma unroll
        for (int b = 0; b < MRQ_BQ; b++)
#pragma unroll
            for (int w = 0; w < W; w++) x[b][w] = code[w] & pl[b * W + w];
        S = csa_weighted_popc<MRQ_BQ, W>(x);
    }
}

// the canonical fp64 evaluation from (pop, S)
__device__ __forceinline__ double mrq_lb1_ps(int pop, int S, const double *qc, double isd, double eps_r, float f1,
                                             float f2, float f3, double *dis_out)
{
    const double t1 = qc[0] * i2d_exact(pop);
    const double t2 = qc[1] * i2d_exact(S);
    const double t4 = (t1 + t2) - qc[2];
    const double ip = t4 * isd;
    const double t5 = (double)f1 + qc[3];
    const double t6 = (double)f2 * ip;
    const double dis = t5 - 2.0 * t6;
    *dis_out = dis;
    return (dis - qc[4] * (double)f3) - eps_r;
}

template <int W>
__device__ __forceinline__ double mrq_lb1(const uint32_t *code, const uint32_t *pl, const double *qc, double isd,
                                          double eps_r, float f1, float f2, float f3, double *dis_out)
{
    int pop, S;
    mrq_pop_S<W>(code, pl, pop, S);
    return mrq_lb1_ps(pop, S, qc, isd, eps_r, f1, f2, f3, dis_out);
}


// -------------------------------------------------------------------------
// Staged warp row gather.  A warp processes entries 0..n-1 in groups of 32
// (lane = entry within the group).  Each group's rows are copied, one
// MRQ_RG_CH-float column batch of [off, off + len) at a time, into the warp's
// shared-memory stage with coalesced 16-byte cp.async (8 lanes cover one
// 128-byte row segment, an instruction covers 4 rows); two stages, so batch
// j+1 is in flight while batch j is consumed.  Each lane then sums its own
// row from shared memory left to right in fp64 (the canonical order,
// DESIGN.md §4):  acc = init(e, slot); acc += ((double)x - q)^2 ...  and
// done(e, valid, acc) is called by the whole warp after the row's last batch.
// Shared-memory reads are conflict-free (row stride CH + 4 floats).
// (A per-lane cp.async.bulk of each row was tried: its operands must be
// warp-uniform, so the compiler serializes the 32 lanes' copies.)
// Per-warp shared memory: MRQ_RG_FLOATS floats.
// Requirements: row stride, off and len multiples of 4 floats (16-B copies).
#ifndef MRQ_RG_CH
#define MRQ_RG_CH 32
#endif
#define MRQ_RG_STRIDE (MRQ_RG_CH + 4)
#define MRQ_RG_STAGE (32 * MRQ_RG_STRIDE)
#define MRQ_RG_FLOATS (2 * MRQ_RG_STAGE)       // >= 32 * 33 (the unaligned fallback's tile)
#define MRQ_QS(D) (((D) + 1) & ~1)              // doubles of a staged query row (16-B multiple)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <class SlotOf, class Init, class Done>
__device__ __forceinline__ void warp_gather_rows(const float *__restrict__ base, int64_t stride, int off, int len,
                                                 const double *__restrict__ q, int n, float *sbuf, SlotOf slot_of,
                                                 Init init, Done done, int g0 = 0, int gs = 1)
{
    // groups g0, g0 + gs, g0 + 2 gs, ... of 32 entries (several warps can split one list)
    const int lane = threadIdx.x & 31;
    const int nchunk = (len + MRQ_RG_CH - 1) / MRQ_RG_CH;
    const int ngroups = (n + 31) / 32;
    const int mygroups = ngroups > g0 ? (ngroups - g0 + gs - 1) / gs : 0;
    const int njobs = mygroups * nchunk;
    if (njobs == 0) return;
    // slots are loaded one group ahead (slot_nxt), so the index load's
    // latency is hidden behind the current group's copies
    auto load_slot = [&](int g) -> uint32_t {
        const int e = g * 32 + lane;
        return e < n ? slot_of(e) : 0u;
    };
    uint32_t slot_cur = 0, slot_nxt = load_slot(g0);
    // job (g, c): 32 rows x MRQ_RG_CH floats; lane copies 16-B unit (lane & 7)
    // of rows (lane >> 3) + 4 i, i = 0..7 (one 128-B row segment per 8 lanes).
    auto issue = [&](int job, int g, int c) {
        const int c0 = c * MRQ_RG_CH;
        const int nu = min(MRQ_RG_CH, len - c0) >> 2;
        const int st = job & 1;
        if (c == 0) {
            slot_cur = slot_nxt;
            slot_nxt = load_slot(g + gs);
        }
        const int cnt = min(32, n - g * 32);
        const int u = lane & 7;
        float *dst0 = sbuf + st * MRQ_RG_STAGE + 4 * u;
        const float *src0 = base + off + c0 + 4 * u;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const int r = (lane >> 3) + 4 * i;
            const uint32_t s = __shfl_sync(0xffffffffu, slot_cur, r);
#pragma unroll
            for (int uu = 0; uu < MRQ_RG_CH / 32; uu++)   // 128-B segments of the row chunk
                if (r < cnt && u + 8 * uu < nu) {
                    const unsigned d = smem_u32(dst0 + 32 * uu + r * MRQ_RG_STRIDE);
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d),
                                 "l"(src0 + 32 * uu + (int64_t)s * stride)
                                 : "memory");
                }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    issue(0, g0, 0);
    double acc = 0.0;
    uint32_t slot_row = slot_cur;
    int g = g0, c = 0;           // current job
    int gi = g0, ci = 0;         // last issued job
    for (int job = 0; job < njobs; job++) {
        const int e = g * 32 + lane;
        const bool v = e < n;
        if (c == 0) slot_row = slot_cur;
        if (job + 1 < njobs) {
            if (++ci == nchunk) {
                ci = 0;
                gi += gs;
            }
            issue(job + 1, gi, ci);
        }
        const int st = job & 1;
        if (c == 0 && v) acc = init(e, slot_row);
        if (job + 1 < njobs)
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        else
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncwarp();
        const int c0 = c * MRQ_RG_CH;
        const int cl = min(MRQ_RG_CH, len - c0);
        const float *row = sbuf + st * MRQ_RG_STAGE + lane * MRQ_RG_STRIDE;
        const double *qq = q + c0;
        if (v) {
#pragma unroll 4
            for (int u = 0; u < cl; u += 4) {
                const float4 x = *(const float4 *)(row + u);
                const double2 qa = *(const double2 *)(qq + u);
                const double2 qb = *(const double2 *)(qq + u + 2);
                const double t0 = (double)x.x - qa.x, t1 = (double)x.y - qa.y;
                const double t2 = (double)x.z - qb.x, t3 = (double)x.w - qb.y;
                acc = acc + t0 * t0;
                acc = acc + t1 * t1;
                acc = acc + t2 * t2;
                acc = acc + t3 * t3;
            }
        }
        __syncwarp();   // the stage is refilled by the next issue
        if (c == nchunk - 1) done(e, v, acc);
        if (++c == nchunk) {
            c = 0;
            g += gs;
        }
    }
}

// Row gather dispatcher: the pipelined cp.async path when the shapes allow
// 16-byte copies, else the register-staged path (same arithmetic, same order).
template <class SlotOf, class Init, class Done>
__device__ __forceinline__ void warp_rows(bool aligned, const float *__restrict__ base, int64_t stride, int off,
                                          int len, const double *__restrict__ q, int n, float *sbuf, SlotOf slot_of,
                                          Init init, Done done, int g0 = 0, int gs = 1)
{
    if (aligned) {
        warp_gather_rows(base, stride, off, len, q, n, sbuf, slot_of, init, done, g0, gs);
        return;
    }
    const int lane = threadIdx.x & 31;
    for (int g = g0 * 32; g < n; g += 32 * gs) {
        const int e = g + lane;
        const bool v = e < n;
        const uint32_t slot = v ? slot_of(e) : 0u;
        double acc = v ? init(e, slot) : 0.0;
        acc = warp_rows_sqdist(base, stride, off, slot, v, len, q, acc, sbuf);
        done(e, v, acc);
    }
}

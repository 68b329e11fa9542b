// mrq_internal.cuh -- internal declarations of libmrq (B200 / sm_100a).
//
// Everything here is the product path.  It shares nothing with oracle/.
// The numeric contract requires that every
// fp64 expression that decides a code bit, a level, a flag or an ordering is
// evaluated left to right without contraction; the library is compiled with
// --fmad=false and the expressions below spell out their evaluation order.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <string>
#include <vector>

#include "../../include/mrq.h"

#define MRQ_BQ 4                 // query bit-planes (levels 0..15), R-7
#define MRQ_MAX_K 1024
#define MRQ_MAX_NPROBE 1024
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

// ------------------------------------------------------------ index object
struct DevArr {
    void *p = nullptr;
    size_t bytes = 0;
};

struct mrq_index {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[12] = {};
    int64_t N = 0, npad = 0;
    int D = 0, d = 0, k = 0, W = 0;
    int rank = 0, world = 1;
    void *nccl_comm = nullptr;
    int sm_count = 148;

    // host mirrors
    std::vector<uint32_t> h_list_off, h_list_size;
    uint32_t max_list = 0;
    double cmax = 0.0;           // max_j ||c_j|| (rounded up), probe error bound

    // device index (HBM layout)
    double *mu = nullptr, *PT = nullptr, *lam = nullptr, *RT = nullptr;   // PT[j][i] = P[i][j], RT[i][j] = R[j][i]
    double *C = nullptr, *Rc = nullptr;                                   // C[k][d], Rc[k][d]
    float *C32T = nullptr;                                                // C32T[i][k] fp32 centroids, transposed
    float *C32 = nullptr;                                                 // C32[k][d] fp32 centroids (GEMM B operand)
    float *cn32 = nullptr;                                                // ||c||^2 fp32 (GEMM epilogue)
    uint32_t *list_off = nullptr, *list_size = nullptr;                   // [k+1], [k]
    uint32_t *ids = nullptr;                                              // [npad] global id of each slot
    uint32_t *codes = nullptr;                                            // [W][npad]
    float *f1 = nullptr, *f2 = nullptr, *f3 = nullptr, *xr2 = nullptr;    // [npad]
    float *heads = nullptr, *tails = nullptr;                             // [npad][d], [npad][D-d]

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
// - q[e])^2, left to right (the oracle's order), with the rows staged through
// shared memory tile[32][33] so global loads are 128-byte coalesced.
__device__ __forceinline__ double warp_rows_sqdist(const float *__restrict__ base, int64_t stride, int off,
                                                   uint32_t slot_lane, bool valid, int len,
                                                   const double *q, double acc, float *tile)
{
    const int lane = threadIdx.x & 31;
    for (int c0 = 0; c0 < len; c0 += 32) {
        const int cl = min(32, len - c0);
        for (int r = 0; r < 32; r++) {
            uint32_t s = __shfl_sync(0xffffffffu, slot_lane, r);
            int v = __shfl_sync(0xffffffffu, (int)valid, r);
            if (v && lane < cl) tile[r * 33 + lane] = __ldg(base + (int64_t)s * stride + off + c0 + lane);
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

// mrq_probe_tc.cu -- the probe screen (Alg.2 L7, on the projected
// centroids of Alg.1 L6 P:286 / Exp-2 P:2405-2408) as a tcgen05 tensor-core
// GEMM on sm_100a.
//
//   approx[q][c] = ||c||^2 - 2 <q_d, c>        (fp32; the q-only term ||q_d||^2 is dropped)
//
// A = q_d, B = centroids, each split into tf32 parts (x = hi + lo + r, hi =
// RN_tf32(x), lo = RN_tf32(x - hi), |r| <= 2^-22 |x|) and laid out as
// A3 = [q_hi | q_hi | q_lo], B3 = [c_hi | c_lo | c_hi] (fp32 [rows][3d],
// K-major), so one K = 3d GEMM gives q_hi c_hi + q_hi c_lo + q_lo c_hi
// ("3xTF32": close to fp32 products instead of tf32 ones);
// kind::tf32 MMAs (M = 128 queries, N = 256 centroids, K = 8) accumulate in
// TMEM.  Warp roles (one CTA = one 128-query block x a range of 256-centroid
// tiles):
//   warp 0  TMA producer: 2-D tensor-map loads of A and B k-blocks (32 fp32 =
//           128 B rows, 128-byte swizzle) into a 4-stage smem ring;
//   warp 1  TMEM allocator + MMA issuer (one elected thread);
//   warps 2-5  epilogue: tcgen05.ld of the 128 x 256 accumulator (each thread
//           owns one query row), ||c||^2 - 2 acc, fp32 stores.
// Two TMEM accumulators (2 x 256 columns) let the epilogue of tile j overlap
// the MMAs of tile j+1.  Out-of-range rows/columns/k are zero-filled by TMA.
//
// Exactness (DESIGN.md §4 "probe exactness"): the three tf32 products (exact
// in fp32) differ from q32 c32 by <= 3.01 2^-22 |q32 c32| (the dropped
// q_lo c_lo and the lo residuals), the fp32 accumulation of 3d products adds
// <= 3d 2^-23 (1 + 2^-10) sum|q_i c_i|, and ||c||^2, q_d, c are fp32
// roundings of fp64 values; with sum|q_i c_i| <= ||q|| ||c|| <= (||q|| +
// ||c||)^2 / 4 the screen is within
//   delta_q = kappa (||q_d|| + max ||c||)^2,  kappa = 2^-20 + 3d 2^-23
// of the exact key ||c||^2 - 2 <q_d, c> (a generous bound: each term is at
// least 2x the derivation).  k_probe_select_w then rescores every centroid
// within 2 delta_q of the np-th smallest screen value in canonical fp64.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>

#include "mrq_probe_tc.cuh"

#define TC_BK 32                       // fp32 elements per 128-byte swizzle row
#define TC_STAGES 4
#define TC_A_BYTES (TC_BM * TC_BK * 4) // 16 KB
#define TC_B_BYTES (TC_BN * TC_BK * 4) // 32 KB
#define TC_STAGE_BYTES (TC_A_BYTES + TC_B_BYTES)
#define TC_THREADS 320                 // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue
#define TC_SMEM (TC_STAGES * TC_STAGE_BYTES + 1024 + 256 + 256 * 32 * 4)

struct ProbeTC {
    bool enabled = false;
    CUtensorMap mapB;                  // centroids, split: B3 [k][3d]
    float *B3 = nullptr;
    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
};

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t n)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity)
{
    uint32_t ok = 0;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(ok)
                     : "r"(su32(b)), "r"(parity)
                     : "memory");
    } while (!ok);
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            su32(dst)),
        "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(su32(bar))
        : "memory");
}
// K-major, 128-byte-swizzled operand: 8-row core groups 1024 B apart (SBO),
// LBO unused for swizzled K-major (1), descriptor version 1 (sm_100),
// layout type 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr)
{
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
// kind::tf32 instruction descriptor: D fp32, A/B tf32, both K-major, N, M.
__host__ __device__ constexpr uint32_t tf32_idesc(int M, int N)
{
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// Fused selection (FUSED = true, np <= NPM, NPM = 16 or TC_NPMAX = 64).  A
// row's columns are split into parts (CTA column range x epilogue half, at
// most P = 2 maxparts); the thread owning (row, part) keeps the np smallest
// screen values of its part sorted in NPM registers (NPM - np placeholders
// first) and appends every (a_c, c) with a_c <= RU(its current np-th
// smallest + 2 delta_q) to the part's candidate buffer.  A part's running
// np-th smallest never drops below the row's final a_(np), so every member of
// the margin set {c : a_c <= a_(np) + 2 delta_q} is appended by its part; the
// parts' np smallest go to kvbuf ([row][part][np]) so that k_probe_finish_w
// can form a_(np) and rescore the margin set.  The parts of a row share
// their bounds: each publishes its running np-th smallest to gkey[row]
// (atomicMin on order-preserving keys) and each tile starts from the
// smallest published one -- every published value is some part's running
// np-th smallest, so >= a_(np), and the append threshold stays valid.  (The
// parts are small -- a CTA range of a 256-column tile run split in two
// halves -- so a fresh part appends about np (1 + ln(n / np)) values; with
// the shared bound the parts a row reaches later start nearly converged.)
#define TC_NPMAX 64

template <bool FUSED, int NPM>
__global__ void __launch_bounds__(TC_THREADS, 1) k_probe_tc(const __grid_constant__ CUtensorMap mapA,
                                                            const __grid_constant__ CUtensorMap mapB, int nq, int k,
                                                            int d, int G, int maxparts, const float *__restrict__ cn32,
                                                            float *__restrict__ approx, int np,
                                                            const double *__restrict__ qnorm, double cmax,
                                                            double kappa, uint2 *__restrict__ cbuf, int capp,
                                                            uint32_t *__restrict__ ccnt, float *__restrict__ kvbuf,
                                                            uint32_t *__restrict__ gkey)
{
    extern __shared__ __align__(1024) unsigned char tsm[];
    unsigned char *ring = (unsigned char *)(((uintptr_t)tsm + 1023) & ~(uintptr_t)1023);
    uint64_t *full = (uint64_t *)(ring + TC_STAGES * TC_STAGE_BYTES);
    uint64_t *empty = full + TC_STAGES;
    uint64_t *tfull = empty + TC_STAGES;    // [2]
    uint64_t *tempty = tfull + 2;           // [2]
    uint32_t *tmem_slot = (uint32_t *)(tempty + 2);
    float *scratch = (float *)(tmem_slot + 4);   // FUSED: 256 x 32 floats (per-thread chunk staging)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = (k + TC_BN - 1) / TC_BN;
    const int64_t U = (int64_t)((nq + TC_BM - 1) / TC_BM) * ntiles;
    const int64_t ub = tc_u0(blockIdx.x, U, G), ue = tc_u0((int64_t)blockIdx.x + 1, U, G);
    const int kb_n = (d + TC_BK - 1) / TC_BK;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < TC_STAGES; s++) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(tfull + b, 1);
            mbar_init(tempty + b, 8);       // one arrival per epilogue warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"((uint64_t)&mapA) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"((uint64_t)&mapB) : "memory");
    }
    if (warp == 1) {   // TMEM: 2 accumulators x 256 fp32 columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {   // ---------------- TMA producer
            int s = 0;
            uint32_t ph = 0;
            for (int64_t u = ub; u < ue; u++) {
                const int mb = (int)(u / ntiles), t = (int)(u % ntiles);
                for (int kb = 0; kb < kb_n; kb++) {
                    mbar_wait(empty + s, ph ^ 1u);
                    unsigned char *sa = ring + s * TC_STAGE_BYTES;
                    mbar_expect_tx(full + s, TC_STAGE_BYTES);
                    tma_load_2d(sa, &mapA, full + s, kb * TC_BK, mb * TC_BM);
                    tma_load_2d(sa + TC_A_BYTES, &mapB, full + s, kb * TC_BK, t * TC_BN);
                    if (++s == TC_STAGES) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {   // ---------------- MMA issuer
            constexpr uint32_t idesc = tf32_idesc(TC_BM, TC_BN);
            int s = 0;
            uint32_t ph = 0;
            int it = 0;
            for (int64_t u = ub; u < ue; u++, it++) {
                const int b = it & 1;
                mbar_wait(tempty + b, (((uint32_t)it >> 1) & 1u) ^ 1u);
                asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                const uint32_t dt = tmem + (uint32_t)(b * TC_BN);
                for (int kb = 0; kb < kb_n; kb++) {
                    mbar_wait(full + s, ph);
                    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                    const uint32_t sa = su32(ring + s * TC_STAGE_BYTES);
                    const uint32_t sb = sa + TC_A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < TC_BK / 8; kk++) {
                        const uint64_t da = sw128_desc(sa + kk * 32);
                        const uint64_t db = sw128_desc(sb + kk * 32);
                        const uint32_t acc = (kb > 0 || kk > 0) ? 1u : 0u;
                        asm volatile(
                            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                            " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(dt),
                            "l"(da), "l"(db), "r"(idesc), "r"(acc)
                            : "memory");
                    }
                    // frees the smem stage once these MMAs have read it
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                                     su32(empty + s))
                                 : "memory");
                    if (++s == TC_STAGES) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                                 su32(tfull + b))
                             : "memory");
            }
        }
    } else {   // ---------------------------- epilogue warps 2..5
        const int quad = warp & 3;            // TMEM lanes 32 quad .. 32 quad + 31
        const int half = (warp - 2) >> 2;     // column chunks half, half + 2, ... of each tile
        const int P = 2 * maxparts;
        const float FINF = __int_as_float(0x7f800000);
        float kv[NPM];                        // FUSED: the np smallest screen values, ascending
        float tf = FINF;                      // FUSED: append threshold RU(kv[np-1] + margin)
        uint32_t cnt = 0;
        float margin = 0.f;                   // RU(2 delta_q): th + margin rounded up >= th + 2 delta_q
        uint2 *rb = nullptr;
        int row = 0, part = 0, cur_mb = -1;
        // FUSED: the (row, part) state goes to kvbuf / ccnt when the query block changes
        auto flush = [&]() {
            if (FUSED && cur_mb >= 0 && row < nq) {
                ccnt[(int64_t)row * P + part] = cnt;
                float *kvo = kvbuf + ((int64_t)row * P + part) * np;
#pragma unroll
                for (int i = 0; i < NPM; i++)   // the np values after the NPM - np placeholders
                    if (i >= NPM - np) kvo[i - (NPM - np)] = kv[i];
            }
        };
        int it = 0;
        for (int64_t u = ub; u < ue; u++, it++) {
            const int mb = (int)(u / ntiles), t = (int)(u % ntiles);
            if (mb != cur_mb) {
                flush();
                cur_mb = mb;
                row = mb * TC_BM + quad * 32 + lane;
                part = 2 * (int)(blockIdx.x - tc_owner((int64_t)mb * ntiles, U, G)) + half;
                cnt = 0;
                tf = FINF;
                if (FUSED) {
                    // kv holds NPM - np placeholders (-inf) followed by the np smallest
                    // values, so the running np-th smallest is always kv[NPM - 1]
#pragma unroll
                    for (int j = 0; j < NPM; j++) kv[j] = j < NPM - np ? -FINF : FINF;
                    if (row < nq) {
                        const double g = qnorm[row] + cmax;
                        margin = __double2float_ru(2.0 * (kappa * (g * g)));
                        rb = cbuf + ((int64_t)row * P + part) * capp;
                    }
                }
            }
            if (FUSED && gkey && row < nq) {   // the row's shared bound, published by any part
                const uint32_t gk = __ldcg(gkey + row);
                if (gk < 0xFF800000u) tf = fminf(tf, __fadd_ru(key2f(gk), margin));
            }
            const int b = it & 1;
            mbar_wait(tfull + b, ((uint32_t)it >> 1) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            const int n0 = t * TC_BN;
#pragma unroll 1
            for (int c = half * 32; c < TC_BN; c += 64) {
                uint32_t v[32];
                const uint32_t ta = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(b * TC_BN + c);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                      "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                      "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                      "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                      "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                    : "r"(ta));
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                if (FUSED) {
                    // screen values of the chunk; mask of those <= the append threshold
                    // (2 acc is exact, so the fma rounds exactly like cn - 2 acc;
                    // cn32 is padded with +inf past k, so padded columns never pass)
                    float av[32];
                    float mn = FINF;
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        const float4 cn = __ldg((const float4 *)(cn32 + n0 + c + j));
                        av[j] = __fmaf_rn(-2.0f, __uint_as_float(v[j]), cn.x);
                        av[j + 1] = __fmaf_rn(-2.0f, __uint_as_float(v[j + 1]), cn.y);
                        av[j + 2] = __fmaf_rn(-2.0f, __uint_as_float(v[j + 2]), cn.z);
                        av[j + 3] = __fmaf_rn(-2.0f, __uint_as_float(v[j + 3]), cn.w);
                        mn = fminf(fminf(mn, fminf(av[j], av[j + 1])), fminf(av[j + 2], av[j + 3]));
                    }
                    uint32_t mask = 0;
                    if (mn <= tf && row < nq) {
#pragma unroll
                        for (int j = 0; j < 32; j++) mask |= av[j] <= tf ? (1u << j) : 0u;
                    }
                    if (mask) {   // rare after warm-up: stage the chunk, walk the passing values
                        // the thread's 32 values as 8 16-byte stores; chunk u of the row
                        // goes to position u ^ (lane & 7), so the 8 lanes of a quarter-warp
                        // hit distinct bank groups
                        float *sc = scratch + ((warp - 2) * 32 + lane) * 32;
                        const int sw = lane & 7;
#pragma unroll
                        for (int u = 0; u < 8; u++)
                            *(float4 *)(sc + 4 * (u ^ sw)) = make_float4(av[4 * u], av[4 * u + 1], av[4 * u + 2], av[4 * u + 3]);
                        while (mask) {
                            const int j = __ffs(mask) - 1;
                            mask &= mask - 1;
                            const float a = sc[4 * ((j >> 2) ^ sw) + (j & 3)];
                            if (!(a <= tf)) continue;
                            if (cnt < (uint32_t)capp) rb[cnt] = make_uint2(__float_as_uint(a), (uint32_t)(n0 + c + j));
                            cnt++;
                            if (a < kv[NPM - 1]) {   // insertion (compare-exchange chain)
                                float x = a;
#pragma unroll
                                for (int i = 0; i < NPM; i++) {
                                    const float lo = fminf(kv[i], x);
                                    x = fmaxf(kv[i], x);
                                    kv[i] = lo;
                                }
                                const float th = kv[NPM - 1];
                                tf = fminf(tf, __fadd_ru(th, margin));   // +inf stays +inf
                                if (gkey && th < FINF) atomicMin(gkey + row, f2key(th));
                            }
                        }
                    }
                } else if (row < nq) {
                    float *dst = approx + (int64_t)row * k + n0 + c;
                    if (n0 + c + 32 <= k && (k & 3) == 0) {
#pragma unroll
                        for (int j = 0; j < 32; j += 4) {
                            const float4 cn = __ldg((const float4 *)(cn32 + n0 + c + j));
                            float4 o;
                            o.x = cn.x - 2.0f * __uint_as_float(v[j]);
                            o.y = cn.y - 2.0f * __uint_as_float(v[j + 1]);
                            o.z = cn.z - 2.0f * __uint_as_float(v[j + 2]);
                            o.w = cn.w - 2.0f * __uint_as_float(v[j + 3]);
                            *(float4 *)(dst + j) = o;
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; j++)
                            if (n0 + c + j < k) dst[j] = cn32[n0 + c + j] - 2.0f * __uint_as_float(v[j]);
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty + b);
        }
        flush();
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// ------------------------------------------------------------------ host
static int make_map(ProbeTC *tc, CUtensorMap *map, const float *ptr, int rows, int d, int box_rows)
{
    cuuint64_t gdim[2] = {(cuuint64_t)d, (cuuint64_t)rows};
    cuuint64_t gstride[1] = {(cuuint64_t)d * 4};
    cuuint32_t box[2] = {TC_BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = tc->encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)ptr, gdim, gstride, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        mrq_set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
        return MRQ_ECUDA;
    }
    return MRQ_OK;
}

// B3 row c = [c_hi | c_lo | c_hi] (see the header comment)
__global__ void k_split3_b(const float *__restrict__ C32, int k, int d, float *__restrict__ B3)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)k * d) return;
    const int64_t c = i / d;
    const int j = (int)(i % d);
    float hi, lo;
    tf32_split(C32[i], hi, lo);
    B3[c * 3 * d + j] = hi;
    B3[c * 3 * d + d + j] = lo;
    B3[c * 3 * d + 2 * d + j] = hi;
}

int mrq_probe_tc_init(mrq_index *ix)
{
    ix->probe_tc = nullptr;
    // TMA needs 16-byte row strides; the tensor-core screen is used when d % 4 == 0
    if (ix->d % 4 != 0) return MRQ_OK;
    ProbeTC *tc = new ProbeTC();
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) != cudaSuccess || !fn ||
        qr != cudaDriverEntryPointSuccess) {
        delete tc;
        mrq_set_error("cuTensorMapEncodeTiled unavailable");
        return MRQ_ECUDA;
    }
    tc->encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    const int d3 = 3 * ix->d;
    if (cudaMalloc(&tc->B3, (size_t)ix->k * d3 * 4) != cudaSuccess) {
        delete tc;
        mrq_set_error("cudaMalloc B3");
        return MRQ_ENOMEM;
    }
    k_split3_b<<<(unsigned)(((int64_t)ix->k * ix->d + 255) / 256), 256, 0, ix->stream>>>(ix->C32, ix->k, ix->d, tc->B3);
    MRQ_CUDA_TRY(cudaStreamSynchronize(ix->stream));
    int rc = make_map(tc, &tc->mapB, tc->B3, ix->k, d3, TC_BN);
    if (rc != MRQ_OK) {
        cudaFree(tc->B3);
        delete tc;
        return rc;
    }
    cudaError_t e = cudaFuncSetAttribute(k_probe_tc<false, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_probe_tc<true, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_probe_tc<true, TC_NPMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM);
    if (e != cudaSuccess) {
        delete tc;
        mrq_set_error("k_probe_tc smem attribute: %s", cudaGetErrorString(e));
        return MRQ_ECUDA;
    }
    tc->enabled = true;
    ix->probe_tc = tc;
    return MRQ_OK;
}

void mrq_probe_tc_free(mrq_index *ix)
{
    ProbeTC *tc = (ProbeTC *)ix->probe_tc;
    if (tc && tc->B3) cudaFree(tc->B3);
    delete tc;
    ix->probe_tc = nullptr;
}

bool mrq_probe_tc_enabled(const mrq_index *ix)
{
    return ix->probe_tc && ((const ProbeTC *)ix->probe_tc)->enabled && !ix->force_cuda_core_probe;
}

double mrq_probe_tc_kappa(const mrq_index *ix)
{
    return std::ldexp(1.0, -20) + 3.0 * (double)ix->d * std::ldexp(1.0, -23);
}

// G <= 7 x (query blocks): a block's tiles then span at most 8 CTAs, i.e. at
// most 16 parts per row (the finisher's limit)
static int tc_grid(const mrq_index *ix, int64_t nq)
{
    const int64_t mblocks = (nq + TC_BM - 1) / TC_BM;
    const int64_t U = mblocks * (int64_t)((ix->k + TC_BN - 1) / TC_BN);
    return (int)std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(ix->sm_count, U), 7 * mblocks));
}

int mrq_probe_tc_run(mrq_index *ix, const float *qd32, int64_t nq, float *approx, cudaStream_t st)
{
    ProbeTC *tc = (ProbeTC *)ix->probe_tc;
    CUtensorMap mapA;
    int rc = make_map(tc, &mapA, qd32, (int)nq, 3 * ix->d, TC_BM);
    if (rc != MRQ_OK) return rc;
    const int G = tc_grid(ix, nq);
    k_probe_tc<false, 16><<<G, TC_THREADS, TC_SMEM, st>>>(mapA, tc->mapB, (int)nq, ix->k, 3 * ix->d, G, 1, ix->cn32, approx,
                                                       0, nullptr, 0.0, 0.0, nullptr, 0, nullptr, nullptr, nullptr);
    MRQ_CUDA_TRY(cudaGetLastError());
    return MRQ_OK;
}

// per-part candidate buffer: a part of n columns appends about np (1 + ln(n /
// np)) values (running top-np records) plus the margin set; 256 covers np <=
// 16, 8 np beyond (an overflow only costs a full rescore of the row)
int mrq_probe_tc_capp(const mrq_index *ix, int np) { return std::max(ix->probe_capp, ix->probe_capp == 256 ? 8 * np : 0); }

bool mrq_probe_tc_fusable(const mrq_index *ix, int np)
{
    return mrq_probe_tc_enabled(ix) && np <= TC_NPMAX && !ix->force_probe_unfused;
}

// parts per query row = 2 x (most CTAs any query block's tiles span)
int mrq_probe_tc_parts(const mrq_index *ix, int64_t nq)
{
    const int64_t mblocks = (nq + TC_BM - 1) / TC_BM, ntiles = (ix->k + TC_BN - 1) / TC_BN;
    const int64_t U = mblocks * ntiles, G = tc_grid(ix, nq);
    int64_t mx = 1;
    for (int64_t mb = 0; mb < mblocks; mb++)
        mx = std::max(mx, tc_owner((mb + 1) * ntiles - 1, U, G) - tc_owner(mb * ntiles, U, G) + 1);
    return (int)(2 * mx);
}

int mrq_probe_tc_run_fused(mrq_index *ix, const float *qd32, int64_t nq, int np, const double *qnorm, double kappa,
                           uint2 *cbuf, int capp, uint32_t *ccnt, float *kvbuf, uint32_t *gkey, cudaStream_t st)
{
    ProbeTC *tc = (ProbeTC *)ix->probe_tc;
    CUtensorMap mapA;
    int rc = make_map(tc, &mapA, qd32, (int)nq, 3 * ix->d, TC_BM);
    if (rc != MRQ_OK) return rc;
    const int G = tc_grid(ix, nq);
    const int maxparts = mrq_probe_tc_parts(ix, nq) / 2;
    if (gkey) MRQ_CUDA_TRY(cudaMemsetAsync(gkey, 0xFF, (size_t)nq * 4, st));   // no bound published yet
    auto fn = np <= 16 ? k_probe_tc<true, 16> : k_probe_tc<true, TC_NPMAX>;
    fn<<<G, TC_THREADS, TC_SMEM, st>>>(mapA, tc->mapB, (int)nq, ix->k, 3 * ix->d, G, maxparts, ix->cn32, nullptr, np,
                                        qnorm, ix->cmax, kappa, cbuf, capp, ccnt, kvbuf, gkey);
    MRQ_CUDA_TRY(cudaGetLastError());
    return MRQ_OK;
}

int mrq_probe_tc_grid(const mrq_index *ix, int64_t nq) { return tc_grid(ix, nq); }

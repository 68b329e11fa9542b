// mrq_kernels.cu -- the B200 kernels of the batched IVF-MRQ query path.
//
// Citations "P:N" are lines of the paper's LaTeX source.  Every
// fp64 expression keeps the evaluation order written here (compiled with
// --fmad=false), which is the canonical order of DESIGN.md: sums run left to
// right over increasing index, products and sums round separately.
#include "mrq_internal.cuh"
#include "mrq_kernels.cuh"
#include "mrq_comm.cuh"

// ===================================================================== a0/a1
// Row-matrix products in the canonical order:
//   out[r][i] = sum_{j=0}^{Din-1} (x[r][j] - mu[j]) * MT[j][i]    (mu optional)
// accumulated j ascending (acc = acc + u p, separately rounded).  Used for
// x_p = P (x - mu) (Alg.1 L3 P:283 for base vectors, Alg.2 L1 P:303 for
// queries; MT = P^T) and for r0 = R q_d (Alg.2 L4 P:306; MT = R^T, mu = 0).
// Register-tiled across rows and outputs only, which leaves each output's
// reduction order untouched: a 32-row x 64-output tile per 128-thread block,
// 4 x 4 outputs per thread, j in shared-memory chunks of 16 (8 shared loads
// feed 16 products); the next chunk's global loads are issued before the
// current chunk is consumed.  Padded j (beyond Din) contribute exact zeros,
// which never change a sum that starts at +0.
#define PJ_TR 32   // rows per block tile (32 x 64 tiles, 128 threads: ~4 resident blocks per SM, no tail wave)
#define PJ_TC 64   // outputs per block tile
#define PJ_K 16
#define PJ_NT ((PJ_TR / 4) * (PJ_TC / 4))
template <typename TIn>
__global__ void __launch_bounds__(PJ_NT) k_rowmat(const TIn *__restrict__ X, int64_t nrows, int ldx, int Din,
                                                  const double *__restrict__ mu, const double *__restrict__ MT,
                                                  int Dout, double *__restrict__ out, int ldo)
{
    __shared__ double us[PJ_K][PJ_TR + 1];
    __shared__ double ps[PJ_K][PJ_TC + 1];
    constexpr int NU = PJ_TR * PJ_K / PJ_NT, NP = PJ_K * PJ_TC / PJ_NT;
    const int tid = threadIdx.x;
    const int tx = tid % (PJ_TC / 4), ty = tid / (PJ_TC / 4);
    const int i0 = blockIdx.x * PJ_TC;
    const int64_t r0 = (int64_t)blockIdx.y * PJ_TR;
    double acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; r++)
#pragma unroll
        for (int c = 0; c < 4; c++) acc[r][c] = 0.0;
    double ur[NU], pr[NP];
    auto fetch = [&](int j0) {
#pragma unroll
        for (int k = 0; k < NU; k++) {
            const int t = tid + PJ_NT * k;
            const int rr = t / PJ_K, jj = t % PJ_K;
            const int64_t r = r0 + rr;
            const int j = j0 + jj;
            ur[k] = 0.0;
            if (r < nrows && j < Din) ur[k] = mu ? ((double)X[r * ldx + j] - mu[j]) : (double)X[r * ldx + j];
        }
#pragma unroll
        for (int k = 0; k < NP; k++) {
            const int t = tid + PJ_NT * k;
            const int ii = t % PJ_TC, jq = t / PJ_TC;
            const int i = i0 + ii, jp = j0 + jq;
            pr[k] = (jp < Din && i < Dout) ? MT[(int64_t)jp * Dout + i] : 0.0;
        }
    };
    fetch(0);
    for (int j0 = 0; j0 < Din; j0 += PJ_K) {
#pragma unroll
        for (int k = 0; k < NU; k++) {
            const int t = tid + PJ_NT * k;
            us[t % PJ_K][t / PJ_K] = ur[k];
        }
#pragma unroll
        for (int k = 0; k < NP; k++) {
            const int t = tid + PJ_NT * k;
            ps[t / PJ_TC][t % PJ_TC] = pr[k];
        }
        __syncthreads();
        if (j0 + PJ_K < Din) fetch(j0 + PJ_K);
#pragma unroll
        for (int jj = 0; jj < PJ_K; jj++) {
            double a[4], b[4];
#pragma unroll
            for (int r = 0; r < 4; r++) a[r] = us[jj][ty + (PJ_TR / 4) * r];
#pragma unroll
            for (int c = 0; c < 4; c++) b[c] = ps[jj][tx + (PJ_TC / 4) * c];
#pragma unroll
            for (int r = 0; r < 4; r++)
#pragma unroll
                for (int c = 0; c < 4; c++) acc[r][c] = acc[r][c] + a[r] * b[c];
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 4; r++) {
        const int64_t row = r0 + ty + (PJ_TR / 4) * r;
        if (row >= nrows) continue;
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const int i = i0 + tx + (PJ_TC / 4) * c;
            if (i < Dout) out[row * ldo + i] = acc[r][c];
        }
    }
}

void launch_rowmat_f32(const float *X, int64_t nrows, int ldx, int Din, const double *mu, const double *MT, int Dout,
                       double *out, int ldo, cudaStream_t st)
{
    const int64_t CH = (int64_t)65535 * PJ_TR;   // grid.y limit
    for (int64_t r = 0; r < nrows; r += CH) {
        const int64_t n = nrows - r < CH ? nrows - r : CH;
        dim3 grid((Dout + PJ_TC - 1) / PJ_TC, (unsigned)((n + PJ_TR - 1) / PJ_TR));
        k_rowmat<float><<<grid, PJ_NT, 0, st>>>(X + r * ldx, n, ldx, Din, mu, MT, Dout, out + r * ldo, ldo);
    }
}

void launch_rowmat_f64(const double *X, int64_t nrows, int ldx, int Din, const double *mu, const double *MT,
                       int Dout, double *out, int ldo, cudaStream_t st)
{
    const int64_t CH = (int64_t)65535 * PJ_TR;   // grid.y limit
    for (int64_t r = 0; r < nrows; r += CH) {
        const int64_t n = nrows - r < CH ? nrows - r : CH;
        dim3 grid((Dout + PJ_TC - 1) / PJ_TC, (unsigned)((n + PJ_TR - 1) / PJ_TR));
        k_rowmat<double><<<grid, PJ_NT, 0, st>>>(X + r * ldx, n, ldx, Din, mu, MT, Dout, out + r * ldo, ldo);
    }
}

// ======================================================================= a0
// Head sketch (an acceleration structure of the stage-2 gather, DESIGN.md
// §5 "head sketch"; not part of the paper's method).  HEAD = ||h - q_d||^2 of
// the STORED fp32 head h is rotation invariant, so it is sketched in the
// quantizer's rotated frame, where the query side R (q_d - c) already exists
// (k_quant_g): y = R (h - c) (fp64, the encoder's matvec on the fp32 head),
// quantized to signed int8 levels a_i (|a_i| <= 127; padding to dq bytes is
// 0) with a per-vector scale s (fp32, rounded up from max|y| / 127) and a
// rigorous bound E >= ||R (h - c) - s a||_2 (fp32, rounded up; it covers the
// rounding of the fp64 matvec and of the quantization residual).  The scan
// turns it into a lower bound of the canonical HEAD that prunes stage-2
// candidates without reading the fp32 head row; every candidate it cannot
// prune is decided by the canonical fp64 HEAD, so F2 is unchanged.  Warp per
// vector; y (d doubles, shared memory) is the rotated residual.
__device__ void mrq_head_sketch(const double *y, double ynorm_bound, float xr2, int d, int dq, uint8_t *out,
                                float4 *se)
{
    const int lane = threadIdx.x & 31;
    double mx = 0.0;
    for (int i = lane; i < d; i += 32) mx = fmax(mx, fabs(y[i]));
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float s = mx > 0.0 ? __double2float_ru(mx / 127.0) : 0.f;
    double e2 = 0.0;
    int aa = 0;   // <a, a> (<= 512 * 127^2 < 2^24: exact in the fp32 record)
    for (int i = lane; i < dq; i += 32) {
        int a = 0;
        if (i < d && s > 0.f) {
            const double q = rint(y[i] / (double)s);
            a = (int)fmin(127.0, fmax(-127.0, q));
            const double e = y[i] - (double)s * (double)a;
            e2 = e2 + e * e;
        } else if (i < d) {
            e2 = e2 + y[i] * y[i];
        }
        out[i] = (uint8_t)(int8_t)a;
        aa += a * a;
    }
    for (int o = 16; o > 0; o >>= 1) e2 = e2 + __shfl_xor_sync(0xffffffffu, e2, o);
    for (int o = 16; o > 0; o >>= 1) aa += __shfl_xor_sync(0xffffffffu, aa, o);
    if (lane == 0) {
        // margins: the fp64 residual e per element <= 2^-50 mx; the matvec
        // y_j = sum_i R_ji (h_i - c_i) (d terms, |R_j| = 1) per element <=
        // (d + 2) 2^-53 ||h - c|| <= (d + 2) 2^-52 ynorm_bound
        const double E = __dsqrt_ru(e2) * (1.0 + 0x1p-40) + 0x1p-49 * mx * sqrt((double)d) +
                         0x1p-50 * (double)(d + 2) * sqrt((double)d) * ynorm_bound;
        *se = make_float4(s, __double2float_ru(E), xr2, (float)aa);   // (s, E, ||x_r||^2, <a,a>)
    }
    __syncwarp();
}

// Alg.1 L4-L8, one warp per vector, results scattered to the
// vector's list slot.  t = x_d - c_{a(x)}; y = R t (y_j = sum_i R[j][i] t_i);
// bit_j = [y_j >= 0]; u = <x_bar, x_b> = sum|y_j| / (sqrt(d) ||t||), clamped
// to 1, = 1 when t = 0; stored fp32 factors f1 = ||t||^2 + ||x_r||^2,
// f2 = ||t||/u, f3 = ||t|| sqrt(1-u^2)/(u sqrt(d-1)) (Eq.4/Eq.5 readings
// A-1/A-2 of DESIGN.md).
__global__ void k_encode_finish(const double *__restrict__ xp, int64_t n0, int64_t cnt, int D, int d, int W,
                                const uint32_t *__restrict__ assign, const uint32_t *__restrict__ slot_of,
                                const double *__restrict__ C, const double *__restrict__ RT, int64_t npad,
                                float *__restrict__ heads, float *__restrict__ tails, float *__restrict__ xr2o,
                                uint32_t *__restrict__ codes, float *__restrict__ f1, float *__restrict__ f2,
                                float *__restrict__ f3, uint8_t *__restrict__ hq, float4 *__restrict__ hs, int dq)
{
    extern __shared__ double esm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t v = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (v >= cnt) return;
    double *t = esm + (size_t)warp * 2 * d;
    double *y = t + d;
    const double *row = xp + v * D;
    const int64_t n = n0 + v;
    const uint32_t c = assign[n];
    const int64_t slot = slot_of[n];
    for (int i = lane; i < d; i += 32) {
        t[i] = row[i] - C[(int64_t)c * d + i];
        heads[slot * d + i] = (float)row[i];
    }
    for (int i = d + lane; i < D; i += 32) tails[slot * (D - d) + (i - d)] = (float)row[i];
    __syncwarp();
    for (int w = 0; w < W; w++) {
        const int j = w * 32 + lane;
        double acc = 0.0;
        if (j < d) {
            for (int i = 0; i < d; i++) acc = acc + RT[(int64_t)i * d + j] * t[i];
            y[j] = acc;
        }
        unsigned bits = __ballot_sync(0xffffffffu, j < d && acc >= 0.0);
        if (lane == 0) codes[(int64_t)w * npad + slot] = bits;
    }
    __syncwarp();
    float xr2f = 0.f;   // lane 0: fp32 ||x_r||^2 (the sketch record carries a copy)
    if (lane == 0) {
        double xr2 = 0.0;
        for (int i = d; i < D; i++) xr2 = xr2 + row[i] * row[i];
        double n2 = 0.0;
        for (int i = 0; i < d; i++) n2 = n2 + t[i] * t[i];
        double abssum = 0.0;
        for (int j = 0; j < d; j++) abssum = abssum + fabs(y[j]);
        double u = 1.0;
        if (n2 != 0.0) {
            u = abssum / (sqrt((double)d) * sqrt(n2));
            if (u > 1.0) u = 1.0;
        }
        const double nrm = sqrt(n2);
        xr2f = (float)xr2;
        xr2o[slot] = xr2f;
        f1[slot] = (float)(n2 + xr2);
        f2[slot] = (float)(nrm / u);
        f3[slot] = (float)(nrm * (sqrt(1.0 - u * u) / (u * sqrt((double)(d - 1)))));
    }
    __syncwarp();   // lane 0's sums above read t and y; the sketch reuses them
    if (hq) {
        // y = R (h - c) for the fp32 head h (the sketch's rotated residual)
        double hn2 = 0.0;
        for (int i = lane; i < d; i += 32) {
            t[i] = (double)(float)row[i] - C[(int64_t)c * d + i];
            hn2 = hn2 + t[i] * t[i];
        }
        for (int o = 16; o > 0; o >>= 1) hn2 = hn2 + __shfl_xor_sync(0xffffffffu, hn2, o);
        __syncwarp();
        for (int j = lane; j < d; j += 32) {
            double acc = 0.0;
            for (int i = 0; i < d; i++) acc = acc + RT[(int64_t)i * d + j] * t[i];
            y[j] = acc;
        }
        __syncwarp();
        mrq_head_sketch(y, sqrt(hn2) * (1.0 + 0x1p-40), xr2f, d, dq, hq + slot * dq, hs + slot);
    }
}

// R c_j for every centroid (warp per centroid): Rc[c][j] = sum_i R[j][i] C[c][i].
__global__ void k_rc(const double *__restrict__ C, const double *__restrict__ RT, int k, int d, int W,
                     double *__restrict__ Rc)
{
    const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (c >= k) return;
    for (int w = 0; w < W; w++) {
        const int j = w * 32 + lane;
        if (j < d) {
            double acc = 0.0;
            for (int i = 0; i < d; i++) acc = acc + RT[(int64_t)i * d + j] * C[(int64_t)c * d + i];
            Rc[(int64_t)c * d + j] = acc;
        }
    }
}

// ======================================================================= a1
// Alg.2 L2-L4, warp per query: ||q_r||^2, sigma^2 = sum_{i>=d}
// q_i^2 lambda_i (Eq.6), eps_r = (resid_scale m) sigma (Eq.7 / Alg.2
// L11, reading R-4); plus the fp32 q_d and ||q_d|| the probe uses (r0 = R q_d
// is k_rowmat).  The query row and lambda are staged in shared memory; the
// three left-to-right sums run on three lanes at once.
__global__ void __launch_bounds__(256) k_qtail(const double *__restrict__ qp, int64_t nq, int D, int d, int W,
                                               const double *__restrict__ lam, const double *__restrict__ RT,
                                               double rscale, double m, double *__restrict__ qr2o,
                                               double *__restrict__ eps_r, double *__restrict__ r0,
                                               float *__restrict__ qd32, double *__restrict__ qnorm,
                                               uint16_t *__restrict__ qkey, float *__restrict__ qa3)
{
    extern __shared__ double qsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    double *lams = qsm;                        // D
    for (int i = threadIdx.x; i < D; i += blockDim.x) lams[i] = lam[i];
    __syncthreads();
    const int64_t q = (int64_t)blockIdx.x * wpb + warp;
    if (q >= nq) return;
    double *row = qsm + D + (size_t)warp * D;
    const double *g = qp + q * D;
    for (int i = lane; i < D; i += 32) row[i] = g[i];
    for (int j = lane; j < d; j += 32) {
        const float x = (float)g[j];
        qd32[q * d + j] = x;
        if (qa3) {   // the tensor-core probe's A3 row [q_hi | q_hi | q_lo]
            float hi, lo;
            tf32_split(x, hi, lo);
            qa3[q * 3 * d + j] = hi;
            qa3[q * 3 * d + d + j] = hi;
            qa3[q * 3 * d + 2 * d + j] = lo;
        }
    }
    __syncwarp();
    if (lane == 0) {
        double a = 0.0;
        for (int i = d; i < D; i++) a = a + row[i] * row[i];
        qr2o[q] = a;
    } else if (lane == 1) {
        double s2 = 0.0;
        for (int i = d; i < D; i++) s2 = s2 + (row[i] * row[i]) * lams[i];
        eps_r[q] = (rscale * m) * sqrt(s2);
    } else if (lane == 2) {
        double n2 = 0.0;
        for (int i = 0; i < d; i++) n2 = n2 + row[i] * row[i];
        qnorm[q] = sqrt(n2);
    } else if (lane == 3 && qkey) {
        qkey[q] = (uint16_t)mrq_qorder_key(row, lams, D);
    }
}

// ======================================================================= a2
// Probe screen on CUDA cores (fallback when the tcgen05 GEMM is not used):
// approx[q][c] = sum_i (q~_i - c~_i)^2 in fp32 with q~, c~ the fp32 roundings.
// The exact selection happens in k_probe_select.
__global__ void __launch_bounds__(256) k_probe_approx(const float *__restrict__ qd32, int64_t nq, int d, int k,
                                                      const float *__restrict__ C32T, float *__restrict__ approx)
{
    constexpr int QB = 8;
    extern __shared__ float qs[];   // QB x d
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t q0 = (int64_t)blockIdx.y * QB;
    for (int i = threadIdx.x; i < QB * d; i += blockDim.x) {
        int64_t q = q0 + i / d;
        qs[i] = q < nq ? qd32[q * d + i % d] : 0.f;
    }
    __syncthreads();
    if (c >= k) return;
    float acc[QB];
#pragma unroll
    for (int b = 0; b < QB; b++) acc[b] = 0.f;
    for (int i = 0; i < d; i++) {
        const float cv = C32T[(int64_t)i * k + c];
#pragma unroll
        for (int b = 0; b < QB; b++) {
            float t = qs[b * d + i] - cv;
            acc[b] = acc[b] + t * t;
        }
    }
#pragma unroll
    for (int b = 0; b < QB; b++)
        if (q0 + b < nq) approx[(q0 + b) * k + c] = acc[b];
}

// ======================================================================= a3
// Per (query, probed list) (Alg.2 L4-L5; readings R-7): r = R q_d - R c (unnormalized), lo/hi = min/max r,
// delta = (hi - lo)/15, L_j = clamp(floor((r_j - lo)/delta + 0.5), 0, 15)
// (all 0 when delta = 0), bit-planes p_b = {j : bit b of L_j}, and the
// constants of the scan epilogue:
//   A = 2 lo, Bc = 2 delta, C0 = d lo + delta sum L, g1 = ||q_d-c||^2 + ||q_r||^2,
//   eb = (2 eps0) ||q_d - c||          (Eq.5 distance-domain scale, R-5)
// G lanes per (query, list) pair (32 / G pairs per warp): lane s of a pair
// holds the E consecutive coordinates j = s E .. s E + E - 1 (E = 8 for d <= 256, 16 up to 512; G = the power of two >= d / E).  min/max
// and sum L reduce over the G lanes (exact: fmin/fmax and integers), the
// level expression is the same per coordinate, and a plane word (32 bits)
// is assembled from 32 / E lanes.
template <int E>
__global__ void __launch_bounds__(256) k_quant_g(const uint32_t *__restrict__ probe,
                                                 const double *__restrict__ probe_qn2, int64_t npairs, int np, int d,
                                                 int W, int G, const double *__restrict__ r0,
                                                 const double *__restrict__ Rc, const double *__restrict__ qr2,
                                                 double eps0, uint32_t *__restrict__ planes,
                                                 double *__restrict__ qconst, uint8_t *__restrict__ qsk_b,
                                                 double *__restrict__ qsk_c, int dq, const double *__restrict__ qnorm,
                                                 double cmax)
{
    const int lane = threadIdx.x & 31;
    const int P = 32 / G;
    const int sub = lane / G, s = lane - sub * G;
    const int64_t gw = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * P + sub;
    const bool pv = gw < npairs;
    const int64_t q = pv ? gw / np : 0;
    const uint32_t c = pv ? probe[gw] : 0xFFFFFFFFu;
    const bool ok = c != 0xFFFFFFFFu;
    const double INF = __longlong_as_double(0x7ff0000000000000ll);
    double rv[E];
    double lo = INF, hi = -INF;
#pragma unroll
    for (int t = 0; t < E; t++) {
        const int j = s * E + t;
        rv[t] = 0.0;
        if (ok && j < d) {
            rv[t] = r0[q * d + j] - Rc[(int64_t)c * d + j];
            lo = fmin(lo, rv[t]);
            hi = fmax(hi, rv[t]);
        }
    }
    for (int o = G >> 1; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o, G));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o, G));
    }
    const double delta = (hi - lo) / 15.0;
    // level = floor((r - lo) / delta + 0.5), canonical (IEEE division).  Fast
    // path: y = (r - lo) * (1/delta) + 0.5 is within 1e-14 of the canonical
    // fl(fl((r - lo) / delta) + 0.5) (both quotients <= 15); unless y is
    // within 1e-12 of an integer the two floors agree, else divide.
    const double inv = delta > 0.0 ? 1.0 / delta : 0.0;
    int sumL = 0;
    uint32_t bits[MRQ_BQ] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int t = 0; t < E; t++) {
        const int j = s * E + t;
        int v = 0;
        if (ok && j < d && delta > 0.0) {
            const double y = (rv[t] - lo) * inv + 0.5;
            double f = floor(y);
            if (y - f < 1e-12 || f + 1.0 - y < 1e-12) f = floor((rv[t] - lo) / delta + 0.5);
            v = f < 0.0 ? 0 : (f > 15.0 ? 15 : (int)f);
        }
        sumL += v;
#pragma unroll
        for (int b = 0; b < MRQ_BQ; b++) bits[b] |= (uint32_t)((v >> b) & 1) << t;
    }
    for (int o = G >> 1; o > 0; o >>= 1) sumL += __shfl_xor_sync(0xffffffffu, sumL, o, G);
    const int L = 32 / E;                     // lanes per plane word
    const int Lg = L < G ? L : G;
    const int w = s / L;
#pragma unroll
    for (int b = 0; b < MRQ_BQ; b++) {
        uint32_t x = bits[b] << ((s % L) * E);
        for (int o = 1; o < Lg; o <<= 1) x |= __shfl_xor_sync(0xffffffffu, x, o, G);
        if (pv && s % L == 0 && w < W) planes[gw * (MRQ_BQ * W) + b * W + w] = ok ? x : 0u;
    }
    if (qsk_b) {
        // the query side of the head sketch (mrq_head_sketch):
        // r = R (q_d - c) = t b + f, b int8 (|b_j| <= 127), ||f|| <= F
        // (rounded up; margins cover the fp64 rounding of f and of r0 - Rc)
        const double mx = fmax(fabs(lo), fabs(hi));
        const double tq = (ok && mx > 0.0) ? mx / 127.0 : 0.0;
        // any int8 b is valid (F bounds the residual of the b actually chosen),
        // so the level uses a reciprocal multiply, not a division
        const double itq = tq > 0.0 ? 1.0 / tq : 0.0;
        double f2 = 0.0;
        int B = 0;
        uint32_t pk[E / 4];
#pragma unroll
        for (int w = 0; w < E / 4; w++) pk[w] = 0u;
#pragma unroll
        for (int t = 0; t < E; t++) {
            const int j = s * E + t;
            int b = 0;
            if (ok && j < d) {
                if (tq > 0.0) b = (int)fmin(127.0, fmax(-127.0, rint(rv[t] * itq)));
                const double f = rv[t] - tq * (double)b;
                f2 = f2 + f * f;
            }
            B += b * b;
            pk[t / 4] |= (uint32_t)(uint8_t)(int8_t)b << (8 * (t % 4));
        }
        for (int o = G >> 1; o > 0; o >>= 1) {
            f2 = f2 + __shfl_xor_sync(0xffffffffu, f2, o, G);
            B += __shfl_xor_sync(0xffffffffu, B, o, G);
        }
        if (pv && s * E < dq) {
            uint32_t *dst = (uint32_t *)(qsk_b + gw * dq + s * E);
#pragma unroll
            for (int w = 0; w < E / 4; w++) dst[w] = pk[w];
        }
        if (pv && s == 0) {
            // r0 = R q_d and R c are d-term fp64 dots (|R_j| = 1): per element
            // <= (d + 1) 2^-53 (||q_d|| + ||c||), plus 2^-53 |r_j| for r0 - Rc
            const double sd = sqrt((double)d);
            qsk_c[gw * 4 + 0] = tq;
            qsk_c[gw * 4 + 1] = __dsqrt_ru(f2) * (1.0 + 0x1p-40) + 0x1p-49 * mx * sd +
                                0x1p-50 * (double)(d + 2) * sd * (qnorm[q] + cmax);
            qsk_c[gw * 4 + 2] = (double)B;
            qsk_c[gw * 4 + 3] = 0.0;
        }
    }
    if (pv && s == 0) {
        double *qc = qconst + gw * 8;
        if (!ok) {
            for (int i = 0; i < 8; i++) qc[i] = 0.0;
        } else {
            const double qn2 = probe_qn2[gw];
            qc[0] = 2.0 * lo;                                  // A
            qc[1] = 2.0 * delta;                               // Bc
            qc[2] = (double)d * lo + delta * (double)sumL;     // C0
            qc[3] = qn2 + qr2[q];                              // g1
            qc[4] = (2.0 * eps0) * sqrt(qn2);                  // eb
            qc[5] = lo;
            qc[6] = delta;
            qc[7] = (double)sumL;
        }
    }
}

void launch_quant(const uint32_t *probe, const double *probe_qn2, int64_t nq, int np, int d, int W,
                  const double *r0, const double *Rc, const double *qr2, double eps0, uint32_t *planes,
                  double *qconst, uint8_t *qsk_b, double *qsk_c, int dq, const double *qnorm, double cmax,
                  cudaStream_t st)
{
    const int64_t npairs = nq * np;
    const int E = d <= 256 ? 8 : 16;
    int G = 1;
    while (G * E < d) G <<= 1;
    if (G > 32) G = 32;
    const int P = 32 / G;
    const int64_t warps = (npairs + P - 1) / P;
    const unsigned grid = (unsigned)((warps + 7) / 8);
    if (E == 8)
        k_quant_g<8><<<grid, 256, 0, st>>>(probe, probe_qn2, npairs, np, d, W, G, r0, Rc, qr2, eps0, planes, qconst,
                                           qsk_b, qsk_c, dq, qnorm, cmax);
    else
        k_quant_g<16><<<grid, 256, 0, st>>>(probe, probe_qn2, npairs, np, d, W, G, r0, Rc, qr2, eps0, planes, qconst,
                                            qsk_b, qsk_c, dq, qnorm, cmax);
}

// Processing order of the queries (a permutation; every query's result is
// independent of it): a counting sort on the 12-bit key k_qtail computes
// (mrq_qorder_key).  Queries close in the leading PCs probe mostly the same
// lists, so the list-major kernels that follow (scan, head gather, re-rank)
// run neighbouring queries at the same time and share the lists' codes and
// rows in L2.  One block; order within a key is arbitrary.
__device__ __forceinline__ void dev_qorder(const uint16_t *__restrict__ qkey, int64_t nq,
                                           uint32_t *__restrict__ order)
{
    __shared__ uint32_t hist[MRQ_QO_KEYS];
    __shared__ uint32_t wsum[32];
    for (int i = threadIdx.x; i < MRQ_QO_KEYS; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int64_t q = threadIdx.x; q < nq; q += blockDim.x) atomicAdd(&hist[qkey[q]], 1u);
    __syncthreads();
    // exclusive scan of hist (MRQ_QO_KEYS / blockDim.x consecutive keys per thread)
    const int per = MRQ_QO_KEYS / blockDim.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t loc = 0;
    for (int j = 0; j < per; j++) loc += hist[threadIdx.x * per + j];
    uint32_t x = loc;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        wsum[lane] = w;
    }
    __syncthreads();
    uint32_t run = (warp > 0 ? wsum[warp - 1] : 0) + x - loc;
    for (int j = 0; j < per; j++) {
        const uint32_t c = hist[threadIdx.x * per + j];
        hist[threadIdx.x * per + j] = run;
        run += c;
    }
    __syncthreads();
    for (int64_t q = threadIdx.x; q < nq; q += blockDim.x) order[atomicAdd(&hist[qkey[q]], 1u)] = (uint32_t)q;
}

__global__ void __launch_bounds__(1024) k_qorder(const uint16_t *__restrict__ qkey, int64_t nq,
                                                 uint32_t *__restrict__ order)
{
    dev_qorder(qkey, nq, order);
}

void launch_qorder(const uint16_t *qkey, int64_t nq, uint32_t *order, cudaStream_t st)
{
    k_qorder<<<1, 1024, 0, st>>>(qkey, nq, order);
}

// Candidate count per query (sum of its probed list sizes) ...
// qkey (qorder = 2): also the query's order key, the locality key of its
// nearest probed list (list_key, built at load time from the centroids:
// mrq_api.cu list_locality_keys).  Queries whose nearest lists are close
// share most of their np probed lists, whatever the dimension; the key from
// three principal coordinates (mrq_qorder_key) separates them poorly when
// the spectrum is flat.
__global__ void k_cand_count(const uint32_t *__restrict__ probe, int64_t nq, int np,
                             const uint32_t *__restrict__ list_size, uint64_t *__restrict__ cnt,
                             const uint16_t *__restrict__ list_key, uint16_t *__restrict__ qkey)
{
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    if (qkey) {
        const uint32_t c0 = probe[q * np];
        qkey[q] = c0 == 0xFFFFFFFFu ? (uint16_t)0 : list_key[c0];
    }
    uint64_t s = 0;
    for (int p = 0; p < np; p++) {
        uint32_t c = probe[q * np + p];
        if (c != 0xFFFFFFFFu) s += list_size[c];
    }
    cnt[q] = s;
}

// ... and its exclusive prefix sum (one block; out[nq] = total).
__device__ __forceinline__ void dev_exclusive_scan(const uint64_t *__restrict__ in, int64_t n,
                                                   uint64_t *__restrict__ out)
{
    // thread t owns the contiguous run [t per, (t + 1) per): its total, a
    // block scan of the totals, then the run's prefixes -- two passes over in[]
    __shared__ uint64_t wsum[32];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t per = (n + blockDim.x - 1) / blockDim.x;
    const int64_t i0 = t * per, i1 = i0 + per < n ? i0 + per : n;
    uint64_t loc = 0;
#pragma unroll 8
    for (int64_t i = i0; i < i1; i++) loc += in[i];
    uint64_t x = loc;
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint64_t w = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        wsum[lane] = w;
    }
    __syncthreads();
    uint64_t run = (warp > 0 ? wsum[warp - 1] : 0) + x - loc;
    for (int64_t i = i0; i < i1; i++) {
        out[i] = run;
        run += in[i];
    }
    if (t == (int)blockDim.x - 1) out[n] = run;
}

__global__ void __launch_bounds__(1024) k_exclusive_scan(const uint64_t *__restrict__ in, int64_t n,
                                                         uint64_t *__restrict__ out)
{
    dev_exclusive_scan(in, n, out);
}

// The two single-block passes of the side stream in one launch of two blocks
// (block 0: the F1 segment offsets; block 1: the query order from qkey): two
// 1024-thread blocks find room beside the quantizer's blocks sooner one after
// the other than two dependent launches do.
__global__ void __launch_bounds__(1024) k_offsets_order(const uint64_t *__restrict__ cnt, int64_t nq,
                                                        uint64_t *__restrict__ off,
                                                        const uint16_t *__restrict__ qkey,
                                                        uint32_t *__restrict__ order)
{
    if (blockIdx.x == 0)
        dev_exclusive_scan(cnt, nq, off);
    else
        dev_qorder(qkey, nq, order);
}

// Sketch arguments of the fused scan (SK = true; LOOSE FULL, tau1 = tau0):
// every F1 candidate is immediately tested against the head-sketch lower
// bound of its canonical dis_o' (mrq_sketch_decide); F1 is only counted
// (f1_cnt), and the candidates the bound cannot prune are appended to f1_pos
// (count surv_cnt) for the canonical fp32 head gather of k_head_b.
struct ScanSketch {
    const uint8_t *hq;      // [npad][dq] int8 sketch rows
    const float4 *hs;       // [npad] (s, E, ||x_r||^2, <a,a>): one 16-byte gather
    const uint8_t *qsk_b;   // [nq][np][dq] query-side int8 rows
    const double *qsk_c;    // [nq][np][4] (t, F, <b,b>, 0)
    const double *qr2;      // [nq]
    int dq;
    uint32_t *surv_cnt;     // [nq]
    int pshift;             // a queue entry is (probe index << pshift) | slot (launch_scan_ws)
};

// Head-sketch test of one F1 candidate (DESIGN.md §5 "head sketch"): in the
// quantizer's rotated frame R (h - q_d) = R (h - c) - R (q_d - c) with
// R (h - c) = s a + e (||e|| <= E, mrq_head_sketch) and R (q_d - c) = t b + f
// (||f|| <= F, k_quant_g), so by the triangle inequality
//   ||h - q_d|| >= ||s a - t b|| - E - F,
//   ||s a - t b||^2 = s^2 <a,a> - 2 s t <a,b> + t^2 <b,b>,
// the inner products exact in int32 (dp4a over the packed bytes; |<a,b>| <=
// d 127^2 < 2^31) and the fp64 combination's rounding bounded by 2^-50 times
// the sum of the magnitudes.  The canonical fp64 HEAD (k_head_b) is >= (lower
// bound)^2 (1 - 2^-40), and fl(fl(fl(HEAD + xr2) + qr2) - eps_r) is monotone
// in HEAD under round-to-nearest, so a candidate whose bound already fails
// the F2 test (dlo - eps_r >= tau1) is not in F2: the canonical test decides
// it the same way.  keep = true: the candidate must be gathered.
// <a,b> over one 16-byte chunk of packed int8 (<a,a> is the record's fourth field)
__device__ __forceinline__ void mrq_dp4a_ab(const uint4 &u, const uint4 &b, int &ab)
{
    ab = __dp4a((int)u.x, (int)b.x, ab);
    ab = __dp4a((int)u.y, (int)b.y, ab);
    ab = __dp4a((int)u.z, (int)b.z, ab);
    ab = __dp4a((int)u.w, (int)b.w, ab);
}
__device__ __forceinline__ bool mrq_sketch_decide(int ab, int aa, float4 se, const double *bc, double qr2, double eps_r,
                                                  double tau1)
{
    const float xv = se.z;   // ||x_r||^2
    const double t = bc[0], F = bc[1], B = bc[2], sv = (double)se.x;
    const double y1 = (sv * sv) * (double)aa, y2 = (2.0 * sv * t) * (double)ab, y3 = (t * t) * B;
    const double y = (y1 - y2) + y3;
    const double ylo = y - 0x1p-50 * ((y1 + fabs(y2)) + y3);
    const double n = ylo > 0.0 ? sqrt(ylo) * (1.0 - 0x1p-50) : 0.0;
    const double L = (n - (double)se.y - F) * (1.0 - 0x1p-50);
    const double lb = L > 0.0 ? (L * L) * (1.0 - 0x1p-40) : 0.0;
    const double dlo = (lb + (double)xv) + qr2;
    return !(dlo - eps_r >= tau1);
}

// The code scan (hot loop of Alg.2 L7-L12): block per query, every
// warp streams (list, 128 H-slot) tiles of the query's probed lists.
// Each lane owns slots base + 128 h .. base + 128 h + 3 of its tile and reads
// them with 128-bit loads (W code words of the word-major planes
// codes[w][slot], then f1/f2/f3) before evaluating any, evaluates LB1 in
// registers and appends slots with LB1 < tau0 (stage 1, F1) to the query's
// segment of f1_pos.  Warp 0 builds the tile prefix of the probed lists in
// shared memory with a shuffle scan.  SK: F1 candidates go through a per-warp
// shared-memory queue and are sketch-tested 32 at a time (lane per
// candidate); only the survivors are appended (see ScanSketch).
// tiles of 128 H slots (H = 1 or 2, a template parameter): H = 2 keeps twice
// the loads in flight per lane, which pays when the code stream comes from
// DRAM (Deep-shaped: scan 0.79 -> 0.74 ms) and costs a little when it sits
// in L2 (SIFT-shaped: 0.315 -> 0.322 ms); launch_scan picks H = 2 when the
// index's code + factor stream exceeds 64 MB
#ifndef MRQ_SCAN_THREADS
#define MRQ_SCAN_THREADS 128   // 4 warps per query: a smaller end-of-query tail than 8 (measured)
#endif
#ifndef MRQ_SKQ
#define MRQ_SKQ 960            // per-warp sketch queue (4-byte entries), drained after the tile loop
#endif
#ifndef MRQ_SK_CB
#define MRQ_SK_CB 2            // 16-byte chunks of a sketch row loaded before any is used
#endif
template <int W, bool SK, int H>
__global__ void __launch_bounds__(MRQ_SCAN_THREADS, (W <= 3 ? 1024 / MRQ_SCAN_THREADS : 1)) k_scan(
    const uint32_t *__restrict__ probe, int np, int64_t npad, const uint32_t *__restrict__ list_off,
    const uint32_t *__restrict__ list_size, const uint32_t *__restrict__ codes, const float *__restrict__ f1,
    const float *__restrict__ f2, const float *__restrict__ f3, const uint32_t *__restrict__ planes,
    const double *__restrict__ qconst, const double *__restrict__ eps_r_arr, const double *__restrict__ tau0_arr,
    double isd, const uint64_t *__restrict__ f1_off, uint32_t *__restrict__ f1_cnt, uint32_t *__restrict__ f1_pos,
    const uint32_t *__restrict__ qorder, ScanSketch sk)
{
    extern __shared__ __align__(16) unsigned char csm[];
    double *qc_s = (double *)csm;                        // np x 5: the (query, list) constants
    double *skc_s = qc_s + np * 5;                       // SK: np x 3 sketch constants (t, F, <b,b>)
    uint32_t *pl_s = (uint32_t *)(skc_s + (SK ? np * 3 : 0));   // np x MRQ_BQ W: the query bit-planes
    uint32_t *tile_pre = pl_s + np * (MRQ_BQ * W);       // np + 1
    uint32_t *lst_start = tile_pre + np + 1;             // np
    uint32_t *lst_end = lst_start + np;                  // np
    // SK: np sketch rows of dq bytes, each padded by 16 bytes (rows of odd and even index fall
    // in different banks: a quarter-warp's 16-byte reads of 8 distinct rows do not conflict);
    // addressed as uint4 off the shared base so that the reads are LDS.128
    uint4 *skb4 = (uint4 *)csm + (((int)((unsigned char *)(lst_end + np) - csm) + 15) >> 4);
    const int skrow = SK ? sk.dq / 16 + 1 : 1;
    __shared__ uint32_t sh_cnt, sh_surv;
    // SK: per-warp queue of F1 entries, (probe index << pshift) | slot in one word
    __shared__ uint32_t skq[SK ? (MRQ_SCAN_THREADS / 32) * MRQ_SKQ : 1];
    const int64_t q = qorder ? (int64_t)qorder[blockIdx.x] : (int64_t)blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    // staged once per query: a warp switches list every tile or two
    for (int i = threadIdx.x; i < np * 5; i += blockDim.x) qc_s[i] = qconst[(q * np + i / 5) * 8 + i % 5];
    for (int i = threadIdx.x; i < np * (MRQ_BQ * W); i += blockDim.x) pl_s[i] = planes[q * np * (MRQ_BQ * W) + i];
    if (SK) {
        for (int i = threadIdx.x; i < np * 3; i += blockDim.x) skc_s[i] = sk.qsk_c[(q * np + i / 3) * 4 + i % 3];
        const uint4 *src = (const uint4 *)(sk.qsk_b + q * np * sk.dq);
        const int nw = sk.dq / 16;
        for (int i = threadIdx.x; i < np * nw; i += blockDim.x) skb4[(i / nw) * skrow + i % nw] = src[i];
    }
    if (warp == 0) {
        uint32_t carry = 0;
        for (int p0 = 0; p0 < np; p0 += 32) {
            const int p = p0 + lane;
            uint32_t nt = 0, st = 0, sz = 0;
            if (p < np) {
                const uint32_t c = probe[q * np + p];
                if (c != 0xFFFFFFFFu) {
                    st = list_off[c];
                    sz = list_size[c];
                    nt = (sz + 128 * H - 1) / (128 * H);
                }
            }
            uint32_t x = nt;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (p < np) {
                tile_pre[p] = carry + x - nt;
                lst_start[p] = st;
                lst_end[p] = st + sz;
            }
            carry += __shfl_sync(0xffffffffu, x, 31);
        }
        if (lane == 0) {
            tile_pre[np] = carry;
            sh_cnt = 0;
            sh_surv = 0;
        }
    }
    __syncthreads();
    const double eps_r = eps_r_arr[q], tau0 = tau0_arr[q];
    uint32_t *out = f1_pos + f1_off[q];
    const uint32_t ntiles = tile_pre[np];
    int p = 0;
    uint32_t pl[MRQ_BQ * W];
    double qc[5];
    int cur_p = -1;
    // SK: the warp's queue of F1 candidates awaiting the sketch test
    uint32_t *wq = skq + warp * MRQ_SKQ;
    const int pshift = SK ? sk.pshift : 0;
    const uint32_t smask = SK ? (pshift < 32 ? (1u << pshift) - 1u : 0xFFFFFFFFu) : 0u;
    int qn = 0;
    const double qr2 = SK ? sk.qr2[q] : 0.0;
    // SK: sketch-test queue entries [i0, i0 + 64): two per lane, both rows in
    // flight before any arithmetic; survivors appended to f1_pos
    auto drain = [&](int i0) {
        const int nw = sk.dq / 16;
        uint32_t slot[2];
        int pp[2];
        bool in[2];
        float4 se[2];
        int ab[2] = {0, 0}, aa[2] = {0, 0};
#pragma unroll
        for (int u = 0; u < 2; u++) {
            const int i = i0 + u * 32 + lane;
            in[u] = i < qn;
            const uint32_t e = in[u] ? wq[i] : 0u;
            slot[u] = e & smask;
            pp[u] = pshift < 32 ? (int)(e >> pshift) : 0;
            se[u] = in[u] ? sk.hs[slot[u]] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        for (int w0 = 0; w0 < nw; w0 += MRQ_SK_CB) {   // MRQ_SK_CB chunks x 2 entries of loads in flight
            uint4 r[2][MRQ_SK_CB];
#pragma unroll
            for (int u = 0; u < 2; u++)
#pragma unroll
                for (int c = 0; c < MRQ_SK_CB; c++)
                    r[u][c] = (in[u] && w0 + c < nw) ? __ldg((const uint4 *)(sk.hq + (int64_t)slot[u] * sk.dq) + w0 + c)
                                                     : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
            for (int u = 0; u < 2; u++)
#pragma unroll
                for (int c = 0; c < MRQ_SK_CB; c++)
                    if (w0 + c < nw) mrq_dp4a_ab(r[u][c], skb4[pp[u] * skrow + w0 + c], ab[u]);
        }
#pragma unroll
        for (int u = 0; u < 2; u++) aa[u] = (int)se[u].w;
#pragma unroll
        for (int u = 0; u < 2; u++) {
            const bool keep = in[u] && mrq_sketch_decide(ab[u], aa[u], se[u], skc_s + pp[u] * 3, qr2, eps_r, tau0);
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (bal) {
                uint32_t o = 0;
                if (lane == 0) o = atomicAdd(&sh_surv, (uint32_t)__popc(bal));
                o = __shfl_sync(0xffffffffu, o, 0) + __popc(bal & ((1u << lane) - 1u));
                if (keep) {
                MRQ_ASSERT(o < (uint32_t)(f1_off[q + 1] - f1_off[q]) && slot[u] < npad);
                out[o] = slot[u];
            }
            }
        }
    };
    for (uint32_t t = warp; t < ntiles; t += nwarps) {
        while (tile_pre[p + 1] <= t) p++;
        if (p != cur_p) {
            cur_p = p;
            const uint32_t *g = pl_s + p * (MRQ_BQ * W);
#pragma unroll
            for (int i = 0; i < MRQ_BQ * W; i++) pl[i] = g[i];
            const double *gc = qc_s + p * 5;
#pragma unroll
            for (int i = 0; i < 5; i++) qc[i] = gc[i];
        }
        const uint32_t lend = lst_end[p];
        const uint32_t base = lst_start[p] + (t - tile_pre[p]) * (128 * H) + lane * 4;
        uint4 cw[H][W];
        float4 a1[H], a2[H], a3[H];
#pragma unroll
        for (int h = 0; h < H; h++) {
            const uint32_t b = base + h * 128;
#pragma unroll
            for (int w = 0; w < W; w++) cw[h][w] = __ldg((const uint4 *)(codes + (int64_t)w * npad + b));
            a1[h] = __ldg((const float4 *)(f1 + b));
            a2[h] = __ldg((const float4 *)(f2 + b));
            a3[h] = __ldg((const float4 *)(f3 + b));
        }
#pragma unroll
        for (int h = 0; h < H; h++) {
            const uint32_t b = base + h * 128;
            bool fl[4];
#pragma unroll
            for (int r = 0; r < 4; r++) {
                uint32_t code[W];
#pragma unroll
                for (int w = 0; w < W; w++)
                    code[w] = r == 0 ? cw[h][w].x : r == 1 ? cw[h][w].y : r == 2 ? cw[h][w].z : cw[h][w].w;
                const float v1 = r == 0 ? a1[h].x : r == 1 ? a1[h].y : r == 2 ? a1[h].z : a1[h].w;
                const float v2 = r == 0 ? a2[h].x : r == 1 ? a2[h].y : r == 2 ? a2[h].z : a2[h].w;
                const float v3 = r == 0 ? a3[h].x : r == 1 ? a3[h].y : r == 2 ? a3[h].z : a3[h].w;
                double dis;
                const double lb1 = mrq_lb1<W>(code, pl, qc, isd, eps_r, v1, v2, v3, &dis);
                fl[r] = (b + r < lend) && (lb1 < tau0);
            }
            const unsigned b0 = __ballot_sync(0xffffffffu, fl[0]), b1 = __ballot_sync(0xffffffffu, fl[1]);
            const unsigned b2 = __ballot_sync(0xffffffffu, fl[2]), b3 = __ballot_sync(0xffffffffu, fl[3]);
            const int n0 = __popc(b0), n1 = __popc(b1), n2 = __popc(b2), n3 = __popc(b3);
            const int tot = n0 + n1 + n2 + n3;
            if (tot) {
                const unsigned lt = (1u << lane) - 1u;
                if (SK && qn + tot <= MRQ_SKQ) {
                    // F1 is counted; its members queue for the sketch test after the tile loop
                    if (lane == 0) atomicAdd(&sh_cnt, (uint32_t)tot);
                    const uint32_t o0 = qn + __popc(b0 & lt), o1 = qn + n0 + __popc(b1 & lt);
                    const uint32_t o2 = qn + n0 + n1 + __popc(b2 & lt), o3 = qn + n0 + n1 + n2 + __popc(b3 & lt);
                    MRQ_ASSERT(qn + tot <= MRQ_SKQ);
                    const uint32_t e = b | (pshift < 32 ? (uint32_t)p << pshift : 0u);
                    if (fl[0]) wq[o0] = e;
                    if (fl[1]) wq[o1] = e + 1;
                    if (fl[2]) wq[o2] = e + 2;
                    if (fl[3]) wq[o3] = e + 3;
                    qn += tot;
                } else {
                    // (SK with a full queue: these F1 members skip the sketch test and are
                    // gathered -- the sketch only ever prunes, so F2 is unchanged)
                    uint32_t *ctr = SK ? &sh_surv : &sh_cnt;
                    if (SK && lane == 0) atomicAdd(&sh_cnt, (uint32_t)tot);
                    uint32_t wb = 0;
                    if (lane == 0) wb = atomicAdd(ctr, (uint32_t)tot);
                    wb = __shfl_sync(0xffffffffu, wb, 0);
                    const uint32_t o0 = wb + __popc(b0 & lt), o1 = wb + n0 + __popc(b1 & lt);
                    const uint32_t o2 = wb + n0 + n1 + __popc(b2 & lt), o3 = wb + n0 + n1 + n2 + __popc(b3 & lt);
                    MRQ_ASSERT(wb + tot <= (uint32_t)(f1_off[q + 1] - f1_off[q]));
                    if (fl[0]) out[o0] = b;
                    if (fl[1]) out[o1] = b + 1;
                    if (fl[2]) out[o2] = b + 2;
                    if (fl[3]) out[o3] = b + 3;
                }
            }
        }
    }
    if (SK) {
        __syncwarp();
        for (int i0 = 0; i0 < qn; i0 += 64) drain(i0);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        f1_cnt[q] = sh_cnt;
        if (SK) sk.surv_cnt[q] = sh_surv;
    }
}

// ------------------------------------------------------------ list-major scan
// The same F1 test (and the same fused sketch test) as k_scan, with the work
// grouped by LIST instead of by query (DESIGN.md §5 "list-major scan"): in a
// batch many queries probe the same list (Deep-shaped: 160k (query, list)
// pairs over 16384 lists), so a warp loads a 128-slot tile of a list's code
// words and factors once, keeps them in registers (factors widened to fp64
// once), and evaluates them against every query of its chunk of the list's
// pairs.  The code stream is read about once per list instead of once per
// pair, and the per-pair work is the AND+POPC + fp64 epilogue only.  Every
// decision is the canonical one (mrq_pop_S + the fp64 LB1 in the oracle's
// order), so F1 and the sketch survivors are the same sets as k_scan's; only
// their order in a query's segment differs (appends are atomic per query).

// pairs per list
__global__ void k_lm_count(const uint32_t *__restrict__ probe, int64_t npairs, const uint32_t *__restrict__ list_size,
                           uint32_t *__restrict__ lcnt)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npairs) return;
    const uint32_t c = probe[i];
    if (c != 0xFFFFFFFFu && list_size[c] > 0) atomicAdd(&lcnt[c], 1u);
}

// one block: exclusive prefixes of the pair counts (loff) and of the units
// (upre) over the k lists; clears the scatter fill counters and the unit counter
__global__ void __launch_bounds__(1024) k_lm_offsets(const uint32_t *__restrict__ lcnt,
                                                     const uint32_t *__restrict__ list_size, int k, int qg,
                                                     uint32_t *__restrict__ lfill, uint32_t *__restrict__ loff,
                                                     uint32_t *__restrict__ upre, uint32_t *__restrict__ unit_ctr)
{
    __shared__ uint32_t wsum[2][32];
    const int per = (k + blockDim.x - 1) / blockDim.x;
    const int c0 = threadIdx.x * per, c1 = min(k, c0 + per);
    uint32_t sp = 0, su = 0;
#pragma unroll 16
    for (int c = c0; c < c1; c++) {   // (unrolled: the loads of a thread's range are in flight together)
        const uint32_t n = lcnt[c];
        sp += n;
        su += ((list_size[c] + 127) / 128) * ((n + qg - 1) / qg);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t xp = sp, xu = su;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t yp = __shfl_up_sync(0xffffffffu, xp, o), yu = __shfl_up_sync(0xffffffffu, xu, o);
        if (lane >= o) {
            xp += yp;
            xu += yu;
        }
    }
    if (lane == 31) {
        wsum[0][warp] = xp;
        wsum[1][warp] = xu;
    }
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        uint32_t a = lane < nw ? wsum[0][lane] : 0u, b = lane < nw ? wsum[1][lane] : 0u;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t ya = __shfl_up_sync(0xffffffffu, a, o), yb = __shfl_up_sync(0xffffffffu, b, o);
            if (lane >= o) {
                a += ya;
                b += yb;
            }
        }
        wsum[0][lane] = a;   // inclusive warp prefixes
        wsum[1][lane] = b;
    }
    __syncthreads();
    uint32_t op = xp - sp + (warp ? wsum[0][warp - 1] : 0u), ou = xu - su + (warp ? wsum[1][warp - 1] : 0u);
#pragma unroll 16
    for (int c = c0; c < c1; c++) {
        const uint32_t n = lcnt[c];
        loff[c] = op;
        upre[c] = ou;
        lfill[c] = 0u;
        op += n;
        ou += ((list_size[c] + 127) / 128) * ((n + qg - 1) / qg);
    }
    if (threadIdx.x == blockDim.x - 1) {
        loff[k] = op;
        upre[k] = ou;
        *unit_ctr = 0u;
    }
}

__global__ void k_lm_scatter(const uint32_t *__restrict__ probe, int64_t npairs, const uint32_t *__restrict__ list_size,
                             const uint32_t *__restrict__ loff, uint32_t *__restrict__ lfill, uint32_t *__restrict__ pairs)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npairs) return;
    const uint32_t c = probe[i];
    if (c != 0xFFFFFFFFu && list_size[c] > 0) pairs[loff[c] + atomicAdd(&lfill[c], 1u)] = (uint32_t)i;
}

// unit -> list table (warp per list)
__global__ void k_lm_units(const uint32_t *__restrict__ upre, int k, uint32_t *__restrict__ unit_list)
{
    const int c = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (c >= k) return;
    const uint32_t e = upre[c + 1];
    for (uint32_t u = upre[c] + (threadIdx.x & 31); u < e; u += 32) unit_list[u] = (uint32_t)c;
}

int mrq_lm_build(const uint32_t *probe, int64_t nq, int np, int k, const uint32_t *list_size, int qg,
                 const LmScratch &s, cudaStream_t st)
{
    const int64_t npairs = nq * np;
    MRQ_CUDA_TRY(cudaMemsetAsync(s.lcnt, 0, (size_t)k * 4, st));
    if (npairs > 0)
        k_lm_count<<<(unsigned)((npairs + 255) / 256), 256, 0, st>>>(probe, npairs, list_size, s.lcnt);
    k_lm_offsets<<<1, 1024, 0, st>>>(s.lcnt, list_size, k, qg, s.lfill, s.loff, s.upre, s.unit_ctr);
    if (npairs > 0)
        k_lm_scatter<<<(unsigned)((npairs + 255) / 256), 256, 0, st>>>(probe, npairs, list_size, s.loff, s.lfill,
                                                                     s.pairs);
    k_lm_units<<<(unsigned)((k + 7) / 8), 256, 0, st>>>(s.upre, k, s.unit_list);
    MRQ_CUDA_TRY(cudaGetLastError());
    return MRQ_OK;
}

// the canonical fp64 LB1 from (pop, S) with the factors already widened
// (the same operations as mrq_lb1_ps: (double)f is exact)
__device__ __forceinline__ double mrq_lb1_psd(int pop, int S, const double *qc, double isd, double eps_r, double f1,
                                              double f2, double f3)
{
    const double t1 = qc[0] * i2d_exact(pop);
    const double t2 = qc[1] * i2d_exact(S);
    const double t4 = (t1 + t2) - qc[2];
    const double ip = t4 * isd;
    const double t5 = f1 + qc[3];
    const double t6 = f2 * ip;
    const double dis = t5 - 2.0 * t6;
    return (dis - qc[4] * f3) - eps_r;
}

#define MRQ_LM_RING 256   // per-warp ring of F1 entries awaiting the sketch test (power of 2, >= 64 + 128)
#ifndef MRQ_LM_MINB
#define MRQ_LM_MINB 6
#endif
template <int W, bool SK>
__global__ void __launch_bounds__(128, MRQ_LM_MINB) k_scan_lm(LaunchScan a)
{
    __shared__ uint2 ring[SK ? 4 * MRQ_LM_RING : 1];   // (slot, pair)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned FULL = 0xffffffffu;
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t np = (uint32_t)a.np;
    const double inv_np = 1.0 / (double)a.np;
    auto qof = [&](uint32_t pair) -> uint32_t {   // pair / np: fp64 estimate (off by at most one), one correction
        uint32_t q = (uint32_t)((double)pair * inv_np);
        const int32_t r = (int32_t)(pair - q * np);
        return r < 0 ? q - 1 : (r >= (int32_t)np ? q + 1 : q);
    };
    uint2 *wr = ring + warp * MRQ_LM_RING;
    uint32_t rh = 0, rt = 0;   // ring head / tail (warp-uniform, monotone)
    const uint32_t nunits = a.upre[a.k];
    // sketch test of ring entries [h0, h0 + n), n <= 64: two per lane, all
    // rows in flight before any arithmetic; survivors appended to their
    // query's segment (one atomic per query present in the batch)
    auto drain = [&](uint32_t h0, uint32_t n) {
        const int nw = a.dq / 16;
        uint32_t slot[2], pair[2], q[2];
        bool in[2];
        float4 se[2];
        int ab[2] = {0, 0};
#pragma unroll
        for (int u = 0; u < 2; u++) {
            const uint32_t i = u * 32 + lane;
            in[u] = i < n;
            const uint2 e = in[u] ? wr[(h0 + i) & (MRQ_LM_RING - 1)] : make_uint2(0u, 0u);
            slot[u] = e.x;
            pair[u] = e.y;
            q[u] = qof(e.y);
            se[u] = in[u] ? a.hs[slot[u]] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        for (int w0 = 0; w0 < nw; w0 += 2) {
            uint4 r[2][2], b[2][2];
#pragma unroll
            for (int u = 0; u < 2; u++)
#pragma unroll
                for (int c = 0; c < 2; c++) {
                    const bool ok = in[u] && w0 + c < nw;
                    r[u][c] = ok ? __ldg((const uint4 *)(a.hq + (int64_t)slot[u] * a.dq) + w0 + c) : make_uint4(0u, 0u, 0u, 0u);
                    b[u][c] = ok ? __ldg((const uint4 *)(a.qsk_b + (int64_t)pair[u] * a.dq) + w0 + c)
                                 : make_uint4(0u, 0u, 0u, 0u);
                }
#pragma unroll
            for (int u = 0; u < 2; u++)
#pragma unroll
                for (int c = 0; c < 2; c++)
                    if (w0 + c < nw) mrq_dp4a_ab(r[u][c], b[u][c], ab[u]);
        }
#pragma unroll
        for (int u = 0; u < 2; u++) {
            bool keep = false;
            if (in[u]) {
                const double *g = a.qsk_c + (int64_t)pair[u] * 4;
                const double bc[3] = {__ldg(g), __ldg(g + 1), __ldg(g + 2)};
                keep = mrq_sketch_decide(ab[u], (int)se[u].w, se[u], bc, __ldg(a.qr2 + q[u]), __ldg(a.eps_r + q[u]),
                                         __ldg(a.tau0 + q[u]));
            }
            if (__ballot_sync(FULL, keep)) {
                const unsigned grp = __match_any_sync(FULL, keep ? q[u] : 0xFFFFFFFFu);
                if (keep) {
                    const int leader = __ffs(grp) - 1;
                    uint32_t o = 0;
                    if (lane == leader) o = atomicAdd(&a.surv_cnt[q[u]], (uint32_t)__popc(grp));
                    o = __shfl_sync(grp, o, leader) + __popc(grp & lt);
                    MRQ_ASSERT(o < (uint32_t)(a.f1_off[q[u] + 1] - a.f1_off[q[u]]) && slot[u] < a.npad);
                    a.f1_pos[a.f1_off[q[u]] + o] = slot[u];
                }
            }
        }
    };
    for (;;) {
        uint32_t u = 0;
        if (lane == 0) u = atomicAdd(a.unit_ctr, 1u);
        u = __shfl_sync(FULL, u, 0);
        if (u >= nunits) break;
        const int c = (int)__ldg(a.unit_list + u);
        const uint32_t pb = __ldg(a.loff + c), pe = __ldg(a.loff + c + 1);
        const uint32_t nch = (pe - pb + a.qg - 1) / a.qg;
        const uint32_t local = u - __ldg(a.upre + c);
        const uint32_t tile = local / nch, ch = local - tile * nch;
        const uint32_t lst = __ldg(a.list_off + c), lend = lst + __ldg(a.list_size + c);
        const uint32_t b = lst + tile * 128 + lane * 4;
        uint4 cw[W];
#pragma unroll
        for (int w = 0; w < W; w++) cw[w] = __ldg((const uint4 *)(a.codes + (int64_t)w * a.npad + b));
        const float4 x1 = __ldg((const float4 *)(a.f1 + b)), x2 = __ldg((const float4 *)(a.f2 + b)),
                     x3 = __ldg((const float4 *)(a.f3 + b));
        const float d1[4] = {x1.x, x1.y, x1.z, x1.w}, d2[4] = {x2.x, x2.y, x2.z, x2.w},
                    d3[4] = {x3.x, x3.y, x3.z, x3.w};
        bool valid[4];
#pragma unroll
        for (int r = 0; r < 4; r++) valid[r] = b + r < lend;
        const uint32_t j1 = min(pe, pb + (ch + 1) * a.qg);
        for (uint32_t j = pb + ch * a.qg; j < j1; j++) {
            const uint32_t pair = __ldg(a.pairs + j);
            const uint32_t q = qof(pair);
            uint32_t pl[MRQ_BQ * W];
            {
                const uint4 *g = (const uint4 *)(a.planes + (int64_t)pair * (MRQ_BQ * W));
#pragma unroll
                for (int i = 0; i < W; i++) {
                    const uint4 v = __ldg(g + i);
                    pl[4 * i] = v.x;
                    pl[4 * i + 1] = v.y;
                    pl[4 * i + 2] = v.z;
                    pl[4 * i + 3] = v.w;
                }
            }
            double qc[5];
            {
                const double2 *g = (const double2 *)(a.qconst + (int64_t)pair * 8);
                const double2 v0 = __ldg(g), v1 = __ldg(g + 1), v2 = __ldg(g + 2);
                qc[0] = v0.x; qc[1] = v0.y; qc[2] = v1.x; qc[3] = v1.y; qc[4] = v2.x;
            }
            const double eps_r = __ldg(a.eps_r + q), tau0 = __ldg(a.tau0 + q);
            bool fl[4];
#pragma unroll
            for (int r = 0; r < 4; r++) {
                uint32_t code[W];
#pragma unroll
                for (int w = 0; w < W; w++) code[w] = r == 0 ? cw[w].x : r == 1 ? cw[w].y : r == 2 ? cw[w].z : cw[w].w;
                int pop, S;
                mrq_pop_S<W>(code, pl, pop, S);
                fl[r] = valid[r] && (mrq_lb1_psd(pop, S, qc, a.isd, eps_r, d1[r], d2[r], d3[r]) < tau0);
            }
            const unsigned b0 = __ballot_sync(FULL, fl[0]), b1 = __ballot_sync(FULL, fl[1]);
            const unsigned b2 = __ballot_sync(FULL, fl[2]), b3 = __ballot_sync(FULL, fl[3]);
            const int n0 = __popc(b0), n1 = __popc(b1), n2 = __popc(b2), n3 = __popc(b3);
            const int tot = n0 + n1 + n2 + n3;
            if (!tot) continue;
            uint32_t wb;
            if (SK) {
                if (lane == 0) atomicAdd(&a.f1_cnt[q], (uint32_t)tot);   // F1 is counted; members queue for the sketch
                wb = rt;
            } else {
                wb = 0;
                if (lane == 0) wb = atomicAdd(&a.f1_cnt[q], (uint32_t)tot);
                wb = __shfl_sync(FULL, wb, 0);
            }
            const uint32_t o0 = wb + __popc(b0 & lt), o1 = wb + n0 + __popc(b1 & lt);
            const uint32_t o2 = wb + n0 + n1 + __popc(b2 & lt), o3 = wb + n0 + n1 + n2 + __popc(b3 & lt);
            if (SK) {
                if (fl[0]) wr[o0 & (MRQ_LM_RING - 1)] = make_uint2(b, pair);
                if (fl[1]) wr[o1 & (MRQ_LM_RING - 1)] = make_uint2(b + 1, pair);
                if (fl[2]) wr[o2 & (MRQ_LM_RING - 1)] = make_uint2(b + 2, pair);
                if (fl[3]) wr[o3 & (MRQ_LM_RING - 1)] = make_uint2(b + 3, pair);
                rt += tot;
                __syncwarp();
                while (rt - rh >= 64) {
                    drain(rh, 64);
                    rh += 64;
                }
                __syncwarp();
            } else {
                uint32_t *out = a.f1_pos + a.f1_off[q];
                MRQ_ASSERT(wb + tot <= (uint32_t)(a.f1_off[q + 1] - a.f1_off[q]));
                if (fl[0]) out[o0] = b;
                if (fl[1]) out[o1] = b + 1;
                if (fl[2]) out[o2] = b + 2;
                if (fl[3]) out[o3] = b + 3;
            }
        }
    }
    if (SK) {
        __syncwarp();
        while (rt != rh) {
            const uint32_t n = min(64u, rt - rh);
            drain(rh, n);
            rh += n;
        }
    }
}

// ------------------------------------------------- list-major scan, tensor-core S
// Work unit = (list, 128-slot tile, chunk of <= 8 of the list's pairs).  The
// integer inner products are dense int8 contractions in this layout, so they
// run on the tensor cores (mma.sync m16n8k32 s8 -> s32, exact):
//   S[slot][pair]  = sum_i code_i(slot) * level_i(pair)   (codes as 0/1 bytes,
//                    levels 0..15 from the query's 4 bit-planes; = the popc form)
//   AB[slot][pair] = <a(slot), b(pair)>                     (SK: head-sketch rows)
// written to the warp's shared memory; then lanes take 4 slots each and run
// the canonical fp64 LB1 (mrq_lb1_ps) per pair, and the F1 entries are
// sketch-tested from AB (mrq_sketch_decide) in compacted batches of 32.
#define MRQ_TC_ROW 132                  // shared row stride (ints) of S / AB: conflict-free fragment stores
#ifndef MRQ_TC_MINB
#define MRQ_TC_MINB 5
#endif
__device__ __forceinline__ uint32_t nib2bytes(uint32_t x)   // 4 low bits -> 4 bytes of 0/1
{
    return ((x & 0xFu) * 0x00204081u) & 0x01010101u;
}
__device__ __forceinline__ void mma_s8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                       uint32_t b1)
{
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};\n"
                 : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int W, bool SK>
__global__ void __launch_bounds__(128, MRQ_TC_MINB) k_scan_tc(LaunchScan a)
{
    constexpr int KQ = 2 * W;   // sketch k-steps of 32 bytes: dq <= 32 W bytes (dq = d rounded up to 16)
    __shared__ __align__(16) int s_S[4][8 * MRQ_TC_ROW];
    __shared__ __align__(16) int s_AB[SK ? 4 : 1][SK ? 8 * MRQ_TC_ROW : 1];
    __shared__ __align__(16) uint32_t s_code[4][W * 128];     // the tile's code words (word-major)
    __shared__ __align__(16) double s_pc[4][8][12];            // per pair: qc[0..4], eps_r, tau0, t, F, B, qr2, -
    __shared__ uint32_t s_pq[4][8][2];                         // per pair: (pair, q)
    __shared__ uint16_t s_ring[SK ? 4 : 1][SK ? 256 : 1];      // F1 entries: slot in the tile | pair index << 8
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const unsigned FULL = 0xffffffffu;
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t np = (uint32_t)a.np;
    const double inv_np = 1.0 / (double)a.np;
    int *sS = s_S[warp];
    int *sAB = s_AB[SK ? warp : 0];
    uint32_t *sC = s_code[warp];
    uint16_t *ring = s_ring[SK ? warp : 0];
    const uint32_t nunits = a.upre[a.k];
    const int dq = a.dq;
    uint32_t u_next = 0;
    if (lane == 0) u_next = atomicAdd(a.unit_ctr, 1u);
    u_next = __shfl_sync(FULL, u_next, 0);
    for (;;) {
        const uint32_t u = u_next;
        if (u >= nunits) break;
        if (lane == 0) u_next = atomicAdd(a.unit_ctr, 1u);   // the next unit, fetched during this one
        const int c = (int)__ldg(a.unit_list + u);
        const uint32_t pb = __ldg(a.loff + c), pe = __ldg(a.loff + c + 1);
        const uint32_t nch = (pe - pb + 7) / 8;
        const uint32_t local = u - __ldg(a.upre + c);
        const uint32_t tile = local / nch, ch = local - tile * nch;
        const uint32_t lst = __ldg(a.list_off + c), lend = lst + __ldg(a.list_size + c);
        const uint32_t tb = lst + tile * 128;
        const uint32_t j0 = pb + ch * 8;
        const int npc = (int)min(8u, pe - j0);   // pairs in this chunk
        const uint32_t b = tb + lane * 4;
        // stage: the tile's code words (coalesced) and the chunk's per-pair constants
        int pop[4];
        {
            uint4 cw[W];
#pragma unroll
            for (int w = 0; w < W; w++) {
                cw[w] = __ldg((const uint4 *)(a.codes + (int64_t)w * a.npad + b));
                *(uint4 *)(sC + w * 128 + lane * 4) = cw[w];
            }
#pragma unroll
            for (int r = 0; r < 4; r++) {
                int pc = 0;
#pragma unroll
                for (int w = 0; w < W; w++) pc += __popc(r == 0 ? cw[w].x : r == 1 ? cw[w].y : r == 2 ? cw[w].z : cw[w].w);
                pop[r] = pc;
            }
        }
        if (lane < npc) {
            const uint32_t pair = __ldg(a.pairs + j0 + lane);
            uint32_t q = (uint32_t)((double)pair * inv_np);   // pair / np (fp64 estimate, one correction)
            const int32_t rr = (int32_t)(pair - q * np);
            q = rr < 0 ? q - 1 : (rr >= (int32_t)np ? q + 1 : q);
            s_pq[warp][lane][0] = pair;
            s_pq[warp][lane][1] = q;
            double *pc = s_pc[warp][lane];
            const double2 *gq = (const double2 *)(a.qconst + (int64_t)pair * 8);
            const double2 w0 = __ldg(gq), w1 = __ldg(gq + 1);
            pc[0] = w0.x; pc[1] = w0.y; pc[2] = w1.x; pc[3] = w1.y; pc[4] = __ldg(a.qconst + (int64_t)pair * 8 + 4);
            pc[5] = __ldg(a.eps_r + q);
            pc[6] = __ldg(a.tau0 + q);
            if (SK) {
                const double *gs = a.qsk_c + (int64_t)pair * 4;
                pc[7] = __ldg(gs); pc[8] = __ldg(gs + 1); pc[9] = __ldg(gs + 2);
                pc[10] = __ldg(a.qr2 + q);
            }
        }
        __syncwarp();
        // ---- phase A: S (and AB) of the tile's 128 slots x the chunk's pairs on the tensor cores
        {
            const bool bval = g < npc;
            const uint32_t pn = bval ? s_pq[warp][g][0] : 0u;   // B column g
            uint32_t b1f[W][2];
#pragma unroll
            for (int kk = 0; kk < W; kk++) {
                uint32_t x0 = 0, x1 = 0;
                if (bval) {
#pragma unroll
                    for (int jb = 0; jb < MRQ_BQ; jb++) {
                        const uint32_t w = __ldg(a.planes + (int64_t)pn * (MRQ_BQ * W) + jb * W + kk);
                        x0 |= nib2bytes(w >> (4 * t)) << jb;
                        x1 |= nib2bytes(w >> (16 + 4 * t)) << jb;
                    }
                }
                b1f[kk][0] = x0;
                b1f[kk][1] = x1;
            }
            uint32_t b2f[SK ? KQ : 1][2];
            if (SK) {
#pragma unroll
                for (int kk = 0; kk < KQ; kk++) {
                    const int k0 = kk * 32 + 4 * t;
                    const uint8_t *row = a.qsk_b + (int64_t)pn * dq;
                    b2f[kk][0] = (bval && k0 < dq) ? __ldg((const uint32_t *)(row + k0)) : 0u;
                    b2f[kk][1] = (bval && k0 + 16 < dq) ? __ldg((const uint32_t *)(row + k0 + 16)) : 0u;
                }
            }
#pragma unroll 4
            for (int mt = 0; mt < 8; mt++) {
                const int col = mt * 16 + g;
                uint32_t ha[SK ? KQ : 1][4];
                if (SK) {   // the sketch rows' fragments first: their loads overlap the code MMAs
                    const uint8_t *h0 = a.hq + (int64_t)(tb + col) * dq, *h1 = h0 + 8 * dq;
#pragma unroll
                    for (int kk = 0; kk < KQ; kk++) {
                        const int k0 = kk * 32 + 4 * t;
                        const bool lo_ok = k0 < dq, hi_ok = k0 + 16 < dq;
                        ha[kk][0] = lo_ok ? __ldg((const uint32_t *)(h0 + k0)) : 0u;
                        ha[kk][1] = lo_ok ? __ldg((const uint32_t *)(h1 + k0)) : 0u;
                        ha[kk][2] = hi_ok ? __ldg((const uint32_t *)(h0 + k0 + 16)) : 0u;
                        ha[kk][3] = hi_ok ? __ldg((const uint32_t *)(h1 + k0 + 16)) : 0u;
                    }
                }
                int acc[4] = {0, 0, 0, 0};
#pragma unroll
                for (int kk = 0; kk < W; kk++) {
                    const uint32_t c0 = sC[kk * 128 + col], c1 = sC[kk * 128 + col + 8];
                    mma_s8(acc, nib2bytes(c0 >> (4 * t)), nib2bytes(c1 >> (4 * t)), nib2bytes(c0 >> (16 + 4 * t)),
                           nib2bytes(c1 >> (16 + 4 * t)), b1f[kk][0], b1f[kk][1]);
                }
                sS[(2 * t) * MRQ_TC_ROW + col] = acc[0];
                sS[(2 * t + 1) * MRQ_TC_ROW + col] = acc[1];
                sS[(2 * t) * MRQ_TC_ROW + col + 8] = acc[2];
                sS[(2 * t + 1) * MRQ_TC_ROW + col + 8] = acc[3];
                if (SK) {
                    int ac2[4] = {0, 0, 0, 0};
#pragma unroll
                    for (int kk = 0; kk < KQ; kk++)
                        if (kk * 32 < dq) mma_s8(ac2, ha[kk][0], ha[kk][1], ha[kk][2], ha[kk][3], b2f[kk][0], b2f[kk][1]);
                    sAB[(2 * t) * MRQ_TC_ROW + col] = ac2[0];
                    sAB[(2 * t + 1) * MRQ_TC_ROW + col] = ac2[1];
                    sAB[(2 * t) * MRQ_TC_ROW + col + 8] = ac2[2];
                    sAB[(2 * t + 1) * MRQ_TC_ROW + col + 8] = ac2[3];
                }
            }
        }
        __syncwarp();
        // ---- phase B: lane-per-slot canonical LB1 for every pair of the chunk
        const float4 x1 = __ldg((const float4 *)(a.f1 + b)), x2 = __ldg((const float4 *)(a.f2 + b)),
                     x3 = __ldg((const float4 *)(a.f3 + b));
        const float v1[4] = {x1.x, x1.y, x1.z, x1.w}, v2[4] = {x2.x, x2.y, x2.z, x2.w}, v3[4] = {x3.x, x3.y, x3.z, x3.w};
        uint32_t rh = 0, rt = 0;   // SK: ring head / tail (warp-uniform; circular, < 256 pending)
        // SK: sketch test of ring entries [rh, rh + n) (n <= 32, lane per entry) from AB; survivors appended
        auto drain = [&](uint32_t n) {
            const bool in = (uint32_t)lane < n;
            const uint32_t e = in ? ring[(rh + lane) & 255u] : 0u;
            const uint32_t sl = e & 0xFFu, j = e >> 8;
            bool keep = false;
            uint32_t q = 0;
            if (in) {
                q = s_pq[warp][j][1];
                const double *pc = s_pc[warp][j];
                const float4 se = a.hs[tb + sl];
                keep = mrq_sketch_decide(sAB[j * MRQ_TC_ROW + sl], (int)se.w, se, pc + 7, pc[10], pc[5], pc[6]);
            }
            if (__ballot_sync(FULL, keep)) {
                const unsigned grp = __match_any_sync(FULL, keep ? q : 0xFFFFFFFFu);
                if (keep) {
                    const int leader = __ffs(grp) - 1;
                    uint32_t o = 0;
                    if (lane == leader) o = atomicAdd(&a.surv_cnt[q], (uint32_t)__popc(grp));
                    o = __shfl_sync(grp, o, leader) + __popc(grp & lt);
                    MRQ_ASSERT(o < (uint32_t)(a.f1_off[q + 1] - a.f1_off[q]));
                    a.f1_pos[a.f1_off[q] + o] = tb + sl;
                }
            }
            rh += n;
        };
        for (int j = 0; j < npc; j++) {
            const uint32_t q = s_pq[warp][j][1];
            const double *pc = s_pc[warp][j];
            const double qc[5] = {pc[0], pc[1], pc[2], pc[3], pc[4]};
            const double eps_r = pc[5], tau0 = pc[6];
            const int4 Sv = *(const int4 *)(sS + j * MRQ_TC_ROW + lane * 4);
            const int Sr[4] = {Sv.x, Sv.y, Sv.z, Sv.w};
            bool fl[4];
#pragma unroll
            for (int r = 0; r < 4; r++) {
                double dis;
                fl[r] = (b + r < lend) && (mrq_lb1_ps(pop[r], Sr[r], qc, a.isd, eps_r, v1[r], v2[r], v3[r], &dis) < tau0);
            }
            const unsigned b0 = __ballot_sync(FULL, fl[0]), b1 = __ballot_sync(FULL, fl[1]);
            const unsigned b2 = __ballot_sync(FULL, fl[2]), b3 = __ballot_sync(FULL, fl[3]);
            const int n0 = __popc(b0), n1 = __popc(b1), n2 = __popc(b2), n3 = __popc(b3);
            const int tot = n0 + n1 + n2 + n3;
            if (!tot) continue;
            uint32_t wb;
            if (SK) {
                if (lane == 0) atomicAdd(&a.f1_cnt[q], (uint32_t)tot);   // F1 is counted; members queue for the sketch
                wb = rt;
            } else {
                wb = 0;
                if (lane == 0) wb = atomicAdd(&a.f1_cnt[q], (uint32_t)tot);
                wb = __shfl_sync(FULL, wb, 0);
            }
            const uint32_t o0 = wb + __popc(b0 & lt), o1 = wb + n0 + __popc(b1 & lt);
            const uint32_t o2 = wb + n0 + n1 + __popc(b2 & lt), o3 = wb + n0 + n1 + n2 + __popc(b3 & lt);
            if (SK) {
                const uint16_t jj = (uint16_t)(j << 8), sl = (uint16_t)(lane * 4);
                if (fl[0]) ring[o0 & 255u] = jj | sl;
                if (fl[1]) ring[o1 & 255u] = jj | (sl + 1);
                if (fl[2]) ring[o2 & 255u] = jj | (sl + 2);
                if (fl[3]) ring[o3 & 255u] = jj | (sl + 3);
                rt += tot;
                __syncwarp();
                while (rt - rh >= 32) drain(32);
            } else {
                uint32_t *out = a.f1_pos + a.f1_off[q];
                MRQ_ASSERT(wb + tot <= (uint32_t)(a.f1_off[q + 1] - a.f1_off[q]));
                if (fl[0]) out[o0] = b;
                if (fl[1]) out[o1] = b + 1;
                if (fl[2]) out[o2] = b + 2;
                if (fl[3]) out[o3] = b + 3;
            }
        }
        if (SK && rt != rh) drain(rt - rh);
        u_next = __shfl_sync(FULL, u_next, 0);
        __syncwarp();   // the next unit's staging overwrites this unit's shared tiles
    }
}

template <int W, bool SK>
static int launch_scan_tc_ws(const LaunchScan &a, cudaStream_t st)
{
    static int grid = 0;
    if (!grid) {
        int dev = 0, nsm = 0, per = 0;
        MRQ_CUDA_TRY(cudaGetDevice(&dev));
        MRQ_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        MRQ_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_scan_tc<W, SK>, 128, 0));
        grid = nsm * std::max(per, 1);
    }
    k_scan_tc<W, SK><<<grid, 128, 0, st>>>(a);
    MRQ_CUDA_TRY(cudaGetLastError());
    return MRQ_OK;
}

template <int W, bool SK>
static int launch_scan_lm_ws(const LaunchScan &a, cudaStream_t st)
{
    static int grid = 0;   // resident blocks of this instance on the device (one per process: one device type)
    if (!grid) {
        int dev = 0, nsm = 0, per = 0;
        MRQ_CUDA_TRY(cudaGetDevice(&dev));
        MRQ_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        MRQ_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_scan_lm<W, SK>, 128, 0));
        grid = nsm * std::max(per, 1);
    }
    k_scan_lm<W, SK><<<grid, 128, 0, st>>>(a);
    MRQ_CUDA_TRY(cudaGetLastError());
    return MRQ_OK;
}

// mode EXACT (IVF*-restricted exact search, every probed candidate is
// re-ranked): F1 = all of them, written in probe order then slot order
// without evaluating any code (so any code length d works in this mode).
// Block per query.
__global__ void k_f1_all(const uint32_t *__restrict__ probe, int np, const uint32_t *__restrict__ list_off,
                         const uint32_t *__restrict__ list_size, const uint64_t *__restrict__ f1_off,
                         uint32_t *__restrict__ f1_cnt, uint32_t *__restrict__ f1_pos)
{
    const int64_t q = blockIdx.x;
    uint32_t *out = f1_pos + f1_off[q];
    uint32_t at = 0;
    for (int p = 0; p < np; p++) {
        const uint32_t c = probe[q * np + p];
        if (c == 0xFFFFFFFFu) continue;
        const uint32_t st = list_off[c], sz = list_size[c];
        MRQ_ASSERT(at + sz <= (uint32_t)(f1_off[q + 1] - f1_off[q]));
        for (uint32_t e = threadIdx.x; e < sz; e += blockDim.x) out[at + e] = st + e;
        at += sz;
    }
    if (threadIdx.x == 0) f1_cnt[q] = at;
}

void launch_f1_all(const uint32_t *probe, int64_t nq, int np, const uint32_t *list_off, const uint32_t *list_size,
                   const uint64_t *f1_off, uint32_t *f1_cnt, uint32_t *f1_pos, cudaStream_t st)
{
    k_f1_all<<<(unsigned)nq, 256, 0, st>>>(probe, np, list_off, list_size, f1_off, f1_cnt, f1_pos);
}

__global__ void k_fill_f64(double *p, int64_t n, double v)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

void launch_fill_f64(double *p, int64_t n, double v, cudaStream_t st)
{
    k_fill_f64<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(p, n, v);
}

// ================================================================ launchers
template <int W, bool SK, int H>
static int launch_scan_ws(const LaunchScan &a, cudaStream_t st)
{
    // the opt-in covers static + dynamic shared memory (SK adds a static per-warp queue)
    if (a.smem + (SK ? (MRQ_SCAN_THREADS / 32) * MRQ_SKQ * 4 + 64 : 64) > 48 * 1024)
        MRQ_CUDA_TRY(cudaFuncSetAttribute(k_scan<W, SK, H>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)a.smem));
    ScanSketch sk;
    sk.hq = a.hq; sk.hs = a.hs; sk.qsk_b = a.qsk_b; sk.qsk_c = a.qsk_c; sk.qr2 = a.qr2;
    sk.dq = a.dq; sk.surv_cnt = a.surv_cnt;
    sk.pshift = mrq_scan_pshift(a.np);
    if (SK && !mrq_scan_sketch_fits(a.np, a.npad)) {
        mrq_set_error("scan sketch queue: np=%d npad=%lld do not pack into one word", a.np, (long long)a.npad);
        return MRQ_EINVAL;
    }
    k_scan<W, SK, H><<<a.nq, MRQ_SCAN_THREADS, a.smem, st>>>(a.probe, a.np, a.npad, a.list_off, a.list_size, a.codes,
                                                           a.f1, a.f2, a.f3, a.planes, a.qconst, a.eps_r, a.tau0,
                                                           a.isd, a.f1_off, a.f1_cnt, a.f1_pos, a.qorder, sk);
    MRQ_CUDA_TRY(cudaGetLastError());
    return MRQ_OK;
}

template <int W>
static int launch_scan_w(const LaunchScan &a, cudaStream_t st)
{
    if (a.lm) {
        if (W > 4) {
            mrq_set_error("list-major scan: W=%d > 4", W);
            return MRQ_EINVAL;
        }
        constexpr int WL = W > 4 ? 1 : W;
        if (a.lm == 2) return a.surv_cnt ? launch_scan_tc_ws<WL, true>(a, st) : launch_scan_tc_ws<WL, false>(a, st);
        return a.surv_cnt ? launch_scan_lm_ws<WL, true>(a, st) : launch_scan_lm_ws<WL, false>(a, st);
    }
#ifndef MRQ_SCAN_H2_MB
#define MRQ_SCAN_H2_MB 64
#endif
    // H = 2 when the stream cannot live in L2 AND the queries run in the given order; in the
    // list-locality order (a.qorder) most of it is served by L2 all the same (Deep-shaped: L2 hit
    // rate 60%, DRAM 1.5 GB of 3.9 GB) and H = 1 is faster (scan 0.686 -> 0.666 ms)
    const bool dram = (uint64_t)a.npad * (4 * W + 12) > ((uint64_t)MRQ_SCAN_H2_MB << 20) && !a.qorder;
    if (a.surv_cnt) return dram ? launch_scan_ws<W, true, 2>(a, st) : launch_scan_ws<W, true, 1>(a, st);
    return dram ? launch_scan_ws<W, false, 2>(a, st) : launch_scan_ws<W, false, 1>(a, st);
}

int launch_scan(int W, const LaunchScan &a, cudaStream_t st)
{
    switch (W) {
    case 1: return launch_scan_w<1>(a, st);
    case 2: return launch_scan_w<2>(a, st);
    case 3: return launch_scan_w<3>(a, st);
    case 4: return launch_scan_w<4>(a, st);
    case 8: return launch_scan_w<8>(a, st);
    case 16: return launch_scan_w<16>(a, st);
    default: mrq_set_error("unsupported W=%d", W); return MRQ_EINVAL;
    }
}

bool supported_W(int W) { return W == 1 || W == 2 || W == 3 || W == 4 || W == 8 || W == 16; }

// Test hook (mrq_debug_set "dump_dis"): dis' and LB1 of every scanned
// candidate, in probe order then slot order -- the oracle's scan order --
// written at f1_off[q] + i.  Uses the same epilogue as k_scan.
template <int W>
__global__ void k_scan_dbg(const uint32_t *__restrict__ probe, int np, int64_t npad,
                           const uint32_t *__restrict__ list_off, const uint32_t *__restrict__ list_size,
                           const uint32_t *__restrict__ codes, const float *__restrict__ f1,
                           const float *__restrict__ f2, const float *__restrict__ f3,
                           const uint32_t *__restrict__ planes, const double *__restrict__ qconst,
                           const double *__restrict__ eps_r_arr, double isd, const uint64_t *__restrict__ f1_off,
                           double *__restrict__ dis_out, double *__restrict__ lb1_out)
{
    const int64_t q = blockIdx.x;
    uint64_t at = f1_off[q];
    const double eps_r = eps_r_arr[q];
    for (int p = 0; p < np; p++) {
        const uint32_t c = probe[q * np + p];
        if (c == 0xFFFFFFFFu) continue;
        const uint32_t off = list_off[c], sz = list_size[c];
        const uint32_t *pl = planes + (q * np + p) * (MRQ_BQ * W);
        const double *qc = qconst + (q * np + p) * 8;
        for (uint32_t e = threadIdx.x; e < sz; e += blockDim.x) {
            const uint32_t slot = off + e;
            uint32_t code[W];
#pragma unroll
            for (int w = 0; w < W; w++) code[w] = codes[(int64_t)w * npad + slot];
            double dis;
            const double lb1 = mrq_lb1<W>(code, pl, qc, isd, eps_r, f1[slot], f2[slot], f3[slot], &dis);
            dis_out[at + e] = dis;
            lb1_out[at + e] = lb1;
        }
        at += sz;
    }
}

void launch_scan_dbg(int W, const LaunchScan &a, double *dis, double *lb1, cudaStream_t st)
{
#define MRQ_DBG(WW)                                                                                           \
    k_scan_dbg<WW><<<a.nq, 256, 0, st>>>(a.probe, a.np, a.npad, a.list_off, a.list_size, a.codes, a.f1, a.f2, \
                                         a.f3, a.planes, a.qconst, a.eps_r, a.isd, a.f1_off, dis, lb1)
    switch (W) {
    case 1: MRQ_DBG(1); break;
    case 2: MRQ_DBG(2); break;
    case 3: MRQ_DBG(3); break;
    case 4: MRQ_DBG(4); break;
    case 8: MRQ_DBG(8); break;
    case 16: MRQ_DBG(16); break;
    default: break;
    }
#undef MRQ_DBG
}

// mrq_build.cu -- GPU index build: Algorithm 1 L1-L6
// plus the quantizer rotation P_r, written as an
// MRQBLD01 build file that mrq_index_load reads.
//
//   L1-L2  PCA: mean and covariance of a strided sample of <= pca_sample rows
//          (fp64 on the GPU), eigen-decomposition on the host (Householder
//          tridiagonalisation + implicit QL), eigenpairs sorted by eigenvalue
//          descending, each eigenvector sign-normalised so its largest-|entry|
//          component is positive, lambda_i = max(eigenvalue, 0);
//   L3-L5  heads x_d = P[0:d] (x - mu) for all N (k_rowmat, fp64);
//   L6     IVF* k-means on the heads: a strided sample of <= km_sample_per_k k
//          rows, initial centroids = k strided sample rows, <= km_iters Lloyd
//          iterations (the assignment step on the tensor cores: the search
//          path's tcgen05 probe with np = 1 and its exact fp64 rescore,
//          TcAssign; fp64 centroid sums), stop when the relative WCSS gain < 1e-4, an empty cluster is
//          re-seeded at the farthest member of the largest cluster; final
//          assignment of all N to the nearest centroid;
//   P_r    Haar d x d rotation: modified Gram-Schmidt (twice) of a Gaussian
//          drawn from a seeded 64-bit generator, columns sign-fixed.
//
// This is the same algorithm as oracle/build.py, not the same bits: the
// samples are strided instead of numpy-random, the solver and the summation
// orders differ.  Its contract is recall-equivalence with the oracle build
// (tests/test_gpu_build.py), which is the parity SURVEY NEXT-1 asks for.
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <random>
#include <vector>

#include "mrq_internal.cuh"
#include "mrq_kernels.cuh"
#include "mrq_probe_tc.cuh"

namespace {

// ------------------------------------------------------------ PCA kernels
// colsum[j] += x[r][j] over the sample rows r = floor(t n / s), t < s.
__global__ void k_sample_mean(const float *__restrict__ X, int64_t n, int D, int64_t s, double *__restrict__ sum)
{
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= D) return;
    double acc = 0.0;
    for (int64_t t = blockIdx.y; t < s; t += gridDim.y) acc += (double)X[(t * n / s) * D + j];
    atomicAdd(&sum[j], acc);
}

// cov[i][j] = sum_t (x_ti - mu_i)(x_tj - mu_j) over the sample (64 x 64 tiles,
// 4 x 4 per thread; the division by s - 1 happens on the host).
__global__ void __launch_bounds__(256) k_sample_cov(const float *__restrict__ X, int64_t n, int D, int64_t s,
                                                    const double *__restrict__ mu, double *__restrict__ cov)
{
    __shared__ double a[16][65], b[16][65];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int i0 = blockIdx.y * 64, j0 = blockIdx.x * 64;
    double acc[4][4] = {};
    const int64_t rows_per = (s + gridDim.z - 1) / gridDim.z;
    const int64_t rb = blockIdx.z * rows_per, re = min(s, rb + rows_per);
    for (int64_t t0 = rb; t0 < re; t0 += 16) {
        for (int q = tid; q < 16 * 64; q += 256) {
            const int tt = q / 64, c = q % 64;
            const int64_t t = t0 + tt;
            double va = 0.0, vb = 0.0;
            if (t < re) {
                const float *row = X + (t * n / s) * D;
                if (i0 + c < D) va = (double)row[i0 + c] - mu[i0 + c];
                if (j0 + c < D) vb = (double)row[j0 + c] - mu[j0 + c];
            }
            a[tt][c] = va;
            b[tt][c] = vb;
        }
        __syncthreads();
#pragma unroll
        for (int tt = 0; tt < 16; tt++) {
            double x[4], y[4];
#pragma unroll
            for (int r = 0; r < 4; r++) x[r] = a[tt][ty + 16 * r];
#pragma unroll
            for (int c = 0; c < 4; c++) y[c] = b[tt][tx + 16 * c];
#pragma unroll
            for (int r = 0; r < 4; r++)
#pragma unroll
                for (int c = 0; c < 4; c++) acc[r][c] += x[r] * y[c];
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 4; r++)
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const int i = i0 + ty + 16 * r, j = j0 + tx + 16 * c;
            if (i < D && j < D) atomicAdd(&cov[(int64_t)i * D + j], acc[r][c]);
        }
}

// --------------------------------------------------------- k-means kernels
__global__ void k_to_f32(const double *__restrict__ a, int64_t n, float *__restrict__ b)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = (float)a[i];
}

__global__ void k_gather_rows(const float *__restrict__ src, int64_t n, int d, int64_t m, float *__restrict__ dst)
{
    const int64_t t = blockIdx.x;
    const int64_t r = t * n / m;
    for (int j = threadIdx.x; j < d; j += blockDim.x) dst[t * d + j] = src[r * d + j];
}

__global__ void k_rownorm(const float *__restrict__ x, int64_t n, int d, float *__restrict__ out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float acc = 0.f;
    for (int j = 0; j < d; j++) acc = fmaf(x[i * d + j], x[i * d + j], acc);
    out[i] = acc;
}

// a[i] = argmin_c (||c||^2 - 2 <x_i, c>) (ties -> smaller c), dmin[i] = ||x_i||^2 + that value.
// 64 points x 64 centroids per tile, 4 x 4 per thread, the point block loops
// over all centroid tiles keeping a running minimum per (point, thread).
__global__ void __launch_bounds__(256) k_assign(const float *__restrict__ X, int64_t n, int d,
                                                const float *__restrict__ Cf, const float *__restrict__ cn, int k,
                                                const float *__restrict__ xn, uint32_t *__restrict__ a,
                                                float *__restrict__ dmin)
{
    __shared__ float xs[16][65], cs[16][65];
    __shared__ float rv[64][17];
    __shared__ uint32_t ri[64][17];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int64_t p0 = (int64_t)blockIdx.x * 64;
    float best[4];
    uint32_t bid[4];
#pragma unroll
    for (int r = 0; r < 4; r++) {
        best[r] = __int_as_float(0x7f800000);
        bid[r] = 0xFFFFFFFFu;
    }
    for (int c0 = 0; c0 < k; c0 += 64) {
        float acc[4][4] = {};
        for (int j0 = 0; j0 < d; j0 += 16) {
            for (int q = tid; q < 16 * 64; q += 256) {
                const int jj = q % 16, rr = q / 16;
                const int64_t p = p0 + rr;
                const int c = c0 + rr, j = j0 + jj;
                xs[jj][rr] = (p < n && j < d) ? X[p * d + j] : 0.f;
                cs[jj][rr] = (c < k && j < d) ? Cf[(int64_t)c * d + j] : 0.f;
            }
            __syncthreads();
#pragma unroll
            for (int jj = 0; jj < 16; jj++) {
                float x[4], y[4];
#pragma unroll
                for (int r = 0; r < 4; r++) x[r] = xs[jj][ty + 16 * r];
#pragma unroll
                for (int c = 0; c < 4; c++) y[c] = cs[jj][tx + 16 * c];
#pragma unroll
                for (int r = 0; r < 4; r++)
#pragma unroll
                    for (int c = 0; c < 4; c++) acc[r][c] = fmaf(x[r], y[c], acc[r][c]);
            }
            __syncthreads();
        }
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const int cc = c0 + tx + 16 * c;
            if (cc >= k) continue;
            const float cnv = cn[cc];
#pragma unroll
            for (int r = 0; r < 4; r++) {
                const float v = fmaf(-2.0f, acc[r][c], cnv);
                if (v < best[r] || (v == best[r] && (uint32_t)cc < bid[r])) {
                    best[r] = v;
                    bid[r] = (uint32_t)cc;
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < 4; r++) {
        rv[ty + 16 * r][tx] = best[r];
        ri[ty + 16 * r][tx] = bid[r];
    }
    __syncthreads();
    if (tid < 64) {
        float b = rv[tid][0];
        uint32_t bi = ri[tid][0];
        for (int t = 1; t < 16; t++)
            if (rv[tid][t] < b || (rv[tid][t] == b && ri[tid][t] < bi)) {
                b = rv[tid][t];
                bi = ri[tid][t];
            }
        const int64_t p = p0 + tid;
        if (p < n) {
            a[p] = bi;
            dmin[p] = fmaxf(xn[p] + b, 0.f);
        }
    }
}

// ------------------------------------------------ tensor-core assignment
// The k-means assignment step (nearest centroid, Alg.1 L6) on the tensor
// cores: the search path's probe (k_probe_tc<true, 16> screen with np = 1 +
// k_probe_finish_w's exact fp64 rescore of the margin set, DESIGN.md §4 "probe
// exactness") run on a build-time pseudo index that holds the current
// centroids.  a[i] = argmin_c ||x_i - c||^2 (ties -> smaller c), evaluated
// exactly in fp64 for the fp32 points; dmin[i] = that squared distance.
__global__ void k_f32_rows_to_probe(const float *__restrict__ X, int64_t n, int d, double *__restrict__ x64,
                                    float *__restrict__ qa3, double *__restrict__ qnorm)
{
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    double n2 = 0.0;
    for (int j = lane; j < d; j += 32) {
        const float x = X[i * d + j];
        x64[i * d + j] = (double)x;
        float hi, lo;
        tf32_split(x, hi, lo);
        qa3[i * 3 * d + j] = hi;
        qa3[i * 3 * d + d + j] = hi;
        qa3[i * 3 * d + 2 * d + j] = lo;
        n2 += (double)x * (double)x;
    }
    for (int o = 16; o > 0; o >>= 1) n2 += __shfl_xor_sync(0xffffffffu, n2, o);
    if (lane == 0) qnorm[i] = sqrt(n2) * (1.0 + 0x1p-40);   // >= ||x|| (the bound's input)
}

__global__ void k_centroid_norms(const double *__restrict__ C, int k, int d, float *__restrict__ cn32,
                                 double *__restrict__ cnorm)
{
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= k) return;
    double s = 0.0;
    for (int j = 0; j < d; j++) {
        const double v = (double)(float)C[(int64_t)c * d + j];   // of the fp32 centroid the screen uses
        s += v * v;
    }
    cn32[c] = (float)s;
    double t = 0.0;
    for (int j = 0; j < d; j++) t += C[(int64_t)c * d + j] * C[(int64_t)c * d + j];
    cnorm[c] = sqrt(t);
}

#define TRY_S(x)                         \
    do {                                 \
        int _r = (x);                    \
        if (_r != MRQ_OK) return _r;     \
    } while (0)

struct TcAssign {
    mrq_index ix;                  // pseudo index: the current centroids only
    float *cn32 = nullptr;
    double *cnorm = nullptr;
    int capp = 32;                 // np = 1: about 1 + ln(k / P) appends per part
    bool ok = false;
    ~TcAssign()
    {
        mrq_probe_tc_free(&ix);
        if (cn32) cudaFree(cn32);
        if (cnorm) cudaFree(cnorm);
        for (auto &kv : ix.scratch)
            if (kv.second.p) cudaFree(kv.second.p);
    }
    int init(int k, int d, int sm_count)
    {
        ix.k = k;
        ix.d = d;
        ix.D = d;
        ix.sm_count = sm_count;
        ix.stream = 0;
        ix.device = -1;
        const int kp = (k + 255) / 256 * 256;
        if (cudaMalloc(&cn32, (size_t)kp * 4) != cudaSuccess || cudaMalloc(&cnorm, (size_t)k * 8) != cudaSuccess) {
            mrq_set_error("cudaMalloc (tensor-core assignment)");
            return MRQ_ENOMEM;
        }
        std::vector<float> inf(kp, INFINITY);
        MRQ_CUDA_TRY(cudaMemcpy(cn32, inf.data(), (size_t)kp * 4, cudaMemcpyHostToDevice));
        ix.cn32 = cn32;
        return MRQ_OK;
    }
    // new centroids: C fp64 [k][d], Cf = fp32(C)
    int set_centroids(double *C, float *Cf)
    {
        ix.C = C;
        ix.C32 = Cf;
        k_centroid_norms<<<(ix.k + 255) / 256, 256>>>(C, ix.k, ix.d, cn32, cnorm);
        std::vector<double> nr(ix.k);
        MRQ_CUDA_TRY(cudaMemcpy(nr.data(), cnorm, (size_t)ix.k * 8, cudaMemcpyDeviceToHost));
        double mx = 0.0;
        for (double v : nr) mx = std::max(mx, v);
        ix.cmax = mx * (1.0 + 1e-9) + 1e-300;
        mrq_probe_tc_free(&ix);
        const int rc = mrq_probe_tc_init(&ix);
        if (rc != MRQ_OK) return rc;
        ok = mrq_probe_tc_fusable(&ix, 1);
        return MRQ_OK;
    }
    // a[i], dmin[i] (fp64) for n fp32 rows X [n][d], in chunks
    int assign(const float *X, int64_t n, uint32_t *a, double *dmin)
    {
        const int d = ix.d, k = ix.k;
        const int64_t CH = 1 << 19;
        for (int64_t r0 = 0; r0 < n; r0 += CH) {
            const int64_t m = std::min<int64_t>(CH, n - r0);
            double *x64, *qn;
            float *qa3;
            TRY_S(mrq_scratch(&ix, "a_x64", (size_t)m * d * 8, (void **)&x64));
            TRY_S(mrq_scratch(&ix, "a_qa3", (size_t)m * 3 * d * 4, (void **)&qa3));
            TRY_S(mrq_scratch(&ix, "a_qn", (size_t)m * 8, (void **)&qn));
            k_f32_rows_to_probe<<<(unsigned)((m + 7) / 8), 256>>>(X + r0 * d, m, d, x64, qa3, qn);
            const int P = mrq_probe_tc_parts(&ix, m);
            uint2 *cbuf;
            uint32_t *ccnt, *cand, *ncand;
            float *kv;
            TRY_S(mrq_scratch(&ix, "a_cbuf", (size_t)m * P * capp * 8, (void **)&cbuf));
            TRY_S(mrq_scratch(&ix, "a_ccnt", (size_t)m * P * 4, (void **)&ccnt));
            TRY_S(mrq_scratch(&ix, "a_kv", (size_t)m * P * 4, (void **)&kv));
            const int64_t cs = std::min<int64_t>(k, (int64_t)P * capp);
            TRY_S(mrq_scratch(&ix, "a_cand", (size_t)m * cs * 4, (void **)&cand));
            TRY_S(mrq_scratch(&ix, "a_ncand", (size_t)m * 4, (void **)&ncand));
            const double kappa = mrq_probe_tc_kappa(&ix);
            uint32_t *gkey;
            TRY_S(mrq_scratch(&ix, "a_gkey", (size_t)m * 4, (void **)&gkey));
            TRY_S(mrq_probe_tc_run_fused(&ix, qa3, m, 1, qn, kappa, cbuf, capp, ccnt, kv, gkey, 0));
            TRY_S(launch_probe_finish_w(m, k, d, 1, x64, d, ix.C, qn, ix.cmax, kappa, cbuf, P, capp,
                                        mrq_probe_tc_grid(&ix, m), ccnt, kv, cand, a + r0, dmin + r0, ncand, 0));
        }
        MRQ_CUDA_TRY(cudaGetLastError());
        return MRQ_OK;
    }
};

__global__ void k_accumulate(const float *__restrict__ X, int64_t n, int d, const uint32_t *__restrict__ a,
                             double *__restrict__ sums, uint32_t *__restrict__ cnt)
{
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    const uint32_t c = a[i];
    for (int j = lane; j < d; j += 32) atomicAdd(&sums[(int64_t)c * d + j], (double)X[i * d + j]);
    if (lane == 0) atomicAdd(&cnt[c], 1u);
}

__global__ void k_centroids(const double *__restrict__ sums, const uint32_t *__restrict__ cnt, int k, int d,
                            double *__restrict__ C, float *__restrict__ Cf, float *__restrict__ cn)
{
    const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (c >= k) return;
    float nrm = 0.f;
    if (cnt[c] > 0)
        for (int j = lane; j < d; j += 32) {
            const double v = sums[(int64_t)c * d + j] / (double)cnt[c];
            C[(int64_t)c * d + j] = v;
            Cf[(int64_t)c * d + j] = (float)v;
        }
    __syncwarp();
    for (int j = lane; j < d; j += 32) nrm = fmaf(Cf[(int64_t)c * d + j], Cf[(int64_t)c * d + j], nrm);
    for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
    if (lane == 0) cn[c] = nrm;
}

__global__ void k_sum_f32(const float *__restrict__ x, int64_t n, double *__restrict__ out)
{
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        acc += x[i];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

// --------------------------------------------------- host linear algebra
// Symmetric eigen-decomposition (Householder tridiagonalisation + implicit
// QL with Wilkinson shifts): a transcription of the classic public-domain
// EISPACK tred2/tql2 pair as given in JAMA's EigenvalueDecomposition (the
// variable names follow it).  Off the hot path (NEXT-1 host PCA, D x D).  a: n x n row-major
// (destroyed); on return w[i] are the eigenvalues and column i of V (row-major
// n x n) the eigenvector of w[i].
void sym_eig(int n, std::vector<double> &a, std::vector<double> &w, std::vector<double> &V)
{
    std::vector<double> d(n), e(n);
    V = a;
    auto Vr = [&](int i, int j) -> double & { return V[(size_t)i * n + j]; };
    for (int j = 0; j < n; j++) d[j] = Vr(n - 1, j);
    for (int i = n - 1; i > 0; i--) {   // Householder reduction to tridiagonal form
        double scale = 0.0, h = 0.0;
        for (int k = 0; k < i; k++) scale += std::fabs(d[k]);
        if (scale == 0.0) {
            e[i] = d[i - 1];
            for (int j = 0; j < i; j++) {
                d[j] = Vr(i - 1, j);
                Vr(i, j) = 0.0;
                Vr(j, i) = 0.0;
            }
        } else {
            for (int k = 0; k < i; k++) {
                d[k] /= scale;
                h += d[k] * d[k];
            }
            double f = d[i - 1];
            double g = std::sqrt(h);
            if (f > 0) g = -g;
            e[i] = scale * g;
            h -= f * g;
            d[i - 1] = f - g;
            for (int j = 0; j < i; j++) e[j] = 0.0;
            for (int j = 0; j < i; j++) {
                f = d[j];
                Vr(j, i) = f;
                g = e[j] + Vr(j, j) * f;
                for (int k = j + 1; k <= i - 1; k++) {
                    g += Vr(k, j) * d[k];
                    e[k] += Vr(k, j) * f;
                }
                e[j] = g;
            }
            f = 0.0;
            for (int j = 0; j < i; j++) {
                e[j] /= h;
                f += e[j] * d[j];
            }
            const double hh = f / (h + h);
            for (int j = 0; j < i; j++) e[j] -= hh * d[j];
            for (int j = 0; j < i; j++) {
                f = d[j];
                g = e[j];
                for (int k = j; k <= i - 1; k++) Vr(k, j) -= (f * e[k] + g * d[k]);
                d[j] = Vr(i - 1, j);
                Vr(i, j) = 0.0;
            }
        }
        d[i] = h;
    }
    for (int i = 0; i < n - 1; i++) {   // accumulate transformations
        Vr(n - 1, i) = Vr(i, i);
        Vr(i, i) = 1.0;
        const double h = d[i + 1];
        if (h != 0.0) {
            for (int k = 0; k <= i; k++) d[k] = Vr(k, i + 1) / h;
            for (int j = 0; j <= i; j++) {
                double g = 0.0;
                for (int k = 0; k <= i; k++) g += Vr(k, i + 1) * Vr(k, j);
                for (int k = 0; k <= i; k++) Vr(k, j) -= g * d[k];
            }
        }
        for (int k = 0; k <= i; k++) Vr(k, i + 1) = 0.0;
    }
    for (int j = 0; j < n; j++) {
        d[j] = Vr(n - 1, j);
        Vr(n - 1, j) = 0.0;
    }
    Vr(n - 1, n - 1) = 1.0;
    e[0] = 0.0;
    // implicit QL on the tridiagonal matrix (d diagonal, e sub-diagonal)
    for (int i = 1; i < n; i++) e[i - 1] = e[i];
    e[n - 1] = 0.0;
    double f = 0.0, tst1 = 0.0;
    const double eps = std::ldexp(1.0, -52);
    for (int l = 0; l < n; l++) {
        tst1 = std::max(tst1, std::fabs(d[l]) + std::fabs(e[l]));
        int m = l;
        while (m < n) {
            if (std::fabs(e[m]) <= eps * tst1) break;
            m++;
        }
        if (m > l) {
            for (int iter = 0; iter < 60; iter++) {
                double g = d[l];
                double p = (d[l + 1] - g) / (2.0 * e[l]);
                double r = std::hypot(p, 1.0);
                if (p < 0) r = -r;
                d[l] = e[l] / (p + r);
                d[l + 1] = e[l] * (p + r);
                const double dl1 = d[l + 1];
                double h = g - d[l];
                for (int i = l + 2; i < n; i++) d[i] -= h;
                f += h;
                p = d[m];
                double c = 1.0, c2 = c, c3 = c, el1 = e[l + 1], s = 0.0, s2 = 0.0;
                for (int i = m - 1; i >= l; i--) {
                    c3 = c2;
                    c2 = c;
                    s2 = s;
                    g = c * e[i];
                    h = c * p;
                    r = std::hypot(p, e[i]);
                    e[i + 1] = s * r;
                    s = e[i] / r;
                    c = p / r;
                    p = c * d[i] - s * g;
                    d[i + 1] = h + s * (c * g + s * d[i]);
                    for (int k = 0; k < n; k++) {
                        h = Vr(k, i + 1);
                        Vr(k, i + 1) = s * Vr(k, i) + c * h;
                        Vr(k, i) = c * Vr(k, i) - s * h;
                    }
                }
                p = -s * s2 * c3 * el1 * e[l] / dl1;
                e[l] = s * p;
                d[l] = c * p;
                if (std::fabs(e[l]) <= eps * tst1) break;
            }
        }
        d[l] = d[l] + f;
        e[l] = 0.0;
    }
    w = d;
}

// Haar d x d rotation: modified Gram-Schmidt, twice, of a Gaussian (Box-Muller
// on a seeded 64-bit Mersenne Twister); columns sign-fixed so the
// triangular factor's diagonal is positive.  Returned row-major (y = R t).
std::vector<double> haar(int d, uint64_t seed)
{
    std::mt19937_64 gen(seed);
    auto unif = [&]() { return ((double)(gen() >> 11) + 0.5) * std::ldexp(1.0, -53); };
    std::vector<double> G((size_t)d * d);
    for (size_t i = 0; i < G.size(); i += 2) {
        const double u1 = unif(), u2 = unif();
        const double rr = std::sqrt(-2.0 * std::log(u1)), th = 2.0 * M_PI * u2;
        G[i] = rr * std::cos(th);
        if (i + 1 < G.size()) G[i + 1] = rr * std::sin(th);
    }
    // columns of G (G[i][j], column j)
    std::vector<double> Q = G;
    for (int j = 0; j < d; j++) {
        for (int pass = 0; pass < 2; pass++)
            for (int p = 0; p < j; p++) {
                double dot = 0.0;
                for (int i = 0; i < d; i++) dot += Q[(size_t)i * d + p] * Q[(size_t)i * d + j];
                for (int i = 0; i < d; i++) Q[(size_t)i * d + j] -= dot * Q[(size_t)i * d + p];
            }
        double nrm = 0.0;
        for (int i = 0; i < d; i++) nrm += Q[(size_t)i * d + j] * Q[(size_t)i * d + j];
        nrm = std::sqrt(nrm);
        for (int i = 0; i < d; i++) Q[(size_t)i * d + j] /= nrm;
    }
    // sign fix: R_qr diagonal = <q_j, g_j> > 0
    for (int j = 0; j < d; j++) {
        double dot = 0.0;
        for (int i = 0; i < d; i++) dot += Q[(size_t)i * d + j] * G[(size_t)i * d + j];
        if (dot < 0)
            for (int i = 0; i < d; i++) Q[(size_t)i * d + j] = -Q[(size_t)i * d + j];
    }
    return Q;
}

double now_ms()
{
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct Dev {
    std::vector<void *> ptrs;
    ~Dev()
    {
        for (void *p : ptrs) cudaFree(p);
    }
    template <class T>
    int alloc(T **p, size_t count)
    {
        if (count == 0) count = 1;
        if (cudaMalloc((void **)p, count * sizeof(T)) != cudaSuccess) {
            mrq_set_error("cudaMalloc(%zu) failed in mrq_build_gpu", count * sizeof(T));
            return MRQ_ENOMEM;
        }
        ptrs.push_back(*p);
        return MRQ_OK;
    }
};

#define BTRY(x)                          \
    do {                                 \
        int _r = (x);                    \
        if (_r != MRQ_OK) return _r;     \
    } while (0)

}  // namespace

static int build_gpu_impl(const float *base, int64_t n, int32_t D, int32_t d, const mrq_build_params *bp,
                          const char *base_sha256_hex, int32_t device, const char *out_path, double *times_ms);

extern "C" int mrq_build_gpu(const float *base, int64_t n, int32_t D, int32_t d, const mrq_build_params *bp,
                             const char *base_sha256_hex, int32_t device, const char *out_path, double *times_ms)
{
    return mrq_guard([&] { return build_gpu_impl(base, n, D, d, bp, base_sha256_hex, device, out_path, times_ms); });
}

static int build_gpu_impl(const float *base, int64_t n, int32_t D, int32_t d, const mrq_build_params *bp,
                          const char *base_sha256_hex, int32_t device, const char *out_path, double *times_ms)
{
    if (!base || !bp || !out_path || n < 2 || D < 1 || d < 2 || d > D || bp->k < 1 || bp->k > n ||
        bp->pca_sample < 2 || bp->km_sample_per_k < 1 || bp->km_iters < 1) {
        mrq_set_error("InvalidConfig: mrq_build_gpu(n=%lld, D=%d, d=%d, k=%d)", (long long)n, D, d,
                      bp ? bp->k : -1);
        return MRQ_EINVAL;
    }
    const double t_start = now_ms();
    if (device >= 0) MRQ_CUDA_TRY(cudaSetDevice(device));
    const int k = bp->k;
    Dev dv;
    float *dX;
    BTRY(dv.alloc(&dX, (size_t)n * D));
    MRQ_CUDA_TRY(cudaMemcpy(dX, base, (size_t)n * D * 4, cudaMemcpyHostToDevice));

    // ---- L1-L2: PCA on a strided sample
    const int64_t s = std::min<int64_t>(n, bp->pca_sample);
    double *dsum, *dcov;
    BTRY(dv.alloc(&dsum, D));
    BTRY(dv.alloc(&dcov, (size_t)D * D));
    MRQ_CUDA_TRY(cudaMemset(dsum, 0, D * 8));
    MRQ_CUDA_TRY(cudaMemset(dcov, 0, (size_t)D * D * 8));
    k_sample_mean<<<dim3((D + 127) / 128, 256), 128>>>(dX, n, D, s, dsum);
    std::vector<double> mu(D);
    MRQ_CUDA_TRY(cudaMemcpy(mu.data(), dsum, D * 8, cudaMemcpyDeviceToHost));
    for (auto &v : mu) v /= (double)s;
    MRQ_CUDA_TRY(cudaMemcpy(dsum, mu.data(), D * 8, cudaMemcpyHostToDevice));
    {
        const int tiles = (D + 63) / 64;
        const int zs = (int)std::max<int64_t>(1, std::min<int64_t>(s / 256, 592 / std::max(1, tiles * tiles)));
        k_sample_cov<<<dim3(tiles, tiles, zs), 256>>>(dX, n, D, s, dsum, dcov);
    }
    std::vector<double> cov((size_t)D * D);
    MRQ_CUDA_TRY(cudaMemcpy(cov.data(), dcov, cov.size() * 8, cudaMemcpyDeviceToHost));
    for (auto &v : cov) v /= (double)(s - 1);
    double trace = 0.0;
    for (int i = 0; i < D; i++) trace += cov[(size_t)i * D + i];
    if (!(trace > 0)) {
        mrq_set_error("DegenerateData: zero total variance");
        return MRQ_EDEGENERATE;
    }
    std::vector<double> w, V;
    sym_eig(D, cov, w, V);
    std::vector<int> order(D);
    for (int i = 0; i < D; i++) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return w[a] > w[b]; });
    std::vector<double> P((size_t)D * D), lam(D);
    for (int r = 0; r < D; r++) {
        const int c = order[r];
        int jm = 0;
        for (int j = 1; j < D; j++)
            if (std::fabs(V[(size_t)j * D + c]) > std::fabs(V[(size_t)jm * D + c])) jm = j;
        const double sg = V[(size_t)jm * D + c] < 0 ? -1.0 : 1.0;
        for (int j = 0; j < D; j++) P[(size_t)r * D + j] = sg * V[(size_t)j * D + c];
        lam[r] = std::max(w[c], 0.0);
    }
    MRQ_CUDA_TRY(cudaDeviceSynchronize());
    const double t_pca = now_ms();

    // ---- L3-L5: heads of all N (x_d = P[0:d] (x - mu))
    std::vector<double> PTd((size_t)D * d);
    for (int j = 0; j < D; j++)
        for (int i = 0; i < d; i++) PTd[(size_t)j * d + i] = P[(size_t)i * D + j];
    double *dPTd, *dmu, *dheads;
    float *dH;
    BTRY(dv.alloc(&dPTd, PTd.size()));
    BTRY(dv.alloc(&dmu, D));
    MRQ_CUDA_TRY(cudaMemcpy(dPTd, PTd.data(), PTd.size() * 8, cudaMemcpyHostToDevice));
    MRQ_CUDA_TRY(cudaMemcpy(dmu, mu.data(), D * 8, cudaMemcpyHostToDevice));
    BTRY(dv.alloc(&dH, (size_t)n * d));
    {
        const int64_t CH = 1 << 20;
        BTRY(dv.alloc(&dheads, (size_t)std::min<int64_t>(n, CH) * d));
        for (int64_t r0 = 0; r0 < n; r0 += CH) {
            const int64_t m = std::min<int64_t>(CH, n - r0);
            launch_rowmat_f32(dX + r0 * D, m, D, D, dmu, dPTd, d, dheads, d, 0);
            k_to_f32<<<(unsigned)((m * d + 255) / 256), 256>>>(dheads, m * d, dH + r0 * d);
        }
    }
    // ---- L6: k-means on a strided sample of the heads
    const int64_t m = std::min<int64_t>(n, (int64_t)bp->km_sample_per_k * k);
    float *dS, *dSn, *dCf, *dcn, *ddmin;
    uint32_t *dA, *dcnt;
    double *dC, *dsums, *dw;
    BTRY(dv.alloc(&dS, (size_t)m * d));
    BTRY(dv.alloc(&dSn, m));
    BTRY(dv.alloc(&dCf, (size_t)k * d));
    BTRY(dv.alloc(&dcn, k));
    BTRY(dv.alloc(&ddmin, std::max<int64_t>(m, n)));
    BTRY(dv.alloc(&dA, std::max<int64_t>(m, n)));
    BTRY(dv.alloc(&dcnt, k));
    BTRY(dv.alloc(&dC, (size_t)k * d));
    BTRY(dv.alloc(&dsums, (size_t)k * d));
    BTRY(dv.alloc(&dw, 1));
    k_gather_rows<<<(unsigned)m, 64>>>(dH, n, d, m, dS);
    k_rownorm<<<(unsigned)((m + 255) / 256), 256>>>(dS, m, d, dSn);
    k_gather_rows<<<(unsigned)k, 64>>>(dS, m, d, k, dCf);   // initial centroids: k strided sample rows
    {
        std::vector<float> cf((size_t)k * d);
        MRQ_CUDA_TRY(cudaMemcpy(cf.data(), dCf, cf.size() * 4, cudaMemcpyDeviceToHost));
        std::vector<double> c64(cf.begin(), cf.end());
        MRQ_CUDA_TRY(cudaMemcpy(dC, c64.data(), c64.size() * 8, cudaMemcpyHostToDevice));
    }
    k_rownorm<<<(unsigned)((k + 255) / 256), 256>>>(dCf, k, d, dcn);
    // the assignment step on the tensor cores (TcAssign: the search's probe with
    // np = 1, exact fp64 nearest centroid) when d % 4 == 0; else CUDA cores
    TcAssign tc;
    int sm_count = 148;
    MRQ_CUDA_TRY(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, device >= 0 ? device : 0));
    BTRY(tc.init(k, d, sm_count));
    double *ddmin64;
    BTRY(dv.alloc(&ddmin64, std::max<int64_t>(m, n)));
    auto assign_step = [&](const float *Xr, const float *xn, int64_t nr) -> int {
        BTRY(tc.set_centroids(dC, dCf));
        if (tc.ok) {
            BTRY(tc.assign(Xr, nr, dA, ddmin64));
            k_to_f32<<<(unsigned)((nr + 255) / 256), 256>>>(ddmin64, nr, ddmin);
        } else {
            k_assign<<<(unsigned)((nr + 63) / 64), 256>>>(Xr, nr, d, dCf, dcn, k, xn, dA, ddmin);
        }
        MRQ_CUDA_TRY(cudaGetLastError());
        return MRQ_OK;
    };
    double prev = INFINITY;
    for (int it = 0; it < bp->km_iters; it++) {
        BTRY(assign_step(dS, dSn, m));
        MRQ_CUDA_TRY(cudaMemset(dw, 0, 8));
        k_sum_f32<<<256, 256>>>(ddmin, m, dw);
        MRQ_CUDA_TRY(cudaMemset(dsums, 0, (size_t)k * d * 8));
        MRQ_CUDA_TRY(cudaMemset(dcnt, 0, (size_t)k * 4));
        k_accumulate<<<(unsigned)((m + 7) / 8), 256>>>(dS, m, d, dA, dsums, dcnt);
        k_centroids<<<(unsigned)((k + 7) / 8), 256>>>(dsums, dcnt, k, d, dC, dCf, dcn);
        double wcss = 0.0;
        MRQ_CUDA_TRY(cudaMemcpy(&wcss, dw, 8, cudaMemcpyDeviceToHost));
        std::vector<uint32_t> cnt(k);
        MRQ_CUDA_TRY(cudaMemcpy(cnt.data(), dcnt, (size_t)k * 4, cudaMemcpyDeviceToHost));
        if (std::count(cnt.begin(), cnt.end(), 0u) > 0) {   // empty-cluster repair (rare): on the host
            std::vector<uint32_t> a(m);
            std::vector<float> dm(m), S((size_t)m * d);
            MRQ_CUDA_TRY(cudaMemcpy(a.data(), dA, (size_t)m * 4, cudaMemcpyDeviceToHost));
            MRQ_CUDA_TRY(cudaMemcpy(dm.data(), ddmin, (size_t)m * 4, cudaMemcpyDeviceToHost));
            MRQ_CUDA_TRY(cudaMemcpy(S.data(), dS, S.size() * 4, cudaMemcpyDeviceToHost));
            for (int j = 0; j < k; j++) {
                if (cnt[j]) continue;
                const int big = (int)(std::max_element(cnt.begin(), cnt.end()) - cnt.begin());
                int64_t far = -1;
                for (int64_t i = 0; i < m; i++)
                    if ((int)a[i] == big && (far < 0 || dm[i] > dm[far])) far = i;
                if (far < 0) continue;
                std::vector<double> c64(S.begin() + far * d, S.begin() + (far + 1) * d);
                std::vector<float> c32(S.begin() + far * d, S.begin() + (far + 1) * d);
                MRQ_CUDA_TRY(cudaMemcpy(dC + (size_t)j * d, c64.data(), d * 8, cudaMemcpyHostToDevice));
                MRQ_CUDA_TRY(cudaMemcpy(dCf + (size_t)j * d, c32.data(), d * 4, cudaMemcpyHostToDevice));
                cnt[big]--;
                cnt[j] = 1;
                a[far] = j;
                dm[far] = 0.f;
            }
            k_rownorm<<<(unsigned)((k + 255) / 256), 256>>>(dCf, k, d, dcn);
        }
        if (prev < INFINITY && (prev - wcss) <= 1e-4 * prev) break;
        prev = wcss;
    }
    MRQ_CUDA_TRY(cudaDeviceSynchronize());
    const double t_km = now_ms();
    // final assignment of all N
    float *dHn;
    BTRY(dv.alloc(&dHn, n));
    k_rownorm<<<(unsigned)((n + 255) / 256), 256>>>(dH, n, d, dHn);
    BTRY(assign_step(dH, dHn, n));
    std::vector<uint32_t> assign(n);
    std::vector<double> C((size_t)k * d);
    MRQ_CUDA_TRY(cudaMemcpy(assign.data(), dA, (size_t)n * 4, cudaMemcpyDeviceToHost));
    MRQ_CUDA_TRY(cudaMemcpy(C.data(), dC, C.size() * 8, cudaMemcpyDeviceToHost));
    MRQ_CUDA_TRY(cudaGetLastError());
    const double t_asg = now_ms();
    // P_r
    const std::vector<double> R = haar(d, bp->seed);
    // ---- the build file (format in include/mrq.h)
    FILE *f = fopen(out_path, "wb");
    if (!f) {
        mrq_set_error("cannot write %s", out_path);
        return MRQ_EIO;
    }
    char sha[64];
    memset(sha, '0', 64);
    if (base_sha256_hex) memcpy(sha, base_sha256_hex, std::min<size_t>(64, strlen(base_sha256_hex)));
    const uint32_t hdr[4] = {1u, (uint32_t)D, (uint32_t)d, (uint32_t)k};
    const uint64_t nn = (uint64_t)n, flags = 0;
    bool ok = fwrite("MRQBLD01", 1, 8, f) == 8 && fwrite(hdr, 4, 4, f) == 4 && fwrite(&nn, 8, 1, f) == 1 &&
              fwrite(&flags, 8, 1, f) == 1 && fwrite(sha, 1, 64, f) == 64 &&
              fwrite(mu.data(), 8, D, f) == (size_t)D && fwrite(P.data(), 8, P.size(), f) == P.size() &&
              fwrite(lam.data(), 8, D, f) == (size_t)D && fwrite(R.data(), 8, R.size(), f) == R.size() &&
              fwrite(C.data(), 8, C.size(), f) == C.size() && fwrite(assign.data(), 4, n, f) == (size_t)n &&
              fwrite("MRQEND01", 1, 8, f) == 8;
    ok = (fclose(f) == 0) && ok;
    if (!ok) {
        mrq_set_error("write error on %s", out_path);
        return MRQ_EIO;
    }
    if (times_ms) {
        times_ms[0] = t_pca - t_start;
        times_ms[1] = t_km - t_pca;
        times_ms[2] = t_asg - t_km;
        times_ms[3] = now_ms() - t_start;
    }
    return MRQ_OK;
}

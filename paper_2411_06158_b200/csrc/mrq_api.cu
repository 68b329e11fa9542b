// mrq_api.cu -- the C ABI of libmrq (include/mrq.h): build-file parsing, HBM
// layout and GPU encoding at load, and the batched search pipeline.
#include <stdarg.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <functional>
#include <cmath>
#include <vector>
#include <thread>

#include <nvtx3/nvToolsExt.h>

#include "mrq_internal.cuh"
#include "mrq_kernels.cuh"
#include "mrq_probe_tc.cuh"
#include "mrq_comm.cuh"

// key of the cached CUDA graph of a search (search_dispatch)
// (gen: the index's scratch generation -- a search that reallocated a
// scratch buffer invalidates every graph captured before, whose kernels hold
// the freed pointers)
struct GraphKey {
    const void *q, *ids, *dist, *stream;
    int64_t nq;
    mrq_search_params p;
    uint64_t gen;
};

// ------------------------------------------------------------------ errors
static thread_local char g_err[1024] = "";

void mrq_set_error(const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

extern "C" const char *mrq_last_error(void) { return g_err; }

#define TRY(expr)                        \
    do {                                 \
        int _rc = (expr);                \
        if (_rc != MRQ_OK) return _rc;   \
    } while (0)

static int dalloc(mrq_index *ix, void **p, size_t bytes)
{
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaSuccess) {
        mrq_set_error("cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
        return MRQ_ENOMEM;
    }
    ix->owned.push_back(*p);
    return MRQ_OK;
}

template <class T>
static int upload(mrq_index *ix, T **dst, const T *src, size_t count)
{
    TRY(dalloc(ix, (void **)dst, count * sizeof(T)));
    MRQ_CUDA_TRY(cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice));
    return MRQ_OK;
}

int mrq_scratch(mrq_index *ix, const char *name, size_t bytes, void **out)
{
    if (bytes == 0) bytes = 16;
    DevArr &a = ix->scratch[name];
    if (a.bytes < bytes) {
        if (a.p) cudaFree(a.p);
        a.p = nullptr;
        size_t want = bytes + bytes / 8;
        cudaError_t e = cudaMalloc(&a.p, want);
        if (e != cudaSuccess) {
            a.bytes = 0;
            mrq_set_error("scratch %s: cudaMalloc(%zu) failed: %s", name, want, cudaGetErrorString(e));
            return MRQ_ENOMEM;
        }
        a.bytes = want;
        ix->scratch_gen++;
    }
    *out = a.p;
    return MRQ_OK;
}

#define SCR(name, T, count, var) TRY(mrq_scratch(ix, name, (size_t)(count) * sizeof(T), (void **)&(var)))

// -------------------------------------------------------------- build file
struct BuildFile {
    uint32_t D = 0, d = 0, k = 0;
    uint64_t N = 0;
    std::vector<double> mu, P, lam, R, C;
    std::vector<uint32_t> assign;
};

// Parses an MRQBLD01 file (format: include/mrq.h) and checks it against the
// caller's D, d, n before any size-dependent allocation: header fields are
// bounded first, the payload size is then computed in 64 bits (no wrap) and
// compared with the file size.  Errors: MRQ_EIO (open/read), MRQ_EVERSION
// (magic, version), MRQ_EDIM (D or d differ), MRQ_EINVAL (n differs from N),
// MRQ_EFORMAT (bad header values, truncation, end marker, assignment >= k;
// the message carries the byte offset).
static int read_build_file(const char *path, BuildFile &b, int32_t D_call, int32_t d_call, int64_t n_call)
{
    FILE *f = fopen(path, "rb");
    if (!f) {
        mrq_set_error("cannot open build file '%s'", path);
        return MRQ_EIO;
    }
    std::vector<unsigned char> buf;
    if (fseek(f, 0, SEEK_END) != 0) {
        fclose(f);
        mrq_set_error("cannot read build file '%s'", path);
        return MRQ_EIO;
    }
    const long fsz = ftell(f);
    rewind(f);
    if (fsz < 0) {
        fclose(f);
        mrq_set_error("cannot read build file '%s'", path);
        return MRQ_EIO;
    }
    buf.resize((size_t)fsz);
    const size_t got = fsz > 0 ? fread(buf.data(), 1, (size_t)fsz, f) : 0;
    fclose(f);
    if (got != (size_t)fsz) {
        mrq_set_error("short read of build file '%s' (%zu of %ld bytes)", path, got, fsz);
        return MRQ_EIO;
    }
    if (buf.size() < 8 || memcmp(buf.data(), "MRQBLD01", 8) != 0) {
        mrq_set_error("build file '%s': bad magic (VersionMismatch)", path);
        return MRQ_EVERSION;
    }
    if (buf.size() < 104) {
        mrq_set_error("build file '%s': truncated header at offset %zu (FormatError)", path, buf.size());
        return MRQ_EFORMAT;
    }
    uint32_t ver;
    memcpy(&ver, buf.data() + 8, 4);
    if (ver != 1) {
        mrq_set_error("build file '%s': version %u != 1 (VersionMismatch)", path, ver);
        return MRQ_EVERSION;
    }
    memcpy(&b.D, buf.data() + 12, 4);
    memcpy(&b.d, buf.data() + 16, 4);
    memcpy(&b.k, buf.data() + 20, 4);
    memcpy(&b.N, buf.data() + 24, 8);
    if (b.D < 1 || b.D > 65536 || b.d < 1 || b.d > b.D || b.k < 1 || b.k > (1u << 24) || b.N > (1ull << 32)) {
        mrq_set_error("build file '%s': bad header D=%u d=%u k=%u N=%llu at offset 12 (FormatError)", path, b.D, b.d,
                      b.k, (unsigned long long)b.N);
        return MRQ_EFORMAT;
    }
    if ((int64_t)b.D != D_call || (int64_t)b.d != d_call) {
        mrq_set_error("DimensionMismatch: file D=%u d=%u, call D=%d d=%d", b.D, b.d, D_call, d_call);
        return MRQ_EDIM;
    }
    if ((int64_t)b.N != n_call) {
        mrq_set_error("InvalidConfig: build file N=%llu, call n=%lld", (unsigned long long)b.N, (long long)n_call);
        return MRQ_EINVAL;
    }
    const uint64_t D = b.D, d = b.d, k = b.k;
    const uint64_t ndbl = D + D * D + D + d * d + k * d;      // all bounded above: no wrap in 64 bits
    const uint64_t need = 104 + 8 * ndbl + 4 * b.N + 8;
    if ((uint64_t)buf.size() < need) {
        // report the offset of the first incomplete section
        uint64_t off = 104;
        const uint64_t sec[6] = {8 * D, 8 * D * D, 8 * D, 8 * d * d, 8 * k * d, 4 * b.N};
        for (uint64_t s : sec) {
            if (off + s > buf.size()) break;
            off += s;
        }
        mrq_set_error("build file '%s': truncated at offset %llu (FormatError; %zu of %llu bytes)", path,
                      (unsigned long long)off, buf.size(), (unsigned long long)need);
        return MRQ_EFORMAT;
    }
    size_t off = 104;
    auto take = [&](std::vector<double> &v, size_t n) {
        v.resize(n);
        memcpy(v.data(), buf.data() + off, n * 8);
        off += n * 8;
    };
    take(b.mu, D);
    take(b.P, D * D);
    take(b.lam, D);
    take(b.R, d * d);
    take(b.C, k * d);
    b.assign.resize(b.N);
    memcpy(b.assign.data(), buf.data() + off, b.N * 4);
    off += b.N * 4;
    if (memcmp(buf.data() + off, "MRQEND01", 8) != 0) {
        mrq_set_error("build file '%s': bad end marker at offset %zu (FormatError)", path, off);
        return MRQ_EFORMAT;
    }
    for (uint64_t n = 0; n < b.N; n++)
        if (b.assign[n] >= b.k) {
            mrq_set_error("build file '%s': assignment %u >= k at vector %llu, offset %llu (FormatError)", path,
                          b.assign[n], (unsigned long long)n, (unsigned long long)(off - b.N * 4 + n * 4));
            return MRQ_EFORMAT;
        }
    return MRQ_OK;
}

// -------------------------------------------------------------------- load
// Locality key of every list (the query processing order, DESIGN.md §5
// "query order"): the centroids are grouped around G = k / 16 (<= 1024)
// centres by a short host k-means (2 Lloyd steps from a strided start, on
// their leading <= 64 principal coordinates; the assignment split over host
// threads), the groups chained greedily (each followed by its nearest
// unvisited group), and a list's key is its rank in (chain position, id)
// order scaled to [0, MRQ_QO_KEYS).  What matters is that the groups are
// fine and that neighbours in the chain are neighbours in space: measured on
// the Deep-shaped probe lists, the lists a window of 1184 consecutive
// queries touches (relative to their probes) fall 0.55 (given order) -> 0.32
// (3 principal coordinates) -> 0.24 (128 groups) -> 0.15 (1024 groups).
// Only the ORDER in which queries are processed depends on it -- never a
// result.
static inline float sqdist_f32(const float *x, const float *y, int n)
{
    float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int i = 0;
    for (; i + 8 <= n; i += 8)
        for (int u = 0; u < 8; u++) {
            const float t = x[i + u] - y[i + u];
            a[u] += t * t;
        }
    float s = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
    for (; i < n; i++) {
        const float t = x[i] - y[i];
        s += t * t;
    }
    return s;
}

static std::vector<uint16_t> list_locality_keys(const std::vector<float> &C32, int k, int d)
{
    std::vector<uint16_t> key((size_t)k, 0);
    int G = std::min(1024, std::max(2, k / 16));
    if (const char *e = getenv("MRQ_QO_GROUPS")) G = std::max(2, std::min(k, atoi(e)));   // A/B experiments
    if (k < 4) return key;
    const int dd = std::min(d, 64);
    std::vector<float> g((size_t)G * dd);
    for (int j = 0; j < G; j++)
        for (int i = 0; i < dd; i++) g[(size_t)j * dd + i] = C32[(size_t)((int64_t)j * k / G) * d + i];
    std::vector<int> asg((size_t)k, 0), cnt((size_t)G);
    std::vector<double> sum((size_t)G * dd);
    const int nth = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    for (int it = 0; it < 2; it++) {
        auto assign = [&](int c0, int c1) {
            for (int c = c0; c < c1; c++) {
                const float *x = &C32[(size_t)c * d];
                float best = INFINITY;
                int bj = 0;
                for (int j = 0; j < G; j++) {
                    const float s = sqdist_f32(x, &g[(size_t)j * dd], dd);
                    if (s < best) {
                        best = s;
                        bj = j;
                    }
                }
                asg[c] = bj;
            }
        };
        std::vector<std::thread> th;
        for (int t = 1; t < nth; t++)
            th.emplace_back(assign, (int)((int64_t)k * t / nth), (int)((int64_t)k * (t + 1) / nth));
        assign(0, (int)((int64_t)k / nth));
        for (auto &t : th) t.join();
        std::fill(cnt.begin(), cnt.end(), 0);
        std::fill(sum.begin(), sum.end(), 0.0);
        for (int c = 0; c < k; c++) {
            cnt[asg[c]]++;
            for (int i = 0; i < dd; i++) sum[(size_t)asg[c] * dd + i] += C32[(size_t)c * d + i];
        }
        for (int j = 0; j < G; j++)
            if (cnt[j] > 0)
                for (int i = 0; i < dd; i++) g[(size_t)j * dd + i] = (float)(sum[(size_t)j * dd + i] / cnt[j]);
    }
    // greedy chain over the groups
    std::vector<int> pos((size_t)G, -1);
    int cur = 0;
    for (int n = 0; n < G; n++) {
        pos[cur] = n;
        float best = INFINITY;
        int bj = -1;
        for (int j = 0; j < G; j++) {
            if (pos[j] >= 0) continue;
            const float s = sqdist_f32(&g[(size_t)cur * dd], &g[(size_t)j * dd], dd);
            if (s < best || bj < 0) {
                best = s;
                bj = j;
            }
        }
        if (bj < 0) break;
        cur = bj;
    }
    std::vector<int> order((size_t)k);
    for (int c = 0; c < k; c++) order[c] = c;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return pos[asg[a]] < pos[asg[b]]; });
    for (int r = 0; r < k; r++) key[order[r]] = (uint16_t)((int64_t)r * MRQ_QO_KEYS / k);
    return key;
}

static int load_impl(mrq_index *ix, const char *build_file, const float *base, int64_t n, int32_t D, int32_t d,
                     const mrq_dist_cfg *dist)
{
    if (!build_file || !base) {
        mrq_set_error("NULL build_file or base");
        return MRQ_EINVAL;
    }
    if (d < 2 || d > D) {
        mrq_set_error("InvalidConfig: need 2 <= d <= D (d=%d, D=%d)", d, D);
        return MRQ_EINVAL;
    }
    BuildFile b;
    TRY(read_build_file(build_file, b, D, d, n));
    ix->N = n;
    ix->D = D;
    ix->d = d;
    ix->k = (int)b.k;
    ix->W = (d + 31) / 32;   // any d loads; the MRQ modes need supported_W (d <= 512), EXACT does not
    const int k = ix->k, W = ix->W;

    // multi-GPU placement: owned lists (greedy by size), device
    int ndev = 0;
    MRQ_CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (ndev < 1) {
        mrq_set_error("no CUDA device");
        return MRQ_ECUDA;
    }
    ix->rank = dist ? dist->rank : 0;
    ix->world = dist && dist->world > 1 ? dist->world : 1;
    ix->device = dist && dist->device >= 0 ? dist->device : -1;
    if (ix->device < 0) MRQ_CUDA_TRY(cudaGetDevice(&ix->device));
    MRQ_CUDA_TRY(cudaSetDevice(ix->device));
    MRQ_CUDA_TRY(cudaDeviceGetAttribute(&ix->sm_count, cudaDevAttrMultiProcessorCount, ix->device));
    MRQ_CUDA_TRY(cudaDeviceGetAttribute(&ix->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ix->device));
    MRQ_CUDA_TRY(cudaStreamCreateWithFlags(&ix->stream, cudaStreamNonBlocking));
    for (auto &e : ix->ev) MRQ_CUDA_TRY(cudaEventCreate(&e));
    MRQ_CUDA_TRY(cudaStreamCreateWithFlags(&ix->side, cudaStreamNonBlocking));
    for (auto &e : ix->ev_fork) MRQ_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));

    std::vector<uint32_t> cnt(k, 0);
    for (int64_t i = 0; i < n; i++) cnt[b.assign[i]]++;
    std::vector<uint8_t> own(k, 1);
    if (ix->world > 1) {
        std::vector<uint32_t> owner;
        mrq_shard_lists(cnt, ix->world, owner);
        for (int c = 0; c < k; c++) own[c] = owner[c] == (uint32_t)ix->rank;
        TRY(mrq_comm_init(ix, dist));
    } else if (dist && dist->nccl_unique_id) {
        // a one-rank NCCL communicator: the sharded path (mrq_debug_set
        // "force_exchange") then runs its all-gathers through NCCL
        TRY(mrq_comm_init(ix, dist));
    }
    // list slots: owned lists only, each start aligned to MRQ_SLOT_ALIGN
    ix->h_list_off.assign(k + 1, 0);
    ix->h_list_size.assign(k, 0);
    uint64_t pos = 0;
    for (int c = 0; c < k; c++) {
        ix->h_list_off[c] = (uint32_t)pos;
        ix->h_list_size[c] = own[c] ? cnt[c] : 0;
        pos += ix->h_list_size[c];
        pos = (pos + MRQ_SLOT_ALIGN - 1) / MRQ_SLOT_ALIGN * MRQ_SLOT_ALIGN;
        ix->max_list = std::max(ix->max_list, ix->h_list_size[c]);
    }
    ix->h_list_off[k] = (uint32_t)pos;
    {
        std::vector<uint32_t> srt(ix->h_list_size);
        std::sort(srt.begin(), srt.end(), std::greater<uint32_t>());
        ix->h_topsum.assign(k + 1, 0);
        for (int c = 0; c < k; c++) ix->h_topsum[c + 1] = ix->h_topsum[c] + srt[c];
    }
    ix->npad = (int64_t)((pos + 256 + 127) / 128 * 128);   // scan tiles may read 256 slots past a list start
    if (ix->npad >= (int64_t)0xFFFFFFF0ll) {
        mrq_set_error("index too large for 32-bit slots");
        return MRQ_EINVAL;
    }
    const int64_t npad = ix->npad;
    std::vector<uint32_t> slot_of(n, 0xFFFFFFFFu), ids(npad, MRQ_PAD_ID), fill(k, 0);
    for (int64_t i = 0; i < n; i++) {
        const uint32_t c = b.assign[i];
        if (!own[c]) continue;
        const uint32_t s = ix->h_list_off[c] + fill[c]++;
        slot_of[i] = s;
        ids[s] = (uint32_t)i;
    }

    // replicated model: mu, P^T, lambda, R^T, centroids (+ transposed/fp32 copies)
    std::vector<double> PT((size_t)D * D), RT((size_t)d * d);
    for (int i = 0; i < D; i++)
        for (int j = 0; j < D; j++) PT[(size_t)j * D + i] = b.P[(size_t)i * D + j];
    for (int j = 0; j < d; j++)
        for (int i = 0; i < d; i++) RT[(size_t)i * d + j] = b.R[(size_t)j * d + i];
    // ||c||^2 padded with +inf to a whole number of 256-column probe tiles
    std::vector<float> C32T((size_t)d * k), C32((size_t)k * d), cn32((k + 255) / 256 * 256, INFINITY);
    double cmax = 0.0;
    for (int c = 0; c < k; c++) {
        double s = 0.0;
        for (int i = 0; i < d; i++) {
            const double v = b.C[(size_t)c * d + i];
            C32T[(size_t)i * k + c] = (float)v;
            C32[(size_t)c * d + i] = (float)v;
            s += v * v;
        }
        cn32[c] = (float)s;
        cmax = std::max(cmax, std::sqrt(s));
    }
    ix->cmax = cmax * (1.0 + 1e-9) + 1e-300;
    TRY(upload(ix, &ix->mu, b.mu.data(), D));
    TRY(upload(ix, &ix->PT, PT.data(), PT.size()));
    TRY(upload(ix, &ix->lam, b.lam.data(), D));
    TRY(upload(ix, &ix->RT, RT.data(), RT.size()));
    TRY(upload(ix, &ix->C, b.C.data(), b.C.size()));
    TRY(upload(ix, &ix->C32T, C32T.data(), C32T.size()));
    TRY(upload(ix, &ix->C32, C32.data(), C32.size()));
    TRY(upload(ix, &ix->cn32, cn32.data(), cn32.size()));
    TRY(upload(ix, &ix->list_off, ix->h_list_off.data(), k + 1));
    TRY(upload(ix, &ix->list_size, ix->h_list_size.data(), k));
    TRY(upload(ix, &ix->list_size_g, cnt.data(), k));
    TRY(upload(ix, &ix->ids, ids.data(), npad));
    {
        const std::vector<uint16_t> lkey = list_locality_keys(C32, k, d);
        TRY(upload(ix, &ix->list_key, lkey.data(), (size_t)k));
    }
    TRY(dalloc(ix, (void **)&ix->Rc, (size_t)k * d * 8));
    k_rc<<<(k + 7) / 8, 256, 0, ix->stream>>>(ix->C, ix->RT, k, d, W, ix->Rc);

    // encoded index in HBM (slot order)
    TRY(dalloc(ix, (void **)&ix->codes, (size_t)W * npad * 4));
    TRY(dalloc(ix, (void **)&ix->f1, (size_t)npad * 4));
    TRY(dalloc(ix, (void **)&ix->f2, (size_t)npad * 4));
    TRY(dalloc(ix, (void **)&ix->f3, (size_t)npad * 4));
    TRY(dalloc(ix, (void **)&ix->xr2, (size_t)npad * 4));
    TRY(dalloc(ix, (void **)&ix->heads, (size_t)npad * d * 4));
    ix->dq = (d + 15) / 16 * 16;
    TRY(dalloc(ix, (void **)&ix->hq, (size_t)npad * ix->dq));
    TRY(dalloc(ix, (void **)&ix->hs, (size_t)npad * sizeof(float4)));
    MRQ_CUDA_TRY(cudaMemsetAsync(ix->hq, 0, (size_t)npad * ix->dq, ix->stream));
    MRQ_CUDA_TRY(cudaMemsetAsync(ix->hs, 0, (size_t)npad * sizeof(float4), ix->stream));
    if (ix->tails_host) {   // NEXT-4: tails in pinned host memory, read through the mapped device pointer
        const size_t tb = (size_t)npad * std::max(D - d, 1) * 4;
        if (cudaHostAlloc(&ix->tails_hbuf, tb, cudaHostAllocMapped) != cudaSuccess) {
            ix->tails_hbuf = nullptr;
            mrq_set_error("cudaHostAlloc(%zu) for host tails failed", tb);
            return MRQ_ENOMEM;
        }
        MRQ_CUDA_TRY(cudaHostGetDevicePointer((void **)&ix->tails, ix->tails_hbuf, 0));
    } else {
        TRY(dalloc(ix, (void **)&ix->tails, (size_t)npad * std::max(D - d, 1) * 4));
    }
    MRQ_CUDA_TRY(cudaMemsetAsync(ix->codes, 0, (size_t)W * npad * 4, ix->stream));
    MRQ_CUDA_TRY(cudaMemsetAsync(ix->f1, 0, (size_t)npad * 4, ix->stream));
    MRQ_CUDA_TRY(cudaMemsetAsync(ix->f2, 0, (size_t)npad * 4, ix->stream));
    MRQ_CUDA_TRY(cudaMemsetAsync(ix->f3, 0, (size_t)npad * 4, ix->stream));
    MRQ_CUDA_TRY(cudaMemsetAsync(ix->xr2, 0, (size_t)npad * 4, ix->stream));

    // encode owned vectors in chunks (Alg.1 L3-L8 on the GPU)
    std::vector<uint32_t> own_ids;
    own_ids.reserve(n);
    for (int64_t i = 0; i < n; i++)
        if (slot_of[i] != 0xFFFFFFFFu) own_ids.push_back((uint32_t)i);
    const int64_t CH = 65536;
    float *dX = nullptr;
    double *dXp = nullptr;
    uint32_t *dAssign = nullptr, *dSlot = nullptr;
    TRY(mrq_scratch(ix, "enc_x", (size_t)CH * D * 4, (void **)&dX));
    TRY(mrq_scratch(ix, "enc_xp", (size_t)CH * D * 8, (void **)&dXp));
    TRY(mrq_scratch(ix, "enc_assign", (size_t)CH * 4, (void **)&dAssign));
    TRY(mrq_scratch(ix, "enc_slot", (size_t)CH * 4, (void **)&dSlot));
    std::vector<float> hx((size_t)CH * D);
    std::vector<uint32_t> ha(CH), hs(CH);
    const int enc_warps = 8;
    const size_t enc_smem = (size_t)enc_warps * 2 * d * 8;
    if (enc_smem > 48 * 1024)
        MRQ_CUDA_TRY(cudaFuncSetAttribute(k_encode_finish, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)enc_smem));
    for (int64_t s = 0; s < (int64_t)own_ids.size(); s += CH) {
        const int64_t m = std::min<int64_t>(CH, (int64_t)own_ids.size() - s);
        for (int64_t r = 0; r < m; r++) {
            const uint32_t id = own_ids[s + r];
            memcpy(&hx[(size_t)r * D], base + (size_t)id * D, (size_t)D * 4);
            ha[r] = b.assign[id];
            hs[r] = slot_of[id];
        }
        MRQ_CUDA_TRY(cudaMemcpyAsync(dX, hx.data(), (size_t)m * D * 4, cudaMemcpyHostToDevice, ix->stream));
        MRQ_CUDA_TRY(cudaMemcpyAsync(dAssign, ha.data(), (size_t)m * 4, cudaMemcpyHostToDevice, ix->stream));
        MRQ_CUDA_TRY(cudaMemcpyAsync(dSlot, hs.data(), (size_t)m * 4, cudaMemcpyHostToDevice, ix->stream));
        launch_rowmat_f32(dX, m, D, D, ix->mu, ix->PT, D, dXp, D, ix->stream);
        k_encode_finish<<<(unsigned)((m + enc_warps - 1) / enc_warps), enc_warps * 32, enc_smem, ix->stream>>>(
            dXp, 0, m, D, d, W, dAssign, dSlot, ix->C, ix->RT, npad, ix->heads, ix->tails, ix->xr2, ix->codes, ix->f1,
            ix->f2, ix->f3, ix->hq, ix->hs, ix->dq);
        MRQ_CUDA_TRY(cudaGetLastError());
        MRQ_CUDA_TRY(cudaStreamSynchronize(ix->stream));   // hx is reused
    }
    MRQ_CUDA_TRY(cudaStreamSynchronize(ix->stream));
    for (const char *nm : {"enc_x", "enc_xp", "enc_assign", "enc_slot"}) {
        DevArr &a = ix->scratch[nm];
        if (a.p) cudaFree(a.p);
        ix->scratch.erase(nm);
    }
    TRY(mrq_probe_tc_init(ix));
    return MRQ_OK;
}

extern "C" int mrq_index_load(const char *build_file, const float *base, int64_t n, int32_t D, int32_t d,
                              const mrq_dist_cfg *dist, mrq_index **out)
{
    return mrq_index_load_ex(build_file, base, n, D, d, dist, 0u, out);
}

extern "C" int mrq_index_load_ex(const char *build_file, const float *base, int64_t n, int32_t D, int32_t d,
                                 const mrq_dist_cfg *dist, uint32_t flags, mrq_index **out)
{
    if (!out) {
        mrq_set_error("NULL out");
        return MRQ_EINVAL;
    }
    *out = nullptr;
    if (flags & ~MRQ_LOAD_TAILS_HOST) {
        mrq_set_error("InvalidConfig: unknown load flags 0x%x", flags);
        return MRQ_EINVAL;
    }
    mrq_index *ix = new mrq_index();
    ix->tails_host = (flags & MRQ_LOAD_TAILS_HOST) != 0;
    ix->g_key = new GraphKey();
    ix->g_pending = new GraphKey();
    memset(ix->g_key, 0, sizeof(GraphKey));
    memset(ix->g_pending, 0, sizeof(GraphKey));
    if (getenv("MRQ_NO_GRAPHS")) ix->graphs = 0;
    if (getenv("MRQ_NO_SKETCH")) ix->sketch_on = 0;
    int rc = mrq_guard([&] { return load_impl(ix, build_file, base, n, D, d, dist); });
    if (rc != MRQ_OK) {
        mrq_free(ix);
        return rc;
    }
    *out = ix;
    return MRQ_OK;
}

extern "C" void mrq_free(mrq_index *ix)
{
    if (!ix) return;
    if (ix->device >= 0) cudaSetDevice(ix->device);
    if (ix->stream) cudaStreamSynchronize(ix->stream);
    for (void *p : ix->owned) cudaFree(p);
    if (ix->tails_hbuf) cudaFreeHost(ix->tails_hbuf);
    for (auto &kv : ix->scratch)
        if (kv.second.p) cudaFree(kv.second.p);
    mrq_probe_tc_free(ix);
    if (ix->gexec) cudaGraphExecDestroy((cudaGraphExec_t)ix->gexec);
    delete (GraphKey *)ix->g_key;
    delete (GraphKey *)ix->g_pending;
    mrq_comm_free(ix);
    for (auto &e : ix->ev)
        if (e) cudaEventDestroy(e);
    if (ix->stream) cudaStreamDestroy(ix->stream);
    for (auto e : ix->ev_fork)
        if (e) cudaEventDestroy(e);
    if (ix->side) cudaStreamDestroy(ix->side);
    delete ix;
}

extern "C" int mrq_index_info(const mrq_index *ix, int64_t *n, int32_t *D, int32_t *d, int32_t *k, int64_t *npad)
{
    if (!ix) {
        mrq_set_error("NULL index");
        return MRQ_EINVAL;
    }
    if (n) *n = ix->N;
    if (D) *D = ix->D;
    if (d) *d = ix->d;
    if (k) *k = ix->k;
    if (npad) *npad = ix->npad;
    return MRQ_OK;
}

// ------------------------------------------------------------------ search
// NVTX ranges: one range per search with a nested range per
// stage (host-side; nvtx3 is header-only and free without a tool attached)
struct NvtxStages {
    bool open = false;
    NvtxStages() { nvtxRangePushA("mrq_search"); }
    void stage(const char *name)
    {
        if (open) nvtxRangePop();
        nvtxRangePushA(name);
        open = true;
    }
    ~NvtxStages()
    {
        if (open) nvtxRangePop();
        nvtxRangePop();
    }
};

static int search_impl(mrq_index *ix, const float *d_q, int64_t nq, const mrq_search_params *p, int64_t *d_ids,
                       float *d_dist, mrq_stats *stats, cudaStream_t st)
{
    const int D = ix->D, d = ix->d, k = ix->k, W = ix->W;
    const int K = p->K, np = std::min(p->nprobe, k);
    const int Kp = p->seed_mult * K;
    const int mode = p->mode, tight = p->tau_schedule == 0;
    const double isd = 1.0 / std::sqrt((double)d);
    const bool timed = stats != nullptr;
    NvtxStages nvtx;
    if (timed) MRQ_CUDA_TRY(cudaEventRecord(ix->ev[0], st));
    uint32_t *qorder = nullptr;

    // Query-sharded front end (world > 1): rank r computes a1-a3
    // (projection, probe, quantization) for the query rows [q0, q0 + nr) only;
    // the per-query results are then all-gathered (in place, rank-major rows
    // of S = ceil(nq / world)) so every rank holds every query's probe order,
    // planes and constants -- bit-identical to computing them itself.
    const bool sharded = ix->world > 1 || ix->force_exchange;
    const bool fshard = ix->world > 1 && ix->front_shard;
    const int64_t S = fshard ? (nq + ix->world - 1) / ix->world : nq;
    const int64_t q0 = fshard ? (int64_t)ix->rank * S : 0;
    const int64_t nr = fshard ? std::max<int64_t>(0, std::min<int64_t>(nq, q0 + S) - q0) : nq;
    const int64_t nrow = fshard ? S * ix->world : nq;   // rows of the per-query front arrays
    double *qp, *qr2, *eps_r, *r0, *qnorm, *tau0, *tau1, *probe_qn2, *qconst, *s0_exact, *s1_exact;
    float *qd32, *approx, *qa3 = nullptr;
    uint32_t *probe, *planes, *s0_cnt, *s0_pos, *s1_cnt, *s1_pos, *f1_cnt, *f2_cnt, *exact_cnt, *fallback;
    uint64_t *cand_cnt, *f1_off;
    SCR("qp", double, nrow * D, qp);
    SCR("qr2", double, nrow, qr2);
    SCR("eps_r", double, nrow, eps_r);
    SCR("r0", double, nrow * d, r0);
    SCR("qnorm", double, nrow, qnorm);
    SCR("qd32", float, nrow * d, qd32);
    if (mrq_probe_tc_enabled(ix)) SCR("qa3", float, nrow * 3 * d, qa3);   // 3xTF32 A operand
    SCR("tau0", double, nq, tau0);
    SCR("tau1", double, nq, tau1);
    SCR("probe", uint32_t, nrow * np, probe);
    SCR("probe_qn2", double, nrow * np, probe_qn2);
    SCR("planes", uint32_t, nrow * np * MRQ_BQ * W, planes);
    SCR("qconst", double, nrow * np * 8, qconst);
    SCR("cand_cnt", uint64_t, nq + 1, cand_cnt);
    SCR("f1_off", uint64_t, nq + 1, f1_off);
    SCR("s0_cnt", uint32_t, nq, s0_cnt);
    SCR("s0_pos", uint32_t, nq * Kp, s0_pos);
    SCR("s0_exact", double, nq * Kp, s0_exact);
    SCR("s1_cnt", uint32_t, nq, s1_cnt);
    SCR("s1_pos", uint32_t, nq * Kp, s1_pos);
    SCR("s1_exact", double, nq * Kp, s1_exact);
    uint32_t *s0_id, *s1_id;
    SCR("s0_id", uint32_t, nq * Kp, s0_id);
    SCR("s1_id", uint32_t, nq * Kp, s1_id);
    const int Lx = std::max(Kp, K);
    XItem *xsend = nullptr, *xrecv = nullptr;
    if (sharded) {
        SCR("xsend", XItem, nq * Lx, xsend);
        SCR("xrecv", XItem, (size_t)nq * Lx * ix->world, xrecv);
    }
    SCR("f1_cnt", uint32_t, nq, f1_cnt);
    SCR("f2_cnt", uint32_t, nq, f2_cnt);
    SCR("exact_cnt", uint32_t, nq, exact_cnt);
    SCR("fallback", uint32_t, 1, fallback);
    MRQ_CUDA_TRY(cudaMemsetAsync(fallback, 0, 4, st));

    // head sketch: the scan drops F1 entries whose lower bound
    // of the canonical dis_o' already fails the F2 test (LOOSE: tau1 = tau0)
    const bool want_sketch = ix->sketch_on && mode == 0 && !tight && !ix->dbg_dump_dis &&
                             mrq_scan_sketch_fits(np, ix->npad) &&
                             mrq_scan_smem_sk(np, W, ix->dq) <= (size_t)std::min(ix->smem_optin, 64 * 1024);
    uint8_t *qsk_b = nullptr;
    double *qsk_c = nullptr;
    if (want_sketch) {
        SCR("qsk_b", uint8_t, (size_t)nrow * np * ix->dq, qsk_b);
        SCR("qsk_c", double, (size_t)nrow * np * 4, qsk_c);
    }
    uint16_t *qkey = nullptr;
    if (ix->qorder_on && nq > 1) {
        SCR("qorder", uint32_t, nq, qorder);
        SCR("qkey", uint16_t, nrow, qkey);
    }
    const bool pc_key = qkey && ix->qorder_on == 1;   // key from the projection (k_qtail); else from the probe
    // side stream: r0 = R q_d (only the quantizer needs it) and, with the
    // order key from the projection (qorder = 1), the order's single-block
    // sort (all queries are local unless the front end is sharded).  Forked
    // right after k_qtail with qorder = 1; with the key from the probe
    // (qorder = 2) after the probe screen has been launched, so that the
    // persistent probe CTAs take their SMs first and r0 runs beside the probe
    // finish (forked before the screen, r0's blocks delayed some probe CTAs:
    // screen + 5 us).
    auto fork_r0 = [&]() -> int {
        MRQ_CUDA_TRY(cudaEventRecord(ix->ev_fork[0], st));
        MRQ_CUDA_TRY(cudaStreamWaitEvent(ix->side, ix->ev_fork[0], 0));
        if (pc_key && !fshard) launch_qorder(qkey, nq, qorder, ix->side);
        launch_rowmat_f64(qp + q0 * D, nr, D, d, nullptr, ix->RT, d, r0 + q0 * d, d, ix->side);
        MRQ_CUDA_TRY(cudaEventRecord(ix->ev_fork[3], ix->side));
        return MRQ_OK;
    };
    // ---- a1: query projection (Alg.2 L1-L4), rows [q0, q0 + nr)
    nvtx.stage("a1 projection");
    if (nr > 0) {
        launch_rowmat_f32(d_q + q0 * D, nr, D, D, ix->mu, ix->PT, D, qp + q0 * D, D, st);   // q_p = P (q - mu)
        const size_t qsmem = (size_t)D * 8 * 9;                                              // lambda + 8 query rows
        if (qsmem > 48 * 1024)
            MRQ_CUDA_TRY(cudaFuncSetAttribute(k_qtail, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qsmem));
        k_qtail<<<(unsigned)((nr + 7) / 8), 256, qsmem, st>>>(
            qp + q0 * D, nr, D, d, W, ix->lam, ix->RT, p->resid_scale, p->m, qr2 + q0, eps_r + q0, r0 + q0 * d,
            qd32 + q0 * d, qnorm + q0, pc_key ? qkey + q0 : nullptr, qa3 ? qa3 + q0 * 3 * d : nullptr);
        if (pc_key) TRY(fork_r0());
    }
    if (timed) MRQ_CUDA_TRY(cudaEventRecord(ix->ev[1], st));

    // ---- a2: probe (Alg.2 L7): screen + exact selection, rows [q0, q0 + nr)
    nvtx.stage("a2 probe");
    if (nr > 0) {
        uint32_t *cand, *ncand;
        // the margin set per query: <= k entries (unfused), <= the parts'
        // buffers when fused (an overflowing row rescores all k without it)
        const bool fused = mrq_probe_tc_fusable(ix, np);
        const int64_t cper = fused ? std::min<int64_t>(k, (int64_t)mrq_probe_tc_parts(ix, nr) * mrq_probe_tc_capp(ix, np))
                                   : k;
        SCR("probe_cand", uint32_t, nr * cper, cand);
        SCR("probe_ncand", uint32_t, nr, ncand);
        double *qp_r = qp + q0 * D, *qn_r = qnorm + q0, *pq_r = probe_qn2 + q0 * np;
        uint32_t *pr_r = probe + q0 * np;
        if (fused) {   // tcgen05 screen with the running top-np in its epilogue
            const int P = mrq_probe_tc_parts(ix, nr), capp = mrq_probe_tc_capp(ix, np);
            uint2 *cbuf;
            uint32_t *ccnt;
            float *kvbuf;
            SCR("probe_cbuf", uint2, (size_t)nr * P * capp, cbuf);
            SCR("probe_ccnt", uint32_t, (size_t)nr * P, ccnt);
            SCR("probe_kv", float, (size_t)nr * P * np, kvbuf);
            uint32_t *gkey = nullptr;
            if (ix->probe_share) SCR("probe_gkey", uint32_t, (size_t)nr, gkey);
            const double kappa = mrq_probe_tc_kappa(ix);
            TRY(mrq_probe_tc_run_fused(ix, qa3 + q0 * 3 * d, nr, np, qn_r, kappa, cbuf, capp, ccnt, kvbuf, gkey, st));
            if (!pc_key) TRY(fork_r0());
            if (timed) MRQ_CUDA_TRY(cudaEventRecord(ix->ev[11], st));
            TRY(launch_probe_finish_w(nr, k, d, np, qp_r, D, ix->C, qn_r, ix->cmax, kappa, cbuf, P, capp,
                                      mrq_probe_tc_grid(ix, nr), ccnt, kvbuf, cand, pr_r, pq_r, ncand, st));
        } else {
            SCR("approx", float, nr * k, approx);
            double kappa;
            if (mrq_probe_tc_enabled(ix)) {
                TRY(mrq_probe_tc_run(ix, qa3 + q0 * 3 * d, nr, approx, st));
                kappa = mrq_probe_tc_kappa(ix);
            } else {
                dim3 grid((k + 255) / 256, (unsigned)((nr + 7) / 8));
                k_probe_approx<<<grid, 256, 8 * d * sizeof(float), st>>>(qd32 + q0 * d, nr, d, k, ix->C32T, approx);
                kappa = std::ldexp(1.0, -24) * (2.0 * d + 8.0);
            }
            if (!pc_key) TRY(fork_r0());
            if (timed) MRQ_CUDA_TRY(cudaEventRecord(ix->ev[11], st));
            TRY(launch_probe_select_w(approx, nr, k, d, np, qp_r, D, ix->C, qn_r, ix->cmax, kappa, cand, pr_r, pq_r,
                                      ncand, st));
        }
    } else if (timed) {
        MRQ_CUDA_TRY(cudaEventRecord(ix->ev[11], st));
    }
    if (timed) MRQ_CUDA_TRY(cudaEventRecord(ix->ev[2], st));

    // ---- a3: per-(query, list) quantization into bit-planes, rows [q0, q0 + nr)
    nvtx.stage("a3 quantization");
    // list-major scan: the (query, list) pairs grouped by list,
    // built on the side stream beside the quantizer
    const bool use_lm = ix->scan_lm && mode != 2 && W <= 4 && !ix->dbg_dump_dis;
    const int lm_qg = ix->scan_lm == 2 ? 8 : ix->lm_qg;   // the tensor-core form takes 8 pairs (one MMA n-block)
    LmScratch lms;
    memset(&lms, 0, sizeof lms);
    if (use_lm) {
        SCR("lm_lcnt", uint32_t, k, lms.lcnt);
        SCR("lm_lfill", uint32_t, k, lms.lfill);
        SCR("lm_loff", uint32_t, k + 1, lms.loff);
        SCR("lm_upre", uint32_t, k + 1, lms.upre);
        SCR("lm_pairs", uint32_t, std::max<int64_t>(nq * np, 1), lms.pairs);
        SCR("lm_unit", uint32_t, 1, lms.unit_ctr);
        // units of list c = tiles_c ceil(n_c / qg) <= tiles_c n_c: at most ceil(max_list / 128) per pair
        SCR("lm_units", uint32_t, std::max<int64_t>(nq * np * (int64_t)((ix->max_list + 127) / 128), 1), lms.unit_list);
    }
    auto fork_offsets = [&]() -> int {   // F1 segment offsets of all nq queries on the side stream
        MRQ_CUDA_TRY(cudaEventRecord(ix->ev_fork[1], st));
        MRQ_CUDA_TRY(cudaStreamWaitEvent(ix->side, ix->ev_fork[1], 0));
        if (pc_key && fshard) launch_qorder(qkey, nq, qorder, ix->side);
        if (use_lm) TRY(mrq_lm_build(probe, nq, np, k, ix->list_size, lm_qg, lms, ix->side));
        // (qorder = 2: the order key of the nearest probed list -- every query's probe row is here by now)
        const bool probe_key = qkey && !pc_key;
        k_cand_count<<<(unsigned)((nq + 255) / 256), 256, 0, ix->side>>>(probe, nq, np, ix->list_size, cand_cnt,
                                                                         ix->list_key, probe_key ? qkey : nullptr);
        if (probe_key)
            k_offsets_order<<<2, 1024, 0, ix->side>>>(cand_cnt, nq, f1_off, qkey, qorder);
        else
            k_exclusive_scan<<<1, 1024, 0, ix->side>>>(cand_cnt, nq, f1_off);
        MRQ_CUDA_TRY(cudaEventRecord(ix->ev_fork[2], ix->side));
        return MRQ_OK;
    };
    if (!fshard) TRY(fork_offsets());   // beside the quantizer
    MRQ_CUDA_TRY(cudaStreamWaitEvent(st, ix->ev_fork[3], 0));   // r0 (joins the side stream in every mode)
    if (nr > 0 && mode != 2) {   // EXACT reads no code: no query quantization
        launch_quant(probe + q0 * np, probe_qn2 + q0 * np, nr, np, d, W, r0 + q0 * d, ix->Rc, qr2 + q0, p->eps0,
                     planes + q0 * np * MRQ_BQ * W, qconst + q0 * np * 8, qsk_b ? qsk_b + q0 * np * ix->dq : nullptr,
                     qsk_c ? qsk_c + q0 * np * 4 : nullptr, ix->dq, qnorm + q0, ix->cmax, st);
    }
    if (fshard) {
        // every rank's rows to every rank: one grouped in-place all-gather
        std::vector<char *> base;
        std::vector<size_t> rowb;
        auto sec = [&](void *ptr, size_t b) {
            base.push_back((char *)ptr);
            rowb.push_back(b);
        };
        sec(qp, (size_t)D * 8);
        sec(qr2, 8);
        sec(eps_r, 8);
        sec(probe, (size_t)np * 4);
        sec(probe_qn2, (size_t)np * 8);
        sec(planes, (size_t)np * MRQ_BQ * W * 4);
        sec(qconst, (size_t)np * 8 * 8);
        if (pc_key) sec(qkey, 2);
        if (qsk_b) {
            sec(qsk_b, (size_t)np * ix->dq);
            sec(qsk_c, (size_t)np * 4 * 8);
        }
        std::vector<const void *> sends(base.size());
        std::vector<void *> recvs(base.size());
        std::vector<size_t> bytes(base.size());
        for (size_t i = 0; i < base.size(); i++) {
            bytes[i] = (size_t)S * rowb[i];
            sends[i] = base[i] + (size_t)ix->rank * bytes[i];
            recvs[i] = base[i];
        }
        TRY(mrq_allgather_group(ix, (int)base.size(), sends.data(), recvs.data(), bytes.data(), st));
    }
    if (fshard) TRY(fork_offsets());      // after the all-gather: every query's probe lists
    MRQ_CUDA_TRY(cudaStreamWaitEvent(st, ix->ev_fork[2], 0));   // join
    // candidate-indexed scratch: sized by the host bound nq x (sum of the np
    // largest lists) when that fits the budget, so the search never waits on
    // the device; else by the exact total (one D2H + stream sync)
    uint64_t total = (uint64_t)nq * ix->h_topsum[std::min(np, k)];
    const uint64_t per_entry = 4 + 8 + 8 + 4 + 4 + 8 + 8;   // f1_pos/head/diso/id, f2_pos/head/exact
    if (total * per_entry > ix->cand_budget || ix->dbg_dump_dis) {
        MRQ_CUDA_TRY(cudaMemcpyAsync(&total, f1_off + nq, 8, cudaMemcpyDeviceToHost, st));
        MRQ_CUDA_TRY(cudaStreamSynchronize(st));
    }
#if defined(MRQ_CHECK) && MRQ_CHECK
    {   // the host bound must cover the exact candidate total (MRQ_CHECK build only: one sync)
        uint64_t exact_total = 0;
        MRQ_CUDA_TRY(cudaMemcpyAsync(&exact_total, f1_off + nq, 8, cudaMemcpyDeviceToHost, st));
        MRQ_CUDA_TRY(cudaStreamSynchronize(st));
        if (exact_total > total) {
            mrq_set_error("MRQ_CHECK: candidate total %llu exceeds the scratch bound %llu",
                          (unsigned long long)exact_total, (unsigned long long)total);
            return MRQ_EINVAL;
        }
    }
#endif
    ix->last_total = total;
    uint32_t *f1_pos, *f2_pos;
    double *f1_head, *f1_diso, *f2_head, *f2_exact;
    SCR("f1_pos", uint32_t, total, f1_pos);
    SCR("f1_head", double, total, f1_head);
    SCR("f1_diso", double, total, f1_diso);
    SCR("f2_pos", uint32_t, total, f2_pos);
    SCR("f2_head", double, total, f2_head);
    SCR("f2_exact", double, total, f2_exact);
    uint32_t *f1_id;
    SCR("f1_id", uint32_t, total, f1_id);
    // head sketch pre-pass of the stage-2 gather (LOOSE): probe index per F1
    // entry (written by the scan) and the compacted survivors
    uint32_t *surv_cnt = nullptr;
    if (want_sketch) SCR("surv_cnt", uint32_t, nq, surv_cnt);
    if (timed) MRQ_CUDA_TRY(cudaEventRecord(ix->ev[3], st));

    StageArgs sa;
    memset(&sa, 0, sizeof sa);
    sa.nq = nq; sa.np = np; sa.K = K; sa.Kp = Kp; sa.D = D; sa.d = d; sa.mode = mode; sa.tight = tight;
    sa.aligned = (D % 4 == 0) && (d % 4 == 0);
    sa.aligned_tails = sa.aligned && !ix->tails_host;   // host tails: direct loads over the link, no cp.async
    sa.npad = ix->npad; sa.isd = isd; sa.probe = probe; sa.list_off = ix->list_off; sa.list_size = ix->list_size;
    sa.ids = ix->ids; sa.codes = ix->codes; sa.planes = planes; sa.f1 = ix->f1; sa.f2 = ix->f2; sa.f3 = ix->f3;
    sa.heads = ix->heads; sa.tails = ix->tails; sa.xr2 = ix->xr2; sa.qconst = qconst; sa.qp = qp; sa.qr2 = qr2;
    sa.eps_r = eps_r; sa.s0_cnt = s0_cnt; sa.s0_pos = s0_pos; sa.s1_cnt = s1_cnt; sa.s1_pos = s1_pos;
    sa.f1_cnt = f1_cnt; sa.f1_pos = f1_pos; sa.f2_cnt = f2_cnt; sa.f2_pos = f2_pos; sa.exact_cnt = timed ? exact_cnt : nullptr;
    sa.qorder = qorder;
    sa.s0_exact = s0_exact; sa.s1_exact = s1_exact; sa.tau0 = tau0; sa.tau1 = tau1; sa.f1_head = f1_head;
    sa.f1_diso = f1_diso; sa.f2_head = f2_head; sa.f2_exact = f2_exact; sa.f1_off = f1_off;
    sa.out_ids = d_ids; sa.out_dist = d_dist;
    sa.f1_id = f1_id;
    sa.seed_lists = p->seed_lists > 0 ? p->seed_lists : 1;
    sa.list_size_g = ix->list_size_g; sa.s0_id = s0_id; sa.s1_id = s1_id; sa.xout = nullptr;
    sa.store_f1 = ix->dbg_dump_dis;
    sa.sketch = want_sketch; sa.surv_cnt = surv_cnt;
    sa.fuse_topk = ix->fuse_topk_on;
    const bool fuse_topk = mode != 3 && mrq_head_topk_used(sa);

    if (mode == 3) {
        // ---- NOCORR: top-K by dis' over every probed candidate, no bounds, no re-rank
        for (uint32_t *z : {s0_cnt, s1_cnt, f1_cnt, f2_cnt})
            MRQ_CUDA_TRY(cudaMemsetAsync(z, 0, (size_t)nq * 4, st));
        if (timed) MRQ_CUDA_TRY(cudaMemsetAsync(exact_cnt, 0, (size_t)nq * 4, st));
        launch_fill_f64(tau0, nq, INFINITY, st);
        launch_fill_f64(tau1, nq, INFINITY, st);
        if (timed)
            for (int e : {4, 5, 10, 6, 7}) MRQ_CUDA_TRY(cudaEventRecord(ix->ev[e], st));
        StageArgs sx = sa;
        if (sharded) sx.xout = xsend;
        TRY(launch_nocorr_w(W, sx, st));
        if (timed) MRQ_CUDA_TRY(cudaEventRecord(ix->ev[8], st));
    } else {
        // ---- a4: seeds S0 and tau0 (decision T); EXACT mode scans everything
        nvtx.stage("a4 seeds");
        if (mode == 2) {
            launch_fill_f64(tau0, nq, INFINITY, st);
            MRQ_CUDA_TRY(cudaMemsetAsync(s0_cnt, 0, nq * 4, st));
        } else {
            if (sharded) {   // local part of S0 -> all-gather -> global S0, tau0
                StageArgs sx = sa;
                sx.xout = xsend;
                TRY(launch_seed_w(W, sx, st));
                TRY(mrq_allgather(ix, xsend, xrecv, (size_t)nq * Kp * sizeof(XItem), st));
                TRY(launch_xmerge(0, sa, ix->world, ix->rank, xrecv, st));
            } else {
                TRY(launch_seed_w(W, sa, st));
            }
        }
        if (timed) MRQ_CUDA_TRY(cudaEventRecord(ix->ev[4], st));

        // ---- a5: the code scan -> F1
        nvtx.stage("a5 scan");
        {
            LaunchScan a;
            a.nq = nq;
            a.smem = mrq_scan_smem(np, W);
            a.probe = probe; a.np = np; a.npad = ix->npad; a.list_off = ix->list_off; a.list_size = ix->list_size;
            a.codes = ix->codes; a.f1 = ix->f1; a.f2 = ix->f2; a.f3 = ix->f3; a.planes = planes; a.qconst = qconst;
            a.eps_r = eps_r; a.tau0 = tau0; a.isd = isd; a.f1_off = f1_off; a.f1_cnt = f1_cnt; a.f1_pos = f1_pos;
            a.qorder = qorder;
            a.hq = ix->hq; a.hs = ix->hs; a.qsk_b = qsk_b; a.qsk_c = qsk_c; a.qr2 = qr2;
            a.dq = ix->dq; a.surv_cnt = surv_cnt;   // NULL: plain F1 (no fused sketch test)
            if (surv_cnt) a.smem = mrq_scan_smem_sk(np, W, ix->dq);
            a.lm = use_lm ? ix->scan_lm : 0; a.k = k; a.qg = lm_qg;
            a.pairs = lms.pairs; a.loff = lms.loff; a.upre = lms.upre; a.unit_ctr = lms.unit_ctr;
            a.unit_list = lms.unit_list;
            if (use_lm) {   // the list-major scan accumulates the per-query counters atomically
                MRQ_CUDA_TRY(cudaMemsetAsync(f1_cnt, 0, (size_t)nq * 4, st));
                if (surv_cnt) MRQ_CUDA_TRY(cudaMemsetAsync(surv_cnt, 0, (size_t)nq * 4, st));
            }
            if (mode == 2)
                launch_f1_all(probe, nq, np, ix->list_off, ix->list_size, f1_off, f1_cnt, f1_pos, st);
            else
                TRY(launch_scan(W, a, st));
            if (ix->dbg_dump_dis && mode != 2) {
                double *dd, *dl;
                SCR("dbg_dis", double, total, dd);
                SCR("dbg_lb1", double, total, dl);
                launch_scan_dbg(W, a, dd, dl, st);
            }
        }
        if (timed) MRQ_CUDA_TRY(cudaEventRecord(ix->ev[5], st));

        // ---- a6: stage 2 -> F2 (and S1, tau1)
        nvtx.stage("a6 stage 2");
        if (sharded && mode == 0 && tight) {   // local S1 -> all-gather -> global S1, tau1 -> F2
            StageArgs sx = sa;
            sx.xout = xsend;
            TRY(launch_stage2_w(sx, st, timed ? ix->ev[10] : nullptr));
            TRY(mrq_allgather(ix, xsend, xrecv, (size_t)nq * Kp * sizeof(XItem), st));
            TRY(launch_xmerge(1, sa, ix->world, ix->rank, xrecv, st));
            TRY(launch_f2_w(sa, st));
        } else if (fuse_topk) {   // stage 2 + a7 + a8 in one kernel (k_head_topk)
            StageArgs sx = sa;
            if (sharded) sx.xout = xsend;
            TRY(launch_head_topk(sx, st));
            if (timed) MRQ_CUDA_TRY(cudaEventRecord(ix->ev[10], st));
        } else {
            TRY(launch_stage2_w(sa, st, timed ? ix->ev[10] : nullptr));
        }
        if (timed) MRQ_CUDA_TRY(cudaEventRecord(ix->ev[6], st));

        // ---- a7: exact re-rank of F2
        // (a7, the exact re-rank of F2, runs inside the top-K kernel)
        if (timed) MRQ_CUDA_TRY(cudaEventRecord(ix->ev[7], st));

        // ---- a8: per-query top-K
        nvtx.stage("a7+a8 re-rank, top-K");
        if (fuse_topk) {
            // (done by k_head_topk)
        } else if (sharded) {
            StageArgs sx = sa;
            sx.xout = xsend;
            TRY(launch_topk_w(sx, st));
        } else {
            TRY(launch_topk_w(sa, st));
        }
        if (timed) MRQ_CUDA_TRY(cudaEventRecord(ix->ev[8], st));
    }
    // ---- a9: multi-GPU merge (all-gather of the per-rank top-K)
    nvtx.stage("a9 merge");
    if (sharded) {
        TRY(mrq_allgather(ix, xsend, xrecv, (size_t)nq * K * sizeof(XItem), st));
        TRY(launch_xmerge(2, sa, ix->world, ix->rank, xrecv, st));
    }
    if (timed) {
        MRQ_CUDA_TRY(cudaEventRecord(ix->ev[9], st));
        TRY(launch_exact_count(sa, st));   // statistic only, outside the timed stages
    }
    MRQ_CUDA_TRY(cudaGetLastError());

    ix->last_nq = nq;
    ix->last_np = np;
    ix->last_K = K;
    ix->last_Kp = Kp;
    if (timed) {
        MRQ_CUDA_TRY(cudaStreamSynchronize(st));
        float ms[10];
        for (int i = 1; i <= 9; i++) MRQ_CUDA_TRY(cudaEventElapsedTime(&ms[i], ix->ev[i - 1], ix->ev[i]));
        float tot;
        MRQ_CUDA_TRY(cudaEventElapsedTime(&tot, ix->ev[0], ix->ev[9]));
        memset(stats, 0, sizeof *stats);
        stats->ms_total = tot;
        stats->ms_qprep = ms[1];
        stats->ms_probe = ms[2];
        stats->ms_quant = ms[3];
        stats->ms_seed = ms[4];
        stats->ms_scan = ms[5];
        stats->ms_stage2 = ms[6];
        stats->ms_rerank = ms[7];
        stats->ms_topk = ms[8];
        stats->ms_comm = ms[9];
        float mh = 0.f;
        MRQ_CUDA_TRY(cudaEventElapsedTime(&mh, ix->ev[5], ix->ev[10]));
        stats->ms_head = mh;
        stats->ms_sketch = 0.0;   // the sketch test runs inside the scan (ms_scan)
        float mg = 0.f;
        MRQ_CUDA_TRY(cudaEventElapsedTime(&mg, ix->ev[1], ix->ev[11]));
        stats->ms_probe_gemm = mg;
        std::vector<uint32_t> h(nq);
        auto sum32 = [&](const uint32_t *dv) -> uint64_t {
            if (cudaMemcpy(h.data(), dv, nq * 4, cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
            uint64_t s = 0;
            for (auto v : h) s += v;
            return s;
        };
        uint64_t scanned = 0;
        MRQ_CUDA_TRY(cudaMemcpy(&scanned, f1_off + nq, 8, cudaMemcpyDeviceToHost));
        stats->scanned = scanned;
        stats->stage1_pass = sum32(f1_cnt);
        stats->stage2_pass = sum32(f2_cnt);
        stats->exact = sum32(exact_cnt);
        stats->seeds = sum32(s0_cnt) + sum32(s1_cnt);
        stats->sketch_pass = surv_cnt ? sum32(surv_cnt) : stats->stage1_pass;
    }
    return MRQ_OK;
}

static int check_params(const mrq_index *ix, int64_t nq, const mrq_search_params *p)
{
    if (!ix || !p) {
        mrq_set_error("NULL index or params");
        return MRQ_EINVAL;
    }
    if (nq < 0 || p->K < 1 || p->K > MRQ_MAX_K || p->nprobe < 1 || p->nprobe > MRQ_MAX_NPROBE ||
        p->nprobe > ix->k || !(p->eps0 > 0) || !(p->m > 0) || p->mode < 0 || p->mode > 3 ||
        p->tau_schedule < 0 || p->tau_schedule > 1 || p->seed_mult < 1 ||
        (int64_t)p->seed_mult * p->K > MRQ_MAX_SEEDS || !(p->resid_scale > 0) || p->seed_lists < 0) {
        mrq_set_error("InvalidConfig: K=%d nprobe=%d (k=%d) eps0=%g m=%g mode=%d tau=%d seed_mult=%d rscale=%g "
                      "(seed_mult*K <= %d)",
                      p->K, p->nprobe, ix->k, p->eps0, p->m, p->mode, p->tau_schedule, p->seed_mult,
                      p->resid_scale, MRQ_MAX_SEEDS);
        return MRQ_EINVAL;
    }
    if (p->mode != 2 && !supported_W(ix->W)) {
        mrq_set_error("InvalidConfig: mode %d needs d <= 512 and ceil(d/32) in {1,2,3,4,8,16} (d=%d); "
                      "mode EXACT works for any d", p->mode, ix->d);
        return MRQ_EINVAL;
    }
    // the scan stages every probed list's constants and bit-planes in shared memory
    const size_t scan_smem = mrq_scan_smem(std::min(p->nprobe, ix->k), ix->W);
    if (p->mode != 2 && scan_smem > (size_t)ix->smem_optin) {
        mrq_set_error("InvalidConfig: nprobe=%d with d=%d needs %zu B of scan shared memory (device max %d)",
                      p->nprobe, ix->d, scan_smem, ix->smem_optin);
        return MRQ_EINVAL;
    }
    return MRQ_OK;
}

// CUDA-graph replay of repeated searches: a search with the same shapes,
// parameters, buffers and stream as the previous one is captured once (on its
// second occurrence, when every scratch buffer has its final size) and then
// replayed with a single cudaGraphLaunch.  Not used with stats, debug dumps,
// the host all-gather, or when the candidate scratch needs the host-read total.

static bool graph_key_eq(const GraphKey &a, const GraphKey &b) { return memcmp(&a, &b, sizeof a) == 0; }

static int search_dispatch(mrq_index *ix, const float *d_q, int64_t nq, const mrq_search_params *p, int64_t *d_ids,
                           float *d_dist, mrq_stats *stats, cudaStream_t st)
{
    const int np = std::min(p->nprobe, ix->k);
    const uint64_t bound = (uint64_t)nq * ix->h_topsum[np];
    const bool eligible = !stats && !ix->dbg_dump_dis && !ix->host_ag && ix->graphs && st != nullptr &&
                          bound * 48 <= ix->cand_budget;
    if (!eligible) return search_impl(ix, d_q, nq, p, d_ids, d_dist, stats, st);
    GraphKey key;
    memset(&key, 0, sizeof key);
    key.q = d_q;
    key.ids = d_ids;
    key.dist = d_dist;
    key.stream = st;
    key.nq = nq;
    key.p = *p;
    key.gen = ix->scratch_gen;
    GraphKey *cur = (GraphKey *)ix->g_key, *pend = (GraphKey *)ix->g_pending;
    if (ix->gexec && graph_key_eq(*cur, key)) {
        MRQ_CUDA_TRY(cudaGraphLaunch((cudaGraphExec_t)ix->gexec, st));
        return MRQ_OK;
    }
    if (!graph_key_eq(*pend, key)) {   // first occurrence: run, remember
        *pend = key;
        return search_impl(ix, d_q, nq, p, d_ids, d_dist, stats, st);
    }
    // second occurrence: capture, instantiate, launch
    if (ix->gexec) cudaGraphExecDestroy((cudaGraphExec_t)ix->gexec);
    ix->gexec = nullptr;
    cudaGraph_t g = nullptr;
    MRQ_CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
    const int rc = search_impl(ix, d_q, nq, p, d_ids, d_dist, nullptr, st);
    const cudaError_t ce = cudaStreamEndCapture(st, &g);
    cudaGraphExec_t ex = nullptr;
    if (rc != MRQ_OK || ce != cudaSuccess || !g || cudaGraphInstantiate(&ex, g, 0) != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        ix->graphs = 0;   // capture not possible here: plain launches from now on
        return search_impl(ix, d_q, nq, p, d_ids, d_dist, stats, st);
    }
    cudaGraphDestroy(g);
    ix->gexec = ex;
    *cur = key;
    MRQ_CUDA_TRY(cudaGraphLaunch(ex, st));
    return MRQ_OK;
}

extern "C" int mrq_search_batch_device(mrq_index *ix, const float *d_queries, int64_t nq, const mrq_search_params *p,
                                       int64_t *d_out_ids, float *d_out_dist, mrq_stats *stats, void *stream)
{
    TRY(check_params(ix, nq, p));
    if (nq == 0) {
        if (stats) memset(stats, 0, sizeof *stats);
        return MRQ_OK;
    }
    if (!d_queries || !d_out_ids || !d_out_dist) {
        mrq_set_error("NULL buffer");
        return MRQ_EINVAL;
    }
    MRQ_CUDA_TRY(cudaSetDevice(ix->device));
    cudaStream_t st = stream ? (cudaStream_t)stream : ix->stream;
    return mrq_guard([&] { return search_dispatch(ix, d_queries, nq, p, d_out_ids, d_out_dist, stats, st); });
}

static int search_host(mrq_index *ix, const float *queries, int64_t nq, const mrq_search_params *p, int64_t *out_ids,
                       float *out_dist, mrq_stats *stats);

extern "C" int mrq_search_batch(mrq_index *ix, const float *queries, int64_t nq, const mrq_search_params *p,
                                int64_t *out_ids, float *out_dist, mrq_stats *stats)
{
    TRY(check_params(ix, nq, p));
    if (nq == 0) {
        if (stats) memset(stats, 0, sizeof *stats);
        return MRQ_OK;
    }
    if (!queries || !out_ids || !out_dist) {
        mrq_set_error("NULL buffer");
        return MRQ_EINVAL;
    }
    return mrq_guard([&] { return search_host(ix, queries, nq, p, out_ids, out_dist, stats); });
}

static int search_host(mrq_index *ix, const float *queries, int64_t nq, const mrq_search_params *p, int64_t *out_ids,
                       float *out_dist, mrq_stats *stats)
{
    MRQ_CUDA_TRY(cudaSetDevice(ix->device));
    float *dq;
    int64_t *dids;
    float *ddist;
    SCR("in_q", float, nq * ix->D, dq);
    SCR("out_ids", int64_t, nq * p->K, dids);
    SCR("out_dist", float, nq * p->K, ddist);
    MRQ_CUDA_TRY(cudaMemcpyAsync(dq, queries, (size_t)nq * ix->D * 4, cudaMemcpyHostToDevice, ix->stream));
    TRY(search_dispatch(ix, dq, nq, p, dids, ddist, stats, ix->stream));
    MRQ_CUDA_TRY(cudaMemcpyAsync(out_ids, dids, (size_t)nq * p->K * 8, cudaMemcpyDeviceToHost, ix->stream));
    MRQ_CUDA_TRY(cudaMemcpyAsync(out_dist, ddist, (size_t)nq * p->K * 4, cudaMemcpyDeviceToHost, ix->stream));
    MRQ_CUDA_TRY(cudaStreamSynchronize(ix->stream));
    return MRQ_OK;
}

// ------------------------------------------------------------- debug fetch
static int debug_fetch(mrq_index *ix, const char *name, void *dst, size_t dst_bytes, size_t *bytes_needed);
extern "C" int mrq_debug_fetch(mrq_index *ix, const char *name, void *dst, size_t dst_bytes, size_t *bytes_needed)
{
    return mrq_guard([&] { return debug_fetch(ix, name, dst, dst_bytes, bytes_needed); });
}

static int debug_fetch(mrq_index *ix, const char *name, void *dst, size_t dst_bytes, size_t *bytes_needed)
{
    if (!ix || !name) {
        mrq_set_error("NULL index or name");
        return MRQ_EINVAL;
    }
    const int64_t npad = ix->npad, nq = ix->last_nq;
    const int k = ix->k, d = ix->d, D = ix->D, W = ix->W, np = ix->last_np, Kp = ix->last_Kp;
    const void *src = nullptr;
    size_t bytes = 0;
    std::string nm(name);
    struct E {
        const char *n;
        const void *p;
        size_t b;
    } fixed[] = {
        {"list_off", ix->list_off, (size_t)(k + 1) * 4}, {"list_size", ix->list_size, (size_t)k * 4},
        {"ids", ix->ids, (size_t)npad * 4},              {"codes", ix->codes, (size_t)W * npad * 4},
        {"f1", ix->f1, (size_t)npad * 4},                {"f2", ix->f2, (size_t)npad * 4},
        {"f3", ix->f3, (size_t)npad * 4},                {"xr2", ix->xr2, (size_t)npad * 4},
        {"heads", ix->heads, (size_t)npad * d * 4},      {"tails", ix->tails, (size_t)npad * std::max(D - d, 0) * 4},
        {"Rc", ix->Rc, (size_t)k * d * 8},
        {"hq", ix->hq, (size_t)npad * ix->dq},          {"hs", ix->hs, (size_t)npad * 16},
    };
    for (auto &e : fixed)
        if (nm == e.n) {
            src = e.p;
            bytes = e.b;
        }
    if (!src) {
        struct S {
            const char *n;
            size_t b;
        } per[] = {
            {"qp", (size_t)nq * D * 8},        {"qr2", (size_t)nq * 8},
            {"eps_r", (size_t)nq * 8},         {"tau0", (size_t)nq * 8},
            {"tau1", (size_t)nq * 8},          {"r0", (size_t)nq * d * 8},
            {"probe", (size_t)nq * np * 4},    {"probe_qn2", (size_t)nq * np * 8},
            {"planes", (size_t)nq * np * MRQ_BQ * W * 4}, {"qconst", (size_t)nq * np * 8 * 8},
            {"f1_off", (size_t)(nq + 1) * 8},  {"f1_cnt", (size_t)nq * 4},
            {"f2_cnt", (size_t)nq * 4},        {"s0_cnt", (size_t)nq * 4},
            {"s1_cnt", (size_t)nq * 4},        {"exact_cnt", (size_t)nq * 4},
            {"s0_pos", (size_t)nq * Kp * 4},   {"s0_exact", (size_t)nq * Kp * 8},
            {"s1_pos", (size_t)nq * Kp * 4},   {"s1_exact", (size_t)nq * Kp * 8},
            {"s0_id", (size_t)nq * Kp * 4},    {"s1_id", (size_t)nq * Kp * 4},
            {"f1_pos", (size_t)ix->last_total * 4}, {"f1_head", (size_t)ix->last_total * 8},
            {"f1_diso", (size_t)ix->last_total * 8}, {"f2_pos", (size_t)ix->last_total * 4},
            {"f2_head", (size_t)ix->last_total * 8}, {"f2_exact", (size_t)ix->last_total * 8},
            {"fallback", 4}, {"approx", (size_t)nq * k * 4}, {"probe_ncand", (size_t)nq * 4},
            {"dbg_dis", (size_t)ix->last_total * 8}, {"dbg_lb1", (size_t)ix->last_total * 8},
            {"surv_cnt", (size_t)nq * 4},
            {"qorder", (size_t)nq * 4},        {"qkey", (size_t)nq * 2},
            {"probe_ccnt", ix->scratch.count("probe_ccnt") ? ix->scratch["probe_ccnt"].bytes : 0},
        };
        for (auto &e : per)
            if (nm == e.n) {
                auto it = ix->scratch.find(nm);
                if (it == ix->scratch.end()) break;
                src = it->second.p;
                bytes = e.b;
            }
    }
    if (!src) {
        mrq_set_error("unknown or unavailable debug buffer '%s'", name);
        return MRQ_EINVAL;
    }
    if (bytes_needed) *bytes_needed = bytes;
    if (!dst) return MRQ_OK;
    if (dst_bytes < bytes) {
        mrq_set_error("debug buffer '%s' needs %zu bytes", name, bytes);
        return MRQ_EINVAL;
    }
    MRQ_CUDA_TRY(cudaSetDevice(ix->device));
    MRQ_CUDA_TRY(cudaStreamSynchronize(ix->stream));
    MRQ_CUDA_TRY(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
    return MRQ_OK;
}

extern "C" int mrq_debug_set(mrq_index *ix, const char *name, int64_t value)
{
    if (!ix || !name) {
        mrq_set_error("NULL index or name");
        return MRQ_EINVAL;
    }
    // a switch changes what search_impl launches: drop the captured graph
    if (ix->gexec) cudaGraphExecDestroy((cudaGraphExec_t)ix->gexec);
    ix->gexec = nullptr;
    memset(ix->g_key, 0, sizeof(GraphKey));
    memset(ix->g_pending, 0, sizeof(GraphKey));
    if (std::string(name) == "qorder") {           // query processing order: 0 as given, 1 key from the projection,
                                                   // 2 (default) key of the nearest probed list
        ix->qorder_on = (int)value;
        return MRQ_OK;
    }
    if (std::string(name) == "dump_dis") {
        ix->dbg_dump_dis = (int)value;
        return MRQ_OK;
    }
    if (std::string(name) == "force_exchange") {   // world 1 runs the sharded (exchange + merge) path
        ix->force_exchange = (int)value;
        return MRQ_OK;
    }
    if (std::string(name) == "cuda_core_probe") {  // probe screen on CUDA cores instead of tcgen05
        ix->force_cuda_core_probe = (int)value;
        return MRQ_OK;
    }
    if (std::string(name) == "graphs") {           // CUDA-graph replay of repeated searches (default 1)
        ix->graphs = (int)value;
        return MRQ_OK;
    }
    if (std::string(name) == "front_shard") {      // world > 1: query-sharded a1-a3 + all-gather (default 1)
        ix->front_shard = (int)value;
        return MRQ_OK;
    }
    if (std::string(name) == "sketch") {           // head-sketch pre-pass of the stage-2 gather (default 1)
        ix->sketch_on = (int)value;
        return MRQ_OK;
    }
    if (std::string(name) == "fuse_topk") {   // stage 2 + re-rank + top-K in one kernel (default 1)
        ix->fuse_topk_on = value ? 1 : 0;
        return MRQ_OK;
    }
    if (std::string(name) == "scan_lm") {   // list-major code scan: 0 off, 1 CUDA-core, 2 tensor-core S (d <= 128)
        ix->scan_lm = value < 0 ? 0 : (value > 2 ? 2 : (int)value);
        return MRQ_OK;
    }
    if (std::string(name) == "scan_lm_qg") {   // pairs of a list per list-major work unit (default 16)
        if (value < 1 || value > 4096) {
            mrq_set_error("scan_lm_qg must be in [1, 4096]");
            return MRQ_EINVAL;
        }
        ix->lm_qg = (int)value;
        return MRQ_OK;
    }
    if (std::string(name) == "probe_share") {   // the fused probe's parts share their bounds (default 1)
        ix->probe_share = value ? 1 : 0;
        return MRQ_OK;
    }
    if (std::string(name) == "probe_capp") {       // per-part candidate buffer of the fused probe (default 256)
        if (value < 1 || value > 4096) {
            mrq_set_error("probe_capp must be in [1, 4096]");
            return MRQ_EINVAL;
        }
        ix->probe_capp = (int)value;
        return MRQ_OK;
    }
    if (std::string(name) == "cand_budget_mb") {   // candidate scratch sized by the host bound below this (8192)
        ix->cand_budget = (uint64_t)std::max<int64_t>(value, 0) << 20;
        return MRQ_OK;
    }
    if (std::string(name) == "probe_unfused") {    // screen to HBM + separate selection kernel
        ix->force_probe_unfused = (int)value;
        return MRQ_OK;
    }
    mrq_set_error("unknown debug switch '%s'", name);
    return MRQ_EINVAL;
}

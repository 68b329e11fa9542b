// mrq_comm.cu -- list sharding across ranks and the all-gather exchanges of
// the multi-GPU path.
//
// NCCL is resolved at run time (dlopen "libnccl.so.2", the library torch
// ships), so libmrq loads on hosts without NCCL; a world > 1 index fails
// loudly (MRQ_ENCCL) if NCCL cannot be loaded.
#include <dlfcn.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <numeric>

#include "mrq_comm.cuh"

#if MRQ_HAVE_NCCL
#include <nccl.h>
#endif

// Greedy longest-processing-time assignment of lists to ranks: lists by size
// descending (ties by id), each to the currently least-loaded rank (ties by
// rank).  Deterministic, so every rank computes the same map.
void mrq_shard_lists(const std::vector<uint32_t> &sizes, int world, std::vector<uint32_t> &owner)
{
    const int k = (int)sizes.size();
    std::vector<int> order(k);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return sizes[a] > sizes[b]; });
    std::vector<uint64_t> load(world, 0);
    owner.assign(k, 0);
    for (int c : order) {
        int best = 0;
        for (int r = 1; r < world; r++)
            if (load[r] < load[best]) best = r;
        owner[c] = (uint32_t)best;
        load[best] += sizes[c];
    }
}

extern "C" int mrq_shard_plan(const uint32_t *sizes, int32_t k, int32_t world, uint32_t *owner)
{
    if (!sizes || !owner || k < 1 || world < 1) {
        mrq_set_error("InvalidConfig: mrq_shard_plan needs sizes, owner, k >= 1, world >= 1");
        return MRQ_EINVAL;
    }
    return mrq_guard([&] {
        std::vector<uint32_t> s(sizes, sizes + k), o;
        mrq_shard_lists(s, world, o);
        memcpy(owner, o.data(), (size_t)k * 4);
        return (int)MRQ_OK;
    });
}

#if MRQ_HAVE_NCCL
namespace {
struct NcclApi {
    bool ok = false;
    char err[256] = "";
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*commAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char *(*getErrorString)(ncclResult_t) = nullptr;
};

NcclApi &nccl()
{
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
#ifdef MRQ_NCCL_LIB
        if (!h) h = dlopen(MRQ_NCCL_LIB, RTLD_NOW | RTLD_GLOBAL);
#endif
        if (!h) {
            snprintf(api.err, sizeof api.err, "cannot load libnccl.so.2: %s", dlerror());
            return;
        }
        api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
        api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
        api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
        api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
        api.getErrorString = (decltype(api.getErrorString))dlsym(h, "ncclGetErrorString");
        api.commAbort = (decltype(api.commAbort))dlsym(h, "ncclCommAbort");
        api.groupStart = (decltype(api.groupStart))dlsym(h, "ncclGroupStart");
        api.groupEnd = (decltype(api.groupEnd))dlsym(h, "ncclGroupEnd");
        api.ok = api.getUniqueId && api.commInitRank && api.allGather && api.commDestroy && api.getErrorString &&
                 api.commAbort && api.groupStart && api.groupEnd;
        if (!api.ok) snprintf(api.err, sizeof api.err, "libnccl.so.2 lacks a required symbol");
    });
    return api;
}
}  // namespace
#endif

extern "C" int mrq_nccl_unique_id(void *out, size_t bytes)
{
    if (!out || bytes < 128) {
        mrq_set_error("InvalidConfig: mrq_nccl_unique_id needs a 128-byte buffer");
        return MRQ_EINVAL;
    }
#if MRQ_HAVE_NCCL
    NcclApi &a = nccl();
    if (!a.ok) {
        mrq_set_error("%s", a.err);
        return MRQ_ENCCL;
    }
    ncclUniqueId id;
    ncclResult_t r = a.getUniqueId(&id);
    if (r != ncclSuccess) {
        mrq_set_error("ncclGetUniqueId: %s", a.getErrorString(r));
        return MRQ_ENCCL;
    }
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
    memcpy(out, &id, 128);
    return MRQ_OK;
#else
    mrq_set_error("libmrq was built without nccl.h");
    return MRQ_ENCCL;
#endif
}

int mrq_comm_init(mrq_index *ix, const mrq_dist_cfg *dist)
{
    if (dist->nccl_unique_id) {
#if MRQ_HAVE_NCCL
        NcclApi &a = nccl();
        if (!a.ok) {
            mrq_set_error("%s", a.err);
            return MRQ_ENCCL;
        }
        ncclUniqueId id;
        memcpy(&id, dist->nccl_unique_id, sizeof id);
        ncclComm_t comm = nullptr;
        ncclResult_t r = a.commInitRank(&comm, ix->world, id, ix->rank);
        if (r != ncclSuccess) {
            mrq_set_error("ncclCommInitRank(world=%d, rank=%d): %s", ix->world, ix->rank, a.getErrorString(r));
            return MRQ_ENCCL;
        }
        ix->nccl_comm = comm;
        return MRQ_OK;
#else
        mrq_set_error("libmrq was built without nccl.h");
        return MRQ_ENCCL;
#endif
    }
    if (dist->host_allgather) {
        ix->host_ag = dist->host_allgather;
        ix->host_ctx = dist->host_ctx;
        return MRQ_OK;
    }
    mrq_set_error("InvalidConfig: world=%d needs nccl_unique_id or host_allgather", ix->world);
    return MRQ_EINVAL;
}

void mrq_comm_free(mrq_index *ix)
{
#if MRQ_HAVE_NCCL
    if (ix->nccl_comm) nccl().commDestroy((ncclComm_t)ix->nccl_comm);
#endif
    ix->nccl_comm = nullptr;
    if (ix->xhost) cudaFreeHost(ix->xhost);
    ix->xhost = nullptr;
    ix->xhost_bytes = 0;
}

int mrq_allgather(mrq_index *ix, const void *send, void *recv, size_t bytes, cudaStream_t st)
{
#if MRQ_HAVE_NCCL
    if (ix->nccl_comm) {
        NcclApi &a = nccl();
        ncclResult_t r = a.allGather(send, recv, bytes, ncclUint8, (ncclComm_t)ix->nccl_comm, st);
        if (r != ncclSuccess) {
            mrq_set_error("ncclAllGather(%zu B): %s", bytes, a.getErrorString(r));
            mrq_comm_fail(ix);
            return MRQ_ENCCL;
        }
        return MRQ_OK;
    }
#endif
    if (ix->comm_failed) {
        mrq_set_error("the NCCL communicator of this index was aborted after a failure");
        return MRQ_ENCCL;
    }
    if (ix->world == 1) {
        if (send != recv) MRQ_CUDA_TRY(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, st));
        return MRQ_OK;
    }
    if (!ix->host_ag) {
        mrq_set_error("no exchange configured for world=%d", ix->world);
        return MRQ_ENCCL;
    }
    const size_t need = bytes * (size_t)(ix->world + 1);
    MRQ_CUDA_TRY(cudaStreamSynchronize(st));
    if (ix->xhost_bytes < need) {
        if (ix->xhost) cudaFreeHost(ix->xhost);
        ix->xhost = nullptr;
        ix->xhost_bytes = 0;
        MRQ_CUDA_TRY(cudaMallocHost(&ix->xhost, need));
        ix->xhost_bytes = need;
    }
    char *h = (char *)ix->xhost;
    MRQ_CUDA_TRY(cudaMemcpyAsync(h, send, bytes, cudaMemcpyDeviceToHost, st));
    MRQ_CUDA_TRY(cudaStreamSynchronize(st));
    if (ix->host_ag(h, h + bytes, bytes, ix->host_ctx) != 0) {
        mrq_set_error("host all-gather callback failed");
        return MRQ_ENCCL;
    }
    MRQ_CUDA_TRY(cudaMemcpyAsync(recv, h + bytes, bytes * (size_t)ix->world, cudaMemcpyHostToDevice, st));
    return MRQ_OK;
}

// Several all-gathers at once (the sharded front end's per-query sections):
// one NCCL group (a single fused launch), else one host exchange per section.
int mrq_allgather_group(mrq_index *ix, int n, const void *const *send, void *const *recv, const size_t *bytes,
                        cudaStream_t st)
{
#if MRQ_HAVE_NCCL
    if (ix->nccl_comm) {
        NcclApi &a = nccl();
        ncclResult_t r = a.groupStart();
        for (int i = 0; i < n && r == ncclSuccess; i++)
            r = a.allGather(send[i], recv[i], bytes[i], ncclUint8, (ncclComm_t)ix->nccl_comm, st);
        const ncclResult_t r2 = a.groupEnd();
        if (r == ncclSuccess) r = r2;
        if (r != ncclSuccess) {
            mrq_set_error("ncclAllGather group (%d sections): %s", n, a.getErrorString(r));
            mrq_comm_fail(ix);
            return MRQ_ENCCL;
        }
        return MRQ_OK;
    }
#endif
    for (int i = 0; i < n; i++) {
        const int rc = mrq_allgather(ix, send[i], recv[i], bytes[i], st);
        if (rc != MRQ_OK) return rc;
    }
    return MRQ_OK;
}

// A failed collective leaves the communicator unusable (and its peers
// possibly blocked): abort it instead of a destroy that could hang, so every
// later call on this index fails fast with MRQ_ENCCL.
void mrq_comm_fail(mrq_index *ix)
{
#if MRQ_HAVE_NCCL
    if (ix->nccl_comm) {
        nccl().commAbort((ncclComm_t)ix->nccl_comm);
        ix->nccl_comm = nullptr;
        ix->comm_failed = 1;
    }
#endif
}

/*
 * mrq.h -- C ABI of libmrq, the B200-native batched IVF-MRQ query path.
 *
 * MRQ = Minimized Residual Quantization, arXiv 2411.06158 (citations "P:N" are
 * lines of its LaTeX source PAPER.md).  The library implements the paper's
 * query process (Algorithm 2) for a batch of queries against an
 * IVF index whose build-time artefacts (Algorithm 1 L1-L6: PCA
 * matrix, eigenvalues, IVF centroids and assignment, plus the quantizer's
 * random rotation P_r) come from a build file.  Encoding (Alg.1 L3-L8)
 * runs on the GPU at load time.
 *
 * All functions return 0 (MRQ_OK) on success or a negative mrq_err; the
 * message of the last failure on the calling thread is mrq_last_error().
 * There is no CPU fallback: a missing GPU or a CUDA failure is an error.
 *
 * Numeric contract: every quantity that
 * decides a bit, a level, a flag or an ordering is computed in fp64 with
 * left-to-right sums and no fused multiply-add, so codes, bit-planes, flags
 * and returned ids are bit-identical to the fp64 oracle (oracle/).
 */
#ifndef MRQ_H
#define MRQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mrq_index mrq_index;  /* opaque; owns all device memory of one rank */

typedef enum {
    MRQ_OK = 0,
    MRQ_EINVAL = -1,      /* InvalidConfig: bad K, nprobe, eps0, m, mode, sizes, NULL;
                             n != the build file's N                      */
    MRQ_EDIM = -2,        /* DimensionMismatch: D or d differ from the build file        */
    MRQ_EFORMAT = -3,     /* FormatError: truncated/corrupt build file (message: offset) */
    MRQ_EVERSION = -4,    /* VersionMismatch: bad magic or version                       */
    MRQ_EDEGENERATE = -5, /* DegenerateData                                              */
    MRQ_ECUDA = -6,       /* CUDA runtime failure (no device, launch error, ...)         */
    MRQ_ENOMEM = -7,      /* device or host allocation failed                            */
    MRQ_ENCCL = -8,       /* NCCL failure (multi-GPU)                                    */
    MRQ_EIO = -9          /* cannot open/read the build file                             */
} mrq_err;

/* Host all-gather used in place of NCCL (tests, virtual ranks): gathers
 * `bytes` from every rank's `send` into `recv` (world * bytes, rank-major).
 * Returns 0 on success.  Called from the thread that called the search. */
typedef int (*mrq_allgather_fn)(const void *send, void *recv, size_t bytes, void *ctx);

/* Multi-GPU placement.  NULL, or world == 1, means
 * one GPU (the current device when device < 0).  With world > 1 every rank
 * calls every function with identical arguments; IVF lists are sharded across
 * ranks (mrq_shard_plan) and the decision-T seed sets and the per-rank top-K
 * are exchanged with an all-gather: NCCL when nccl_unique_id (128 bytes from
 * mrq_nccl_unique_id, the same on all ranks) is non-NULL, else the host
 * callback host_allgather(ctx).  Results are identical for every world size. */
typedef struct {
    int32_t rank, world, device;
    const void *nccl_unique_id;
    mrq_allgather_fn host_allgather;
    void *host_ctx;
} mrq_dist_cfg;

/* Search parameters (Alg.2 inputs N^probe, eps0, m). */
typedef struct {
    int32_t K;            /* results per query, 1 <= K <= 1024                               */
    int32_t nprobe;       /* probed lists, 1 <= nprobe <= min(k, 1024); the scan keeps every
                             probed list's bit-planes in shared memory, so nprobe * (52 +
                             16 ceil(d/32)) + 4 bytes must fit the device (d = 512: nprobe
                             <= ~750), else MRQ_EINVAL                                       */
    double eps0;          /* Eq.5 confidence parameter, > 0; default 1.9              */
    double m;             /* Chebyshev multiplier (Eq.7), > 0; default 4.0             */
    int32_t mode;         /* 0 FULL (IVF-MRQ+: stage 1 + stage 2), 1 STAGE1_ONLY (IVF-MRQ),
                             2 EXACT (exact distance of every probed candidate),
                             3 NOCORR (no correction, no re-rank: the K smallest (dis', id)
                               of every probed candidate; the distance returned is dis',
                               Eq.4 P:245-250 -- SPEC S:425)                                  */
    int32_t tau_schedule; /* 0 TIGHT, 1 LOOSE (DESIGN.md decision T)                          */
    int32_t seed_mult;    /* K' = seed_mult * K seeds (>= 1, seed_mult * K <= 4096; default 2)  */
    double resid_scale;   /* eps_r = (resid_scale * m) * sigma; 2 = distance domain (default) */
    int32_t seed_lists;   /* decision T seed pool: the first probed lists until they hold >= K'
                             candidates AND at least seed_lists lists (>= 1; 0 means 1)      */
} mrq_search_params;

/* Per-call counters (summed over queries; at world > 1 over this rank's lists
 * only -- "seeds" counts the owned members of the global S0/S1) and per-stage device milliseconds
 * (CUDA events on the library's stream; filled only when stats != NULL, which
 * makes the call synchronous). */
typedef struct {
    uint64_t scanned;      /* candidates whose code was scanned                 */
    uint64_t stage1_pass;  /* |F1|: LB1 < tau0                                  */
    uint64_t stage2_pass;  /* |F2|: dis_o' - eps_r < tau1                       */
    uint64_t exact;        /* distinct exact distances computed (F2 u S0 u S1)  */
    uint64_t seeds;        /* |S0| + |S1|                                        */
    double ms_total, ms_qprep, ms_probe, ms_quant, ms_seed, ms_scan, ms_stage2, ms_rerank, ms_topk, ms_comm;
    double ms_head;        /* the stage-2 head gather alone (part of ms_stage2)  */
    double ms_probe_gemm;  /* the probe screen GEMM alone (part of ms_probe)     */
    double ms_sketch;      /* the head-sketch pre-pass alone (part of ms_head; 0 if not run) */
    uint64_t sketch_pass;  /* F1 entries the head sketch could not prune (= stage1_pass
                              when the pre-pass does not run): the fp32 head rows read   */
} mrq_stats;

/*
 * Load an index.  build_file: path of an MRQBLD01 file (format below).
 * base: HOST pointer, row-major n x D float32, borrowed for the call (copied
 * to the device).  D and d must equal the file's; n must equal its N.
 * Encodes every vector on the GPU (Alg.1 L3-L8): PCA rotation, head/tail
 * split, centring on the own centroid, sign code under P_r, stored factors.
 * On success *out owns the device memory until mrq_free.
 * Errors (checked in this order, before any device work):
 *   MRQ_EINVAL  NULL argument, d < 2 or d > D, unknown flags;
 *   MRQ_EIO     the file cannot be opened or read;
 *   MRQ_EVERSION  bad magic or version;
 *   MRQ_EFORMAT header values out of range (message names the offset);
 *   MRQ_EDIM    D or d differ from the file's;  MRQ_EINVAL  n != the file's N;
 *   MRQ_EFORMAT truncated payload, bad end marker, assignment >= k;
 * then MRQ_ECUDA (no device, launch failure), MRQ_ENOMEM, MRQ_ENCCL.
 */
int mrq_index_load(const char *build_file, const float *base, int64_t n, int32_t D, int32_t d,
                   const mrq_dist_cfg *dist, mrq_index **out);

/*
 * mrq_index_load with flags.  MRQ_LOAD_TAILS_HOST: the fp32 tail rows
 * x_p[d:D] (read only by the exact re-rank of the few surviving candidates,
 * Alg.2 L14 P:316) stay in pinned, device-mapped HOST memory instead of HBM --
 * the memory-limited ("disk-based") setting of P:296 / SURVEY NEXT-4; codes,
 * factors and heads stay in HBM.  Results are identical; tails are read over
 * the host link.  Errors as mrq_index_load; MRQ_EINVAL for unknown flags.
 */
#define MRQ_LOAD_TAILS_HOST 1u
int mrq_index_load_ex(const char *build_file, const float *base, int64_t n, int32_t D, int32_t d,
                      const mrq_dist_cfg *dist, uint32_t flags, mrq_index **out);

/*
 * Batched search with HOST buffers: queries row-major nq x D float32
 * (borrowed); out_ids (nq x K int64) and out_dist (nq x K float32) are
 * caller-owned.  Row i of the outputs belongs to query i; within a row the
 * results are ascending (distance, id); distance = exact squared L2 in the
 * PCA-rotated space rounded to float32.  Fewer than K
 * candidates: the tail is padded with id -1, distance +inf.  Synchronous.
 * nq = 0 is valid and returns immediately.
 */
int mrq_search_batch(mrq_index *idx, const float *queries, int64_t nq, const mrq_search_params *p,
                     int64_t *out_ids, float *out_dist, mrq_stats *stats);

/*
 * Same with DEVICE buffers (queries, out_ids, out_dist in device memory of
 * the index's GPU) on `stream` (a cudaStream_t; 0 = the library's stream).
 * Asynchronous unless stats != NULL.  Scratch is owned by the index and grows
 * on demand (growing synchronizes once).
 */
int mrq_search_batch_device(mrq_index *idx, const float *d_queries, int64_t nq, const mrq_search_params *p,
                            int64_t *d_out_ids, float *d_out_dist, mrq_stats *stats, void *stream);

/*
 * Multi-GPU bootstrap: writes a fresh 128-byte NCCL unique id to out (rank 0
 * calls it and broadcasts the bytes).  NCCL is loaded at run time
 * (libnccl.so.2); errors: MRQ_EINVAL (out NULL or bytes < 128), MRQ_ENCCL.
 */
int mrq_nccl_unique_id(void *out, size_t bytes);

/*
 * The list -> rank plan used by mrq_index_load at world > 1 (host only, no
 * GPU needed): greedy longest-processing-time on list size -- lists by size
 * descending (ties by list id) each go to the least-loaded rank (ties by
 * rank).  sizes: host u32[k]; owner: host u32[k] written with ranks in
 * [0, world).  Errors: MRQ_EINVAL (NULL, k < 1, world < 1).
 */
int mrq_shard_plan(const uint32_t *sizes, int32_t k, int32_t world, uint32_t *owner);

/*
 * GPU index build (Algorithm 1 L1-L6, plus the
 * quantizer rotation P_r): PCA of a strided sample of <= pca_sample
 * rows, heads x_d = P[0:d](x - mu), IVF* k-means on a strided sample of
 * <= km_sample_per_k * k heads (<= km_iters Lloyd iterations), final
 * assignment of all n, Haar rotation from `seed`; written to out_path as an
 * MRQBLD01 build file (format below) that mrq_index_load reads.
 * base: HOST n x D float32 (borrowed); base_sha256_hex: the 64-character hex
 * SHA-256 of the base bytes to record in the header (NULL: zeros).  Same
 * algorithm as the oracle's build, not the same bits (strided samples, other
 * solvers): the contract is recall-equivalence.  times_ms (nullable, 4
 * doubles): PCA, k-means, final assignment, total.
 * Errors: MRQ_EINVAL, MRQ_EDEGENERATE (zero variance), MRQ_ENOMEM, MRQ_ECUDA,
 * MRQ_EIO (cannot write).
 */
typedef struct {
    int32_t k;               /* IVF clusters                          */
    int32_t pca_sample;      /* PCA sample rows (e.g. 100000)         */
    int32_t km_sample_per_k; /* k-means sample = this x k rows (64)   */
    int32_t km_iters;        /* Lloyd iterations (25)                 */
    uint64_t seed;           /* P_r seed (7)                          */
} mrq_build_params;
int mrq_build_gpu(const float *base, int64_t n, int32_t D, int32_t d, const mrq_build_params *bp,
                  const char *base_sha256_hex, int32_t device, const char *out_path, double *times_ms);

/* Free the index (NULL-safe): device memory, streams, NCCL communicator. */
void mrq_free(mrq_index *idx);

/* Thread-local message of the last error (never NULL). */
const char *mrq_last_error(void);

/* Index facts: n, D, d, k, W (code words), npad (list slots), local lists. */
int mrq_index_info(const mrq_index *idx, int64_t *n, int32_t *D, int32_t *d, int32_t *k, int64_t *npad);

/*
 * Test hook: copy the named internal device buffer of the index or of the
 * LAST search into host memory.  *bytes_needed receives its size; with
 * dst == NULL only the size is reported.  Names and layouts (DESIGN.md
 * "HBM layout"): "list_off" u32[k+1] slot offsets, "list_size" u32[k],
 * "ids" u32[npad], "codes" u32[W][npad], "f1" "f2" "f3" "xr2" f32[npad],
 * "heads" f32[npad][d], "tails" f32[npad][D-d], "Rc" f64[k][d], and per
 * search: "qp" f64[nq][D], "qr2" "eps_r" "tau0" "tau1" f64[nq],
 * "probe" u32[nq][np], "probe_qn2" f64[nq][np], "planes" u32[nq][np][4][W],
 * "qconst" f64[nq][np][8], "f1_off" u64[nq], "f1_cnt" u32[nq], "f1_pos" u32[..],
 * "f1_diso" f64[..], "f2_cnt" u32[nq], "f2_pos" u32[..], "f2_exact" f64[..],
 * "s0_cnt" u32[nq], "s0_pos" u32[nq][Kp], "s0_id" u32[nq][Kp],
 * "s0_exact" f64[nq][Kp], "s1_cnt", "s1_pos", "s1_id", "s1_exact".
 * Errors: MRQ_EINVAL (unknown name, dst too small), MRQ_ECUDA.
 */
int mrq_debug_fetch(mrq_index *idx, const char *name, void *dst, size_t dst_bytes, size_t *bytes_needed);

/*
 * Test hook: set a debug switch of the index.  "dump_dis" = 1 makes every
 * later search also write dis' and LB1 of every scanned candidate (debug
 * buffers "dbg_dis", "dbg_lb1" f64, per query at f1_off[q] in probe order,
 * then slot order).  "force_exchange" = 1 makes a world-1 index run the
 * multi-rank path (exchange buffers, device-copy all-gather, k_xmerge).
 * "cuda_core_probe" = 1 screens the probe on CUDA cores (fp32) instead of
 * the tcgen05 tf32 GEMM (the exact fp64 selection is the same).
 * "probe_unfused" = 1 writes the screen to HBM and selects in a separate
 * kernel.  "graphs" = 0 disables the CUDA-graph replay of repeated searches
 * (also: environment MRQ_NO_GRAPHS).  "probe_capp" = n (1..4096, default
 * 256) sizes the fused probe's per-part candidate buffer (a small value
 * forces its overflow path: every centroid rescored).  "cand_budget_mb" = n
 * (default 8192): candidate scratch above this is sized by the exact total
 * read back from the device (one sync) instead of the host bound.
 * "qorder" = 0 disables the list-locality query order.
 * Errors: MRQ_EINVAL (unknown name, value out of range).
 */
int mrq_debug_set(mrq_index *idx, const char *name, int64_t value);

/*
 * Build file MRQBLD01 (little-endian), written by oracle/build.py:
 *   char magic[8] "MRQBLD01"; u32 version (=1); u32 D; u32 d; u32 k; u64 N;
 *   u64 flags (=0); char base_sha256_hex[64];
 *   f64 mu[D]; f64 P[D*D] (row i = i-th principal axis, eigenvalue
 *   descending); f64 lambda[D]; f64 R[d*d] (y = R t); f64 centroids[k*d];
 *   u32 assign[N]; char end[8] "MRQEND01".
 */

#ifdef __cplusplus
}
#endif
#endif /* MRQ_H */

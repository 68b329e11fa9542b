"""ctypes binding of libmrq with the C ABI's names (include/mrq.h).

Argument marshalling only.  Host arrays are numpy; device arrays are torch
CUDA tensors (PyTorch supplies device memory and streams: plumbing).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# MRQ_LIB_VARIANT=name loads libmrq_<name>.so built next to it (A/B timing of
# compile-time variants, scripts/variant.sh); default: libmrq.so
LIB_PATH = os.path.join(HERE, "libmrq%s.so" % (("_" + os.environ["MRQ_LIB_VARIANT"]) if os.environ.get("MRQ_LIB_VARIANT")
                                                 else ""))

MRQ_MODES = {"FULL": 0, "STAGE1_ONLY": 1, "EXACT": 2, "NOCORR": 3}
ERRORS = {-1: "EINVAL", -2: "EDIM", -3: "EFORMAT", -4: "EVERSION", -5: "EDEGENERATE", -6: "ECUDA",
          -7: "ENOMEM", -8: "ENCCL", -9: "EIO"}


class MRQError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("%s (%d): %s" % (ERRORS.get(code, "?"), code, msg))
        self.code = code


ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


class DistCfg(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("device", C.c_int32), ("nccl_unique_id", C.c_void_p),
                ("host_allgather", ALLGATHER_FN), ("host_ctx", C.c_void_p)]


class SearchParams(C.Structure):
    _fields_ = [("K", C.c_int32), ("nprobe", C.c_int32), ("eps0", C.c_double), ("m", C.c_double),
                ("mode", C.c_int32), ("tau_schedule", C.c_int32), ("seed_mult", C.c_int32),
                ("resid_scale", C.c_double), ("seed_lists", C.c_int32)]

    @classmethod
    def make(cls, K=10, nprobe=16, eps0=1.9, m=4.0, mode="FULL", tau_schedule="TIGHT", seed_mult=2,
             resid_scale=2.0, seed_lists=1):
        return cls(K, nprobe, eps0, m, MRQ_MODES[mode] if isinstance(mode, str) else mode,
                   0 if tau_schedule in ("TIGHT", 0) else 1, seed_mult, resid_scale, seed_lists)


class Stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("scanned", "stage1_pass", "stage2_pass", "exact", "seeds")] + \
               [(n, C.c_double) for n in ("ms_total", "ms_qprep", "ms_probe", "ms_quant", "ms_seed", "ms_scan",
                                          "ms_stage2", "ms_rerank", "ms_topk", "ms_comm", "ms_head",
                                          "ms_probe_gemm", "ms_sketch")] + [("sketch_pass", C.c_uint64)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


_lib = None


def lib():
    """Load libmrq.so; fails loudly when the CUDA extension is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libmrq.so not built (run __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        L.mrq_last_error.restype = C.c_char_p
        for f in ("mrq_index_load", "mrq_search_batch", "mrq_search_batch_device", "mrq_debug_fetch",
                  "mrq_index_info"):
            getattr(L, f).restype = C.c_int
        L.mrq_index_load.argtypes = [C.c_char_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p,
                                     C.POINTER(C.c_void_p)]
        L.mrq_index_load_ex.restype = C.c_int
        L.mrq_index_load_ex.argtypes = [C.c_char_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p,
                                        C.c_uint32, C.POINTER(C.c_void_p)]
        L.mrq_search_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(SearchParams), C.c_void_p,
                                       C.c_void_p, C.c_void_p]
        L.mrq_search_batch_device.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(SearchParams),
                                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.mrq_free.argtypes = [C.c_void_p]
        L.mrq_free.restype = None
        L.mrq_debug_fetch.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]
        L.mrq_index_info.argtypes = [C.c_void_p] + [C.c_void_p] * 5
        L.mrq_debug_set.restype = C.c_int
        L.mrq_debug_set.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
        L.mrq_nccl_unique_id.restype = C.c_int
        L.mrq_nccl_unique_id.argtypes = [C.c_void_p, C.c_size_t]
        L.mrq_shard_plan.restype = C.c_int
        L.mrq_shard_plan.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]
        _lib = L
    return _lib


def mrq_last_error() -> str:
    return lib().mrq_last_error().decode()


def _check(rc):
    if rc != 0:
        raise MRQError(rc, mrq_last_error())


def _ptr(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


_CALLBACKS = {}   # handle value -> ctypes callback (kept alive while the index lives)


def host_allgather_callback(fn):
    """Wraps fn(send: bytes, world_bytes_out: memoryview) ... as the C callback:
    fn(send_bytes) must return the rank-major concatenation of every rank's
    bytes (len = world * len(send_bytes))."""
    def cb(send, recv, nbytes, ctx):
        try:
            data = fn(C.string_at(send, nbytes))
            C.memmove(recv, data, len(data))
            return 0
        except Exception:  # pragma: no cover - reported as MRQ_ENCCL by the library
            return 1
    return ALLGATHER_FN(cb)


MRQ_LOAD_TAILS_HOST = 1


def mrq_index_load(build_file: str, base: np.ndarray, d: int, rank=0, world=1, device=-1, nccl_unique_id=None,
                   host_allgather=None, tails_host=False):
    """host_allgather: optional python callable send_bytes -> all ranks' bytes
    (rank-major), used in place of NCCL when nccl_unique_id is None."""
    base = np.ascontiguousarray(base, dtype=np.float32)
    n, D = base.shape
    h = C.c_void_p()
    uid = None
    if nccl_unique_id is not None:
        uid = C.create_string_buffer(bytes(nccl_unique_id), 128)
    cb = host_allgather_callback(host_allgather) if host_allgather is not None else ALLGATHER_FN()
    cfg = DistCfg(rank, world, device, C.cast(uid, C.c_void_p) if uid is not None else None, cb, None)
    flags = MRQ_LOAD_TAILS_HOST if tails_host else 0
    _check(lib().mrq_index_load_ex(build_file.encode(), _ptr(base), n, D, d, C.byref(cfg), flags, C.byref(h)))
    if host_allgather is not None:
        _CALLBACKS[h.value] = cb
    return h


class BuildParams(C.Structure):
    _fields_ = [("k", C.c_int32), ("pca_sample", C.c_int32), ("km_sample_per_k", C.c_int32),
                ("km_iters", C.c_int32), ("seed", C.c_uint64)]


def mrq_build_gpu(base: np.ndarray, d: int, k: int, out_path: str, pca_sample=100_000, km_sample_per_k=64,
                  km_iters=25, seed=7, device=-1):
    """GPU index build -> MRQBLD01 file; returns the phase
    times in ms (PCA, k-means, final assignment, total)."""
    import hashlib
    base = np.ascontiguousarray(base, dtype=np.float32)
    n, D = base.shape
    sha = hashlib.sha256(base.tobytes()).hexdigest().encode()
    bp = BuildParams(k, pca_sample, km_sample_per_k, km_iters, seed)
    t = (C.c_double * 4)()
    L = lib()
    L.mrq_build_gpu.restype = C.c_int
    L.mrq_build_gpu.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.POINTER(BuildParams), C.c_char_p,
                                C.c_int32, C.c_char_p, C.c_void_p]
    _check(L.mrq_build_gpu(_ptr(base), n, D, d, C.byref(bp), sha, device, out_path.encode(), t))
    return {"pca_ms": t[0], "kmeans_ms": t[1], "assign_ms": t[2], "total_ms": t[3]}


def mrq_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().mrq_nccl_unique_id(buf, 128))
    return buf.raw


nccl_unique_id = mrq_nccl_unique_id


def mrq_shard_plan(sizes, world: int) -> np.ndarray:
    s = np.ascontiguousarray(sizes, dtype=np.uint32)
    owner = np.empty(s.shape[0], np.uint32)
    _check(lib().mrq_shard_plan(_ptr(s), s.shape[0], world, _ptr(owner)))
    return owner


MRQ_EDIM = -2
MRQ_EINVAL = -1


def _index_D(h):
    return mrq_index_info(h)["D"]


def mrq_search_batch(h, queries: np.ndarray, params: SearchParams, with_stats=True, out_ids=None, out_dist=None):
    """Host buffers in and out; out_ids/out_dist (nq x K int64 / float32,
    e.g. pinned) are filled in place when given."""
    q = np.ascontiguousarray(queries, dtype=np.float32)
    if q.ndim != 2 or q.shape[1] != _index_D(h):
        raise MRQError(MRQ_EDIM, "queries must be (nq, D=%d), got %s" % (_index_D(h), q.shape))
    nq = q.shape[0]
    ids = out_ids if out_ids is not None else np.empty((nq, params.K), np.int64)
    dist = out_dist if out_dist is not None else np.empty((nq, params.K), np.float32)
    if not (ids.shape == (nq, params.K) and ids.dtype == np.int64 and ids.flags.c_contiguous):
        raise MRQError(MRQ_EINVAL, "out_ids must be C-contiguous int64 (%d, %d)" % (nq, params.K))
    if not (dist.shape == (nq, params.K) and dist.dtype == np.float32 and dist.flags.c_contiguous):
        raise MRQError(MRQ_EINVAL, "out_dist must be C-contiguous float32 (%d, %d)" % (nq, params.K))
    st = Stats()
    _check(lib().mrq_search_batch(h, _ptr(q), nq, C.byref(params), _ptr(ids), _ptr(dist),
                                  C.byref(st) if with_stats else None))
    return ids, dist, st


def _check_dev(t, name, dtype, shape):
    import torch
    if not isinstance(t, torch.Tensor) or t.device.type != "cuda":
        raise MRQError(MRQ_EINVAL, "%s must be a CUDA tensor" % name)
    if t.dtype != dtype or not t.is_contiguous() or tuple(t.shape) != tuple(shape):
        raise MRQError(MRQ_EDIM if name == "d_queries" else MRQ_EINVAL,
                       "%s must be contiguous %s %s, got %s %s" % (name, dtype, tuple(shape), t.dtype, tuple(t.shape)))


def mrq_search_batch_device(h, d_queries, params: SearchParams, d_ids, d_dist, stats: Stats | None = None,
                            stream=None):
    import torch
    nq = d_queries.shape[0] if d_queries.ndim == 2 else -1
    _check_dev(d_queries, "d_queries", torch.float32, (max(nq, 0), _index_D(h)))
    _check_dev(d_ids, "d_ids", torch.int64, (nq, params.K))
    _check_dev(d_dist, "d_dist", torch.float32, (nq, params.K))
    s = C.c_void_p(stream) if stream else None
    _check(lib().mrq_search_batch_device(h, _ptr(d_queries), nq, C.byref(params), _ptr(d_ids), _ptr(d_dist),
                                         C.byref(stats) if stats is not None else None, s))


def mrq_free(h):
    if h:
        lib().mrq_free(h)
        _CALLBACKS.pop(getattr(h, "value", h), None)


def mrq_index_info(h):
    n, npad = C.c_int64(), C.c_int64()
    D, d, k = C.c_int32(), C.c_int32(), C.c_int32()
    _check(lib().mrq_index_info(h, C.byref(n), C.byref(D), C.byref(d), C.byref(k), C.byref(npad)))
    return {"n": n.value, "D": D.value, "d": d.value, "k": k.value, "npad": npad.value}


_DT = {"u16": np.uint16, "u32": np.uint32, "u64": np.uint64, "f32": np.float32, "f64": np.float64}


def mrq_debug_set(h, name: str, value: int):
    _check(lib().mrq_debug_set(h, name.encode(), value))


def mrq_debug_fetch(h, name: str, dtype: str):
    need = C.c_size_t()
    _check(lib().mrq_debug_fetch(h, name.encode(), None, 0, C.byref(need)))
    out = np.empty(need.value // np.dtype(_DT[dtype]).itemsize, _DT[dtype])
    _check(lib().mrq_debug_fetch(h, name.encode(), _ptr(out), out.nbytes, C.byref(need)))
    return out


class Index:
    """Convenience owner of an mrq_index handle."""

    def __init__(self, build_file, base, d, **kw):
        self.build_file = build_file
        self.h = mrq_index_load(build_file, base, d, **kw)
        self.info = mrq_index_info(self.h)

    def search(self, queries, K=10, nprobe=16, **kw):
        return mrq_search_batch(self.h, queries, SearchParams.make(K=K, nprobe=nprobe, **kw))

    def fetch(self, name, dtype):
        return mrq_debug_fetch(self.h, name, dtype)

    def close(self):
        mrq_free(self.h)
        self.h = None

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.close()
        except Exception:
            pass

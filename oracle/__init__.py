"""The MRQ oracle -- TEST INFRASTRUCTURE ONLY.

A plain, slow, fp64 CPU implementation of the paper's query path
(oracle/mrq_oracle.c) plus the index build (oracle/build.py).  Only
``tests/``, ``__graft_entry__.smoke()``, ``scripts/make_artifacts.py`` (which
calls nothing but this package) and bench.py's ``cpu_baseline`` /
``--impl reference`` leg may import it.  The CUDA path never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from . import build as build_mod  # noqa: F401

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "mrq_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

MODES = {"FULL": 0, "STAGE1_ONLY": 1, "EXACT": 2, "NOCORR": 3, "SEQ": 4}


def compile_oracle(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                               "-fPIC", "-shared", "-o", LIB, SRC, "-lm"])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(compile_oracle())
        _lib.orc_search.restype = C.c_int
        _lib.orc_encode_head.restype = C.c_double
        _lib.orc_quantize.restype = C.c_int64
        _lib.orc_ip_quantized.restype = C.c_double
        _lib.orc_ip_unquantized.restype = C.c_double
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


class OrcIndex(C.Structure):
    _fields_ = [("N", C.c_int32), ("D", C.c_int32), ("d", C.c_int32), ("k", C.c_int32), ("W", C.c_int32)] + \
               [(n, C.c_void_p) for n in ("mu", "P", "lam", "R", "C", "assign", "head", "tail", "xr2f", "code",
                                          "f1", "f2", "f3", "list_off", "list_ids", "Rc")]


class OrcParams(C.Structure):
    _fields_ = [("K", C.c_int32), ("nprobe", C.c_int32), ("eps0", C.c_double), ("m", C.c_double),
                ("mode", C.c_int32), ("tau_schedule", C.c_int32), ("seed_mult", C.c_int32),
                ("resid_scale", C.c_double), ("Bq", C.c_int32), ("est_kind", C.c_int32),
                ("seed_lists", C.c_int32)]


class OrcStats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("scanned", "f1", "f2", "exact", "s0", "s1")]


_DUMP_FIELDS = ["qp", "qr2", "eps_r", "r0", "probe", "probe_qn2", "levels", "qconst", "tau0", "tau1", "cap",
                "scan_cnt", "scan_ids", "scan_dis", "scan_lb1", "s0_cnt", "s0_ids", "s0_exact",
                "s1_cnt", "s1_ids", "s1_exact", "f1_cnt", "f1_ids", "f1_diso", "f2_cnt", "f2_ids", "f2_exact"]


class OrcDump(C.Structure):
    _fields_ = [(n, C.c_int64 if n == "cap" else C.c_void_p) for n in _DUMP_FIELDS]


class Index:
    """Oracle index: build-file arrays + Alg.1 L3-L8 encoding of the base."""

    def __init__(self, bf, X: np.ndarray, lists=None):
        """lists: optional iterable of IVF list ids -- only their vectors are
        encoded (searches must then probe only those lists; see
        probe_lists()).  The arrays stay full-size (untouched pages cost no
        memory)."""
        X = np.ascontiguousarray(X, dtype=np.float32)
        N, D = X.shape
        if D != bf.D or N != bf.N:
            raise ValueError("DimensionMismatch")
        self.bf = bf
        self.N, self.D, self.d, self.k = N, D, bf.d, bf.k
        d = bf.d
        self.W = (d + 31) // 32
        self.mu = np.ascontiguousarray(bf.mu, np.float64)
        self.P = np.ascontiguousarray(bf.P, np.float64)
        self.lam = np.ascontiguousarray(bf.lam, np.float64)
        self.R = np.ascontiguousarray(bf.R, np.float64)
        self.C = np.ascontiguousarray(bf.C, np.float64)
        self.assign = np.ascontiguousarray(bf.assign, np.uint32)
        self.head = np.zeros((N, d), np.float32)
        self.tail = np.zeros((N, max(D - d, 0)), np.float32)
        self.xr2f = np.zeros(N, np.float32)
        self.code = np.zeros((N, self.W), np.uint32)
        self.f1 = np.zeros(N, np.float32)
        self.f2 = np.zeros(N, np.float32)
        self.f3 = np.zeros(N, np.float32)
        self.list_off = np.zeros(self.k + 1, np.int64)
        self.list_ids = np.zeros(N, np.int64)
        self.Rc = np.zeros((self.k, d), np.float64)
        self.s = OrcIndex(N, D, d, self.k, self.W, *[_p(getattr(self, n)) for n in (
            "mu", "P", "lam", "R", "C", "assign", "head", "tail", "xr2f", "code", "f1", "f2", "f3",
            "list_off", "list_ids", "Rc")])
        if lists is None:
            lib().orc_encode(C.byref(self.s), _p(X))
        else:
            only = np.zeros(self.k, np.uint8)
            only[np.asarray(list(lists), np.int64)] = 1
            self.only = only
            lib().orc_encode_subset(C.byref(self.s), _p(X), _p(only))

    def list_sizes(self):
        return np.diff(self.list_off)

    def search(self, queries, K=10, nprobe=4, eps0=1.9, m=4.0, mode="FULL", tau_schedule="TIGHT",
               seed_mult=2, resid_scale=2.0, Bq=4, est_kind=0, dump=False, cap=None, seed_lists=1):
        Qv = np.ascontiguousarray(queries, dtype=np.float32)
        nq = Qv.shape[0]
        pr = OrcParams(K, nprobe, eps0, m, MODES[mode] if isinstance(mode, str) else mode,
                       0 if tau_schedule == "TIGHT" else 1, seed_mult, resid_scale, Bq, est_kind, seed_lists)
        ids = np.zeros((nq, K), np.int64)
        dist = np.zeros((nq, K), np.float32)
        st = OrcStats()
        dp = None
        out = {}
        if dump:
            npb = min(nprobe, self.k)
            if cap is None:
                cap = int(np.sort(self.list_sizes())[::-1][:npb].sum())
            D, d = self.D, self.d
            shapes = {"qp": ((nq, D), np.float64), "qr2": ((nq,), np.float64), "eps_r": ((nq,), np.float64),
                      "r0": ((nq, d), np.float64), "probe": ((nq, npb), np.int32),
                      "probe_qn2": ((nq, npb), np.float64), "levels": ((nq, npb, d), np.uint8),
                      "qconst": ((nq, npb, 5), np.float64), "tau0": ((nq,), np.float64),
                      "tau1": ((nq,), np.float64)}
            for nm in ("scan", "s0", "s1", "f1", "f2"):
                shapes[nm + "_cnt"] = ((nq,), np.int64)
                shapes[nm + "_ids"] = ((nq, cap), np.int64)
            shapes["scan_dis"] = ((nq, cap), np.float64)
            shapes["scan_lb1"] = ((nq, cap), np.float64)
            shapes["s0_exact"] = ((nq, cap), np.float64)
            shapes["s1_exact"] = ((nq, cap), np.float64)
            shapes["f1_diso"] = ((nq, cap), np.float64)
            shapes["f2_exact"] = ((nq, cap), np.float64)
            for nm, (shp, dt) in shapes.items():
                out[nm] = np.zeros(shp, dt)
            dp = OrcDump(*[cap if n == "cap" else _p(out[n]) for n in _DUMP_FIELDS])
        rc = lib().orc_search(C.byref(self.s), nq, _p(Qv), C.byref(pr), _p(ids), _p(dist), C.byref(st),
                              C.byref(dp) if dp is not None else None)
        if rc != 0:
            raise ValueError("InvalidConfig")
        stats = {n: getattr(st, n) for n, _ in OrcStats._fields_}
        if dump:
            return ids, dist, stats, out
        return ids, dist, stats


def probe_lists(bf, X_queries, nprobe, margin=8):
    """The lists a search of these queries can probe: for each query the
    nprobe + margin nearest projected centroids (fp64 numpy; the margin covers
    any ordering difference against the oracle's own canonical probe, which
    orc_search re-derives).  Used to encode only what a sampled search reads."""
    Qv = np.asarray(X_queries, np.float64)
    qd = (Qv - bf.mu) @ bf.P[:bf.d].T
    cn = (bf.C * bf.C).sum(1)
    out = set()
    for s in range(0, qd.shape[0], 256):
        dd = cn[None, :] - 2.0 * qd[s:s + 256] @ bf.C.T
        m = min(bf.k, nprobe + margin)
        out.update(np.argpartition(dd, m - 1, axis=1)[:, :m].ravel().tolist())
    return sorted(out)


def bruteforce(X, Qv, K):
    """Exact KNN in the original space, fp64 plain loops.  Small inputs."""
    X = np.ascontiguousarray(X, np.float32)
    Qv = np.ascontiguousarray(Qv, np.float32)
    ids = np.zeros((Qv.shape[0], K), np.int64)
    dist = np.zeros((Qv.shape[0], K), np.float64)
    lib().orc_bruteforce(C.c_int64(X.shape[0]), C.c_int32(X.shape[1]), _p(X), C.c_int64(Qv.shape[0]), _p(Qv),
                         C.c_int32(K), _p(ids), _p(dist))
    return ids, dist


def groundtruth(X, Qv, K, extra=64, block=4096):
    """Exact KNN for larger inputs: a fp64 matmul screens the top K+extra per
    query, then each survivor is rescored with the plain fp64 loop and the K
    smallest (dist, id) are kept.  The screen's error (~1e-13 relative) is far
    below the screen depth's margin at the sizes used."""
    X = np.ascontiguousarray(X, np.float32)
    Qv = np.ascontiguousarray(Qv, np.float32)
    Xd = X.astype(np.float64)
    xn = np.einsum("ij,ij->i", Xd, Xd)
    ids = np.zeros((Qv.shape[0], K), np.int64)
    dist = np.zeros((Qv.shape[0], K), np.float64)
    M = min(X.shape[0], K + extra)
    for s in range(0, Qv.shape[0], 64):
        q = Qv[s:s + 64].astype(np.float64)
        best_v = np.full((q.shape[0], M), np.inf)
        best_i = np.zeros((q.shape[0], M), np.int64)
        for b in range(0, X.shape[0], block * 64):
            dd = xn[None, b:b + block * 64] - 2.0 * (q @ Xd[b:b + block * 64].T)
            idx = np.argpartition(dd, min(M, dd.shape[1]) - 1, axis=1)[:, :M] if dd.shape[1] > M else \
                np.broadcast_to(np.arange(dd.shape[1]), dd.shape)
            vals = np.take_along_axis(dd, idx, 1)
            cv = np.concatenate([best_v, vals], 1)
            ci = np.concatenate([best_i, idx + b], 1)
            keep = np.argpartition(cv, M - 1, axis=1)[:, :M]
            best_v = np.take_along_axis(cv, keep, 1)
            best_i = np.take_along_axis(ci, keep, 1)
        for r in range(q.shape[0]):
            cand = np.ascontiguousarray(best_i[r][np.isfinite(best_v[r])], np.int64)
            ex = np.zeros(cand.shape[0])
            lib().orc_exact_original(C.c_int32(X.shape[1]), _p(X), _p(Qv[s + r]), C.c_int64(cand.shape[0]),
                                     _p(cand), _p(ex))
            o = np.lexsort((cand, ex))[:K]
            ids[s + r, :len(o)] = cand[o]
            dist[s + r, :len(o)] = ex[o]
    return ids, dist


def recall_at_k(found, gt, K):
    """Recall@K = |T n G| / |G| averaged over queries (A-26)."""
    found = np.asarray(found)[:, :K]
    gt = np.asarray(gt)[:, :K]
    hits = 0
    for f, g in zip(found, gt):
        hits += len(set(f.tolist()) & set(g.tolist()))
    return hits / float(gt.shape[0] * K)


# ---- unit entry points (the same C functions the search uses) ----

def encode_head(R, t):
    """(code u32[W], u, ||t||^2) for one head residual t (Alg.1 L7-L8)."""
    R = np.ascontiguousarray(R, np.float64)
    t = np.ascontiguousarray(t, np.float64)
    d = t.shape[0]
    code = np.zeros((d + 31) // 32, np.uint32)
    n2 = C.c_double()
    u = lib().orc_encode_head(C.c_int(d), _p(R), _p(t), _p(code), C.byref(n2))
    return code, u, n2.value


def quantize(r, Bq=4):
    """(levels, lo, delta, sumL) -- Alg.2 L5 uniform Bq-bit quantizer."""
    r = np.ascontiguousarray(r, np.float64)
    L = np.zeros(r.shape[0], np.uint8)
    lo = C.c_double()
    de = C.c_double()
    s = lib().orc_quantize(C.c_int(r.shape[0]), _p(r), C.c_int(Bq), _p(L), C.byref(lo), C.byref(de))
    return L, lo.value, de.value, int(s)


def ip_quantized(code, L, lo, delta, sumL):
    """<x_hat, r_bar> via the oracle's plain-loop S = sum_{bit=1} L_j."""
    d = L.shape[0]
    A, Bc = 2.0 * lo, 2.0 * delta
    C0 = float(d) * lo + delta * float(sumL)
    isd = 1.0 / np.sqrt(float(d))
    return lib().orc_ip_quantized(C.c_int(d), _p(np.ascontiguousarray(code, np.uint32)),
                                  _p(np.ascontiguousarray(L, np.uint8)), C.c_double(A), C.c_double(Bc),
                                  C.c_double(C0), C.c_double(isd))


def ip_unquantized(code, r):
    r = np.ascontiguousarray(r, np.float64)
    d = r.shape[0]
    return lib().orc_ip_unquantized(C.c_int(d), _p(np.ascontiguousarray(code, np.uint32)), _p(r),
                                    C.c_double(1.0 / np.sqrt(float(d))))


def prepare_query(ix, q, resid_scale=2.0, m=4.0):
    """(q_p, ||q_r||^2, eps_r, r0) -- Alg.2 L1-L4."""
    q = np.ascontiguousarray(q, np.float32)
    qp = np.zeros(ix.D)
    r0 = np.zeros(ix.d)
    qr2 = C.c_double()
    er = C.c_double()
    lib().orc_prepare_query(C.byref(ix.s), _p(q), C.c_double(resid_scale), C.c_double(m), _p(qp),
                            C.byref(qr2), C.byref(er), _p(r0))
    return qp, qr2.value, er.value, r0

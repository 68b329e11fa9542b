"""Oracle index build (Alg.1 L1-L6) -- TEST INFRASTRUCTURE ONLY.

Writes the seeded build file the CUDA path reads (BASELINE.json north_star:
"The GPU path reads the PCA matrix and centroids from the oracle's seeded
build file").  Only tests/, scripts that call nothing but oracle/, smoke()
and bench.py's cpu_baseline leg may import this module.

Steps (numpy fp64; library primitives -- eigh, QR, matmul -- serve as steps):
  L1-L2  PCA on a seeded subsample (<= 100k rows, seed 42; SPEC S:89-92,
         SURVEY A-15): mu = mean, Sigma = (X-mu)^T (X-mu)/(n-1), eigenpairs
         sorted by eigenvalue descending (ties by index), each eigenvector's
         largest-|entry| made positive; P rows = eigenvectors; lambda_i =
         max(eigenvalue, 0) are the per-dimension variances sigma_i^2 (A-17).
  L3-L5  x_p = P (x - mu); heads x_d = x_p[:d].
  L6     IVF* on the heads (projected centroids, Exp-2 P:2405):
         Lloyd k-means (<= 25 iterations, stop at relative WCSS gain < 1e-4,
         SPEC S:310) from a seeded Forgy init on a sample of min(64k, N)
         rows (seed 7; SURVEY A-20 reading), empty clusters re-seeded at the
         farthest member of the largest cluster; final assignment of all N
         by argmin distance.
  P_r    Haar d x d rotation for the quantizer: QR of a
         seed-7 Gaussian with sign-fixed columns; applied as y = R t.

File format MRQBLD01 (little-endian), documented in include/mrq.h:
  char magic[8] = "MRQBLD01"; u32 version = 1; u32 D; u32 d; u32 k; u64 N;
  u64 flags = 0; char base_sha256_hex[64];
  f64 mu[D]; f64 P[D*D]; f64 lambda[D]; f64 R[d*d]; f64 centroids[k*d];
  u32 assign[N]; char end[8] = "MRQEND01".
"""
from __future__ import annotations

import hashlib
import struct
from dataclasses import dataclass

import numpy as np

MAGIC = b"MRQBLD01"
END = b"MRQEND01"
VERSION = 1


@dataclass
class BuildFile:
    D: int
    d: int
    k: int
    N: int
    mu: np.ndarray
    P: np.ndarray
    lam: np.ndarray
    R: np.ndarray
    C: np.ndarray
    assign: np.ndarray
    sha: str = ""


def pca(X: np.ndarray, sample_limit: int = 100_000, seed: int = 42):
    """Alg.1 L1-L2."""
    n = X.shape[0]
    if n < 2:
        raise ValueError("DegenerateData: N < 2")
    if n > sample_limit:
        idx = np.sort(np.random.default_rng(seed).choice(n, sample_limit, replace=False))
        S = X[idx].astype(np.float64)
    else:
        S = X.astype(np.float64)
    mu = S.mean(axis=0)
    Sc = S - mu
    cov = (Sc.T @ Sc) / (S.shape[0] - 1)
    if not np.any(np.diag(cov) > 0):
        raise ValueError("DegenerateData: zero total variance")
    w, V = np.linalg.eigh(cov)
    order = np.argsort(-w, kind="stable")
    w = w[order]
    V = V[:, order]
    for i in range(V.shape[1]):
        j = int(np.argmax(np.abs(V[:, i])))
        if V[j, i] < 0:
            V[:, i] = -V[:, i]
    P = np.ascontiguousarray(V.T)
    lam = np.maximum(w, 0.0)
    return mu, P, lam


def random_orthogonal(dim: int, seed: int = 7) -> np.ndarray:
    """Haar rotation P_r: sign-fixed QR of a seeded Gaussian."""
    g = np.random.default_rng(seed).standard_normal((dim, dim))
    q, r = np.linalg.qr(g)
    s = np.sign(np.diag(r))
    s[s == 0] = 1.0
    return np.ascontiguousarray(q * s[None, :])


def _assign(X: np.ndarray, C: np.ndarray, block: int = 8192):
    """argmin_j ||x - c_j||^2 (ties -> smaller j) and the min value."""
    cn = np.einsum("ij,ij->i", C, C)
    a = np.empty(X.shape[0], dtype=np.int64)
    dmin = np.empty(X.shape[0])
    for s in range(0, X.shape[0], block):
        x = X[s:s + block]
        dist = cn[None, :] - 2.0 * (x @ C.T) + np.einsum("ij,ij->i", x, x)[:, None]
        a[s:s + block] = np.argmin(dist, axis=1)
        dmin[s:s + block] = np.maximum(dist[np.arange(x.shape[0]), a[s:s + block]], 0.0)
    return a, dmin


def kmeans(X: np.ndarray, k: int, max_iters: int = 25, seed: int = 7, tol: float = 1e-4):
    """Lloyd k-means; returns centroids k x d."""
    n = X.shape[0]
    if k > n:
        raise ValueError("InvalidConfig: k > N")
    rng = np.random.default_rng(seed)
    C = X[np.sort(rng.choice(n, k, replace=False))].copy()
    prev = np.inf
    for _ in range(max_iters):
        a, dmin = _assign(X, C)
        wcss = float(dmin.sum())
        cnt = np.bincount(a, minlength=k)
        sums = np.zeros_like(C)
        np.add.at(sums, a, X)
        nz = cnt > 0
        C[nz] = sums[nz] / cnt[nz][:, None]
        for j in np.nonzero(~nz)[0]:               # empty cluster repair
            big = int(np.argmax(cnt))
            members = np.nonzero(a == big)[0]
            far = members[int(np.argmax(dmin[members]))]
            C[j] = X[far]
            cnt[big] -= 1
            cnt[j] = 1
            a[far] = j
            dmin[far] = 0.0
        if prev < np.inf and (prev - wcss) <= tol * prev:
            break
        prev = wcss
    return C


def build(X: np.ndarray, d: int, k: int, *, pca_sample: int = 100_000, km_sample_per_k: int = 64,
          km_iters: int = 25) -> BuildFile:
    """Alg.1 L1-L6 plus P_r.  X: base vectors float32 [N, D]."""
    N, D = X.shape
    if not (2 <= d <= D):
        raise ValueError("InvalidConfig: need 2 <= d <= D")
    mu, P, lam = pca(X, pca_sample)
    heads = np.empty((N, d))
    for s in range(0, N, 65536):
        heads[s:s + 65536] = (X[s:s + 65536].astype(np.float64) - mu) @ P[:d].T
    m = min(N, km_sample_per_k * k)
    sidx = np.sort(np.random.default_rng(7).choice(N, m, replace=False)) if m < N else np.arange(N)
    C = kmeans(heads[sidx], k, km_iters)
    assign, _ = _assign(heads, C)
    R = random_orthogonal(d, 7)
    sha = hashlib.sha256(np.ascontiguousarray(X, dtype=np.float32).tobytes()).hexdigest()
    return BuildFile(D, d, k, N, mu, P, lam, R, np.ascontiguousarray(C), assign.astype(np.uint32), sha)


def write(path: str, b: BuildFile) -> None:
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<IIIIQQ", VERSION, b.D, b.d, b.k, b.N, 0))
        f.write(b.sha.encode("ascii").ljust(64, b"0")[:64])
        for a in (b.mu, b.P, b.lam, b.R, b.C):
            f.write(np.ascontiguousarray(a, dtype="<f8").tobytes())
        f.write(np.ascontiguousarray(b.assign, dtype="<u4").tobytes())
        f.write(END)


def read(path: str) -> BuildFile:
    with open(path, "rb") as f:
        buf = f.read()
    if buf[:8] != MAGIC:
        raise ValueError("VersionMismatch: bad magic")
    ver, D, d, k, N, _flags = struct.unpack_from("<IIIIQQ", buf, 8)
    if ver != VERSION:
        raise ValueError("VersionMismatch")
    sha = buf[40:104].decode("ascii")
    off = 104
    out = []
    for n in (D, D * D, D, d * d, k * d):
        out.append(np.frombuffer(buf, "<f8", n, off).copy())
        off += 8 * n
    assign = np.frombuffer(buf, "<u4", N, off).copy()
    off += 4 * N
    if buf[off:off + 8] != END:
        raise ValueError("FormatError: truncated at offset %d" % off)
    mu, P, lam, R, C = out
    return BuildFile(D, d, k, N, mu, P.reshape(D, D), lam, R.reshape(d, d), C.reshape(k, d), assign, sha)

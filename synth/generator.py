"""Seeded Gaussian-mixture generator G(D, alpha, C, post, seeds).

Recipe (BASELINE.json ``configs``):

1. R_D = Haar(D): modified Gram-Schmidt of a standard Gaussian D x D drawn
   with ``seed_R``.
2. lambda_i = i^-alpha (i = 1..D), normalised to mean 1.
3. C > 0: component means m_c = sqrt(1/2) R_D (sqrt(lambda) * z_c) with
   z_c ~ N(0, I) (``seed_means``); labels uniform (``seed_data``);
   x = m_label + sqrt(1/2) R_D (sqrt(lambda) * z).  The population covariance
   is R_D diag(lambda) R_D^T whatever C is.
   C = 0: x = R_D (sqrt(lambda) * z).
4. ``post`` maps the Gaussian sample to the workload's value domain.
5. N + Q points are drawn; the first N are the base, the last Q the queries
   (held-out queries, as PAPER.md line 2095 does for query-less datasets).

Bit reproducibility across machines: random numbers come from one numpy
PCG64 stream in fixed 65536-row chunks, and every product/sum is written as
an explicit sequence of elementwise IEEE operations (no BLAS, whose blocking
depends on the CPU), so the host that builds artefacts and the GPU box draw
identical float32 vectors.  The elementwise loop runs on CUDA when a device
is given (same IEEE results, faster).

All arithmetic here is input synthesis; nothing in this file belongs to the
MRQ method.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

CHUNK = 65536


@dataclass(frozen=True)
class Config:
    name: str
    index: int            # config index c: seeds are 1000+c, 2000+c, 3000+c
    N: int
    Q: int
    D: int
    alpha: float
    C: int                # mixture components (0 = single Gaussian)
    post: str             # "none" | "sift" | "unit" | "gist"
    k: int                # IVF clusters
    d: tuple              # code lengths evaluated
    K: tuple              # result sizes evaluated
    nprobe: tuple         # nprobe grid
    default_nprobe: int = 0

    @property
    def seed_R(self):
        return 1000 + self.index

    @property
    def seed_means(self):
        return 2000 + self.index

    @property
    def seed_data(self):
        return 3000 + self.index


GRID = (16, 24, 32, 48, 64, 96, 128, 192, 256)

CONFIGS = (
    # BASELINE.json configs[0]
    Config("tiny", 0, 10_000, 100, 64, 1.5, 0, "none", 16, (16,), (10,), (1, 2, 4, 8, 16), 4),
    # configs[1]: the bench workload
    Config("sift", 1, 1_000_000, 10_000, 128, 1.2, 64, "sift", 4096, (64,), (10,), GRID, 64),
    # configs[2]
    Config("deep", 2, 10_000_000, 10_000, 96, 1.0, 256, "unit", 16384, (32, 64), (10, 100), GRID, 64),
    # configs[3]
    Config("gist", 3, 1_000_000, 1_000, 960, 2.0, 64, "gist", 4096, (128, 256), (10,), GRID, 64),
    # configs[4]
    Config("emb", 4, 5_000_000, 10_000, 1536, 0.8, 1024, "unit", 16384, (256, 512), (10, 100), GRID, 64),
)


def config_by_name(name: str) -> Config:
    for c in CONFIGS:
        if c.name == name:
            return c
    raise KeyError(name)


def haar(D: int, seed: int) -> np.ndarray:
    """Haar-distributed orthogonal D x D matrix (columns orthonormal).

    Modified Gram-Schmidt with one re-orthogonalisation pass; dot products
    are column-wise ``np.add.reduce(..., axis=0)`` over C-contiguous rows,
    which numpy evaluates as a sequential row-by-row accumulation.
    """
    V = np.random.default_rng(seed).standard_normal((D, D))
    for i in range(D):
        for _ in range(2):
            if i > 0:
                Qi = V[:, :i]
                coef = np.add.reduce(Qi * V[:, i:i + 1], axis=0)
                proj = np.add.reduce(np.ascontiguousarray((Qi * coef[None, :]).T), axis=0)
                V[:, i] = V[:, i] - proj
        nrm = np.sqrt(np.add.reduce(np.ascontiguousarray(V[:, i:i + 1] * V[:, i:i + 1]), axis=0)[0])
        V[:, i] = V[:, i] / nrm
    return V


def _post(x: np.ndarray, post: str) -> np.ndarray:
    if post == "none":
        return x
    if post == "sift":
        return np.rint(np.clip(40.0 + 30.0 * x, 0.0, 255.0))
    if post == "gist":
        return np.clip(0.5 + 0.15 * x, 0.0, 1.0)
    if post == "unit":
        n2 = np.zeros(x.shape[0])
        for j in range(x.shape[1]):
            n2 = n2 + x[:, j] * x[:, j]
        n = np.sqrt(n2)
        n[n == 0] = 1.0
        return x / n[:, None]
    raise ValueError(post)


def _matvec_rows(z, A, device):
    """x[n, i] = sum_j A[i, j] z[n, j], accumulated j = 0..D-1 (elementwise)."""
    if device is not None:
        import torch
        zt = torch.from_numpy(z).to(device)
        At = torch.from_numpy(np.ascontiguousarray(A.T)).to(device)   # At[j, i] = A[i, j]
        x = torch.zeros_like(zt)
        for j in range(z.shape[1]):
            x = x + zt[:, j:j + 1] * At[j:j + 1, :]
        return x.cpu().numpy()
    At = np.ascontiguousarray(A.T)
    x = np.zeros_like(z)
    blk = max(256, (1 << 18) // max(1, z.shape[1]))      # keep the block cache-resident
    tmp = np.empty((blk, z.shape[1]))
    for s in range(0, z.shape[0], blk):
        xs = x[s:s + blk]
        zs = z[s:s + blk]
        t = tmp[:xs.shape[0]]
        for j in range(z.shape[1]):
            np.multiply(zs[:, j:j + 1], At[j:j + 1, :], out=t)
            np.add(xs, t, out=xs)
    return x


def generate(cfg: Config, N: int | None = None, Q: int | None = None, D: int | None = None,
             device=None):
    """Return (base float32 [N, D], queries float32 [Q, D]).

    ``N``/``Q``/``D`` override the config's sizes (smaller test cases keep the
    config's distribution and seeds).  ``device`` ("cuda"/"cpu"/None) only
    chooses where the elementwise loop runs; the output is identical.
    """
    N = cfg.N if N is None else N
    Q = cfg.Q if Q is None else Q
    D = cfg.D if D is None else D
    lam = np.arange(1, D + 1, dtype=np.float64) ** (-cfg.alpha)
    lam = lam / np.add.reduce(lam) * D
    A = haar(D, cfg.seed_R) * np.sqrt(lam)[None, :]          # x = A z
    rng = np.random.default_rng(cfg.seed_data)
    if cfg.C > 0:
        zc = np.random.default_rng(cfg.seed_means).standard_normal((cfg.C, D))
        means = np.sqrt(0.5) * _matvec_rows(zc, A, None)
        w = np.sqrt(0.5)
    else:
        means = None
        w = 1.0
    total = N + Q
    out = np.empty((total, D), dtype=np.float32)
    for s in range(0, total, CHUNK):
        n = min(CHUNK, total - s)
        z = rng.standard_normal((n, D))
        x = _matvec_rows(z, A, device)
        if w != 1.0:
            x = w * x
        if means is not None:
            lab = rng.integers(0, cfg.C, size=n)
            x = x + means[lab]
        out[s:s + n] = _post(x, cfg.post).astype(np.float32)
    return out[:N], out[N:]


def base_sha256(x: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.float32).tobytes()).hexdigest()

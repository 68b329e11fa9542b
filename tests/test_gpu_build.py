"""GPU index build (Algorithm 1 L1-L6 + P_r on the GPU).

Its contract is recall-equivalence with the oracle build (same algorithm,
strided instead of random samples, other solvers -- not the same bits):
orthonormal PCA with descending eigenvalues close to the oracle's, a valid
assignment (every vector in the list of its nearest centroid), a Haar
rotation, and the same recall on the parity workloads.
"""
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _recall(ids, gt, K=10):
    return sum(len(set(a.tolist()) & set(b.tolist())) for a, b in zip(ids[:, :K], gt[:, :K])) / float(gt.shape[0] * K)


@pytest.mark.parametrize("cfgname,d,k,nps", [("tiny", 16, 16, (1, 4)), ("sift", 64, 4096, (16,))])
def test_gpu_build_recall_equivalent(tmp_path, cfgname, d, k, nps):
    import oracle
    import synth
    from oracle import build as B
    import paper_2411_06158_b200 as m
    cfg = synth.config_by_name(cfgname)
    X, Q = synth.generate(cfg, device="cuda")
    path = str(tmp_path / "gpu.mrqb")
    t = m.mrq_build_gpu(X, d, k, path, device=0)
    assert t["total_ms"] > 0
    g = B.read(path)
    o = B.read(os.path.join(ROOT, "data", cfgname, "build_d%d.mrqb" % d))
    assert g.sha == synth.base_sha256(X) and g.N == X.shape[0] and g.k == k and g.d == d
    assert np.abs(g.P @ g.P.T - np.eye(g.D)).max() < 1e-9                   # orthonormal PCA
    assert np.all(np.diff(g.lam) <= 0) and np.all(g.lam >= 0)               # descending eigenvalues
    top = slice(0, 8)
    assert np.all(np.abs(g.lam[top] - o.lam[top]) <= 0.05 * o.lam[top])     # the same spectrum (samples differ)
    assert np.abs(g.R @ g.R.T - np.eye(d)).max() < 1e-9                     # Haar rotation
    heads = (X[:2000].astype(np.float64) - g.mu) @ g.P[:d].T              # a valid IVF assignment
    dd = ((heads[:, None, :] - g.C[None, :, :]) ** 2).sum(-1)
    best = dd.min(1)
    mine = dd[np.arange(2000), g.assign[:2000].astype(np.int64)]
    assert np.all(mine <= best * (1 + 1e-4) + 1e-6)
    gt = np.load(os.path.join(ROOT, "data", cfgname, "gt_k10.npy"))
    gx = m.Index(path, X, d)
    ox = m.Index(os.path.join(ROOT, "data", cfgname, "build_d%d.mrqb" % d), X, d)
    try:
        for npb in nps:
            rg = _recall(gx.search(Q, K=10, nprobe=npb)[0], gt)
            ro = _recall(ox.search(Q, K=10, nprobe=npb)[0], gt)
            assert rg >= ro - 0.02, (npb, rg, ro)
    finally:
        gx.close()
        ox.close()

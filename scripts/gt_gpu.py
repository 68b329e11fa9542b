"""Ground truth for the large configs on the GPU box (harness plumbing, SURVEY
§8d.4): a torch fp64 screen (||x||^2 - 2 <q, x> via float64 matmuls on the
GPU, in blocks) keeps the K + 64 best per query, every survivor is rescored
with the oracle's plain fp64 loop (oracle.groundtruth's rescoring) and the K
smallest (dist, id) are kept.  Cross-checked against the plain-loop
oracle.bruteforce on a query subsample (--check N) before anything is written.
  python scripts/gt_gpu.py deep --out=gpurun_out/data --check 64
"""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402


def gt_gpu(X, Q, K, extra=64, qb=1024, xb=1 << 21):
    import torch
    dev = torch.device("cuda", 0)
    M = K + extra
    ids = np.zeros((Q.shape[0], K), np.int64)
    dist = np.zeros((Q.shape[0], K))
    Xg = [torch.from_numpy(X[b:b + xb]).to(dev, torch.float64) for b in range(0, X.shape[0], xb)]
    xn = [(x * x).sum(1) for x in Xg]
    for s in range(0, Q.shape[0], qb):
        q = torch.from_numpy(Q[s:s + qb]).to(dev, torch.float64)
        bv, bi = None, None
        for j, x in enumerate(Xg):
            dd = xn[j][None, :] - 2.0 * (q @ x.T)
            v, i = torch.topk(dd, min(M, dd.shape[1]), dim=1, largest=False)
            i = i + j * xb
            if bv is None:
                bv, bi = v, i
            else:
                cv, ci = torch.cat([bv, v], 1), torch.cat([bi, i], 1)
                bv, k2 = torch.topk(cv, M, dim=1, largest=False)
                bi = torch.gather(ci, 1, k2)
        cand = bi.cpu().numpy()
        for r in range(cand.shape[0]):
            c = np.ascontiguousarray(np.sort(cand[r]), np.int64)
            ex = np.zeros(c.shape[0])
            oracle.lib().orc_exact_original(C.c_int32(X.shape[1]), oracle._p(X), oracle._p(Q[s + r]),
                                            C.c_int64(c.shape[0]), oracle._p(c), oracle._p(ex))
            o = np.lexsort((c, ex))[:K]
            ids[s + r] = c[o]
            dist[s + r] = ex[o]
    return ids, dist


def main(name, outroot, check):
    cfg = synth.config_by_name(name)
    t = time.time()
    X, Q = synth.generate(cfg, device="cuda")
    print(name, "generated", X.shape, "%.1fs" % (time.time() - t), flush=True)
    Kmax = max(cfg.K)
    t = time.time()
    ids, _ = gt_gpu(X, Q, Kmax)
    print(name, "gpu gt K=%d %.1fs" % (Kmax, time.time() - t), flush=True)
    if check:
        t = time.time()
        # plain-loop fp64 brute force (oracle.bruteforce; pinned equal to
        # oracle.groundtruth by tests/test_oracle_pins.py) on the first queries
        oi, _ = oracle.bruteforce(X, Q[:check], Kmax)
        assert np.array_equal(oi, ids[:check]), "GPU ground truth differs from oracle.bruteforce"
        print(name, "cross-check vs oracle.bruteforce on %d queries ok %.1fs" % (check, time.time() - t), flush=True)
    out = os.path.join(outroot, name)
    os.makedirs(out, exist_ok=True)
    for K in cfg.K:
        np.save(os.path.join(out, "gt_k%d.npy" % K), ids[:, :K].astype(np.int32))


if __name__ == "__main__":
    outroot = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")), os.path.join(ROOT, "data"))
    check = int(sys.argv[sys.argv.index("--check") + 1]) if "--check" in sys.argv else 64
    main([a for a in sys.argv[1:] if not a.startswith("--") and not a.isdigit()][0], outroot, check)

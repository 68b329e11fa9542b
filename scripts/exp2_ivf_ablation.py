#!/usr/bin/env python
"""Exp-2 of the paper on the SIFT-shaped
workload: IVF with full-D centroids vs IVF* with centroids on the d leading
PCA dimensions, at equal nprobe, exact distances (mode EXACT).

Full-D IVF is the d = D build (k-means on x_p[0:D], the probe on all D
dimensions); IVF* is the bench's d = 64 build.  Both run through libmrq on
the GPU; recall@10 is against the fp64 ground truth.  The paper reports that
IVF* loses "almost no recall" at equal nprobe.
  python scripts/exp2_ivf_ablation.py > profiles/r01_exp2_ivf_ablation.json
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    import paper_2411_06158_b200 as mrq
    import synth
    from oracle import build as B
    cfg = synth.config_by_name("sift")
    X, Q = synth.generate(cfg, device="cuda")
    gt = np.load(os.path.join(ROOT, "data", "sift", "gt_k10.npy"))
    full = os.path.join(ROOT, "data", "sift", "build_d128.mrqb")
    if not os.path.exists(full):
        B.write(full, B.build(X, 128, cfg.k))          # the oracle's build, d = D
    out = {"workload": bench.WORKLOADS["sift"], "mode": "EXACT", "K": 10, "curves": {}}
    for name, d in (("IVF* (d=64 centroids)", 64), ("IVF (full-D centroids)", 128)):
        h = mrq.mrq_index_load(os.path.join(ROOT, "data", "sift", "build_d%d.mrqb" % d), X, d, device=0)
        pts = []
        for npb in (1, 2, 4, 8, 16, 24, 32, 48, 64):
            ids, _, st = mrq.mrq_search_batch(h, Q, mrq.SearchParams.make(K=10, nprobe=npb, mode="EXACT"))
            pts.append({"nprobe": npb, "recall10": round(bench.recall_at_k(ids, gt, 10), 4),
                        "scanned_per_q": round(st.scanned / Q.shape[0], 1)})
            print(name, pts[-1], file=sys.stderr, flush=True)
        out["curves"][name] = pts
        mrq.mrq_free(h)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

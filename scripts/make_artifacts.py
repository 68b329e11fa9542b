"""Writes the committed oracle artefacts under data/<config>/.

  build_d<d>.mrqb   the oracle's seeded build file (Alg.1 L1-L6 + P_r), read by
                    the CUDA path (BASELINE.json north_star)
  gt_k<K>.npy       exact KNN ids of the config's queries (fp64 ground truth)

Calls nothing but ``synth`` (seeded inputs) and ``oracle`` -- no value here
comes from the CUDA path (``--cuda`` only runs the generator's elementwise
loop on a GPU; its output is bit-identical).
Usage: python scripts/make_artifacts.py tiny sift [--cuda] [--out=DIR]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402
from oracle import build as B  # noqa: E402


def main(names, device=None, outroot=None):
    for name in names:
        cfg = synth.config_by_name(name)
        out = os.path.join(outroot or os.path.join(ROOT, "data"), name)
        os.makedirs(out, exist_ok=True)
        t = time.time()
        X, Q = synth.generate(cfg, device=device)   # the device only runs the elementwise loop: same bits
        print(name, "generated", X.shape, Q.shape, "%.1fs" % (time.time() - t), flush=True)
        for d in cfg.d:
            p = os.path.join(out, "build_d%d.mrqb" % d)
            if os.path.exists(p):
                continue
            t = time.time()
            bf = B.build(X, d, cfg.k)
            B.write(p, bf)
            print(name, "build d=%d" % d, "%.1fs" % (time.time() - t), flush=True)
        for K in cfg.K:
            p = os.path.join(out, "gt_k%d.npy" % K)
            if os.path.exists(p):
                continue
            t = time.time()
            ids, _ = oracle.groundtruth(X, Q, K)
            np.save(p, ids.astype(np.int32))
            print(name, "gt K=%d" % K, "%.1fs" % (time.time() - t), flush=True)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    dev = "cuda" if "--cuda" in sys.argv else None
    outroot = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")), None)
    main(args or ["tiny", "sift"], dev, outroot)

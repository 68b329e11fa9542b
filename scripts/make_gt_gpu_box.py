"""Ground truth for the large configs, run on the GPU box: the base is drawn
with the CUDA generator loop (bit-identical to the CPU one) and the exact KNN
is oracle.groundtruth (fp64, CPU).  Writes gt_k10.npy / gt_k100.npy under
--out (default data/<config>).  The build files for these configs are made
by the GPU builder (mrq_build_gpu) when bench.py first needs them.
  python scripts/make_gt_gpu_box.py deep --out=gpurun_out/data
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402


def main(name, outroot):
    cfg = synth.config_by_name(name)
    t = time.time()
    X, Q = synth.generate(cfg, device="cuda")
    print(name, "generated", X.shape, "%.1fs" % (time.time() - t), flush=True)
    out = os.path.join(outroot, name)
    os.makedirs(out, exist_ok=True)
    Kmax = max(cfg.K)
    t = time.time()
    ids, _ = oracle.groundtruth(X, Q, Kmax)
    print(name, "gt K=%d" % Kmax, "%.1fs" % (time.time() - t), flush=True)
    for K in cfg.K:
        np.save(os.path.join(out, "gt_k%d.npy" % K), ids[:, :K].astype(np.int32))


if __name__ == "__main__":
    outroot = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")), os.path.join(ROOT, "data"))
    main([a for a in sys.argv[1:] if not a.startswith("--")][0], outroot)

#!/usr/bin/env python
"""QPS-recall sweep on one GPU (the curve behind bench.py's operating point).

For every (nprobe, schedule, mode[, K]) point: recall@10 (and @K) against the
fp64 ground truth, device-resident QPS (CUDA events, mean of --steps
asynchronous searches, L2 flushed in between), and the per-query survivor
counts.  Usage:
  python scripts/sweep.py --config sift [--d 64] [--steps 5] > profiles/r01_sweep_sift.json
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="sift")
    ap.add_argument("--d", type=int, default=0)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--nprobe", default="16,24,32,48,64,96,128,192,256")
    ap.add_argument("--K", default="10")
    ap.add_argument("--modes", default="FULL/TIGHT,FULL/LOOSE,STAGE1_ONLY/TIGHT")
    # SURVEY NEXT-2 parameter sweeps: every combination is a point
    ap.add_argument("--eps0", default="1.9")
    ap.add_argument("--m", default="4")
    ap.add_argument("--rscale", default="2")
    args = ap.parse_args()
    import torch
    import bench
    import paper_2411_06158_b200 as mrq
    import synth
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    d = args.d or {"tiny": 16, "sift": 64, "gist": 128}.get(args.config, 64)
    bfile = os.path.join(ROOT, "data", args.config, "build_d%d.mrqb" % d)
    cfg = synth.config_by_name(args.config)
    X, Q = synth.generate(cfg, device="cuda")
    h = mrq.mrq_index_load(bfile, X, d, device=0)
    nq = Q.shape[0]
    dq = torch.from_numpy(Q).to(dev)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    out = {"workload": bench.WORKLOADS.get(args.config, args.config), "d": d, "points": []}
    for K in [int(x) for x in args.K.split(",")]:
        gtf = os.path.join(ROOT, "data", args.config, "gt_k%d.npy" % K)
        gt10 = np.load(os.path.join(ROOT, "data", args.config, "gt_k10.npy"))
        gt100 = os.path.join(ROOT, "data", args.config, "gt_k100.npy")
        gtK = np.load(gtf) if os.path.exists(gtf) else (np.load(gt100)[:, :K] if os.path.exists(gt100) and K < 100
                                                       else None)   # exact KNN lists are sorted: a prefix
        d_ids = torch.empty((nq, K), dtype=torch.int64, device=dev)
        d_dist = torch.empty((nq, K), dtype=torch.float32, device=dev)
        for mt in args.modes.split(","):
            mode, tau = mt.split("/")
            grid = [(npb, e0, mm, rs) for npb in [int(x) for x in args.nprobe.split(",")]
                    for e0 in [float(x) for x in args.eps0.split(",")] for mm in [float(x) for x in args.m.split(",")]
                    for rs in [float(x) for x in args.rscale.split(",")]]
            for npb, e0, mm, rs in grid:
                if npb > cfg.k:
                    continue
                p = mrq.SearchParams.make(K=K, nprobe=npb, mode=mode, tau_schedule=tau, seed_lists=2, eps0=e0, m=mm,
                                          resid_scale=rs)
                st = mrq.Stats()
                mrq.mrq_search_batch_device(h, dq, p, d_ids, d_dist, st, stream.cuda_stream)
                ids = d_ids.cpu().numpy()
                for _ in range(2):
                    mrq.mrq_search_batch_device(h, dq, p, d_ids, d_dist, None, stream.cuda_stream)
                ev = []
                for i in range(args.steps):
                    flush.fill_(float(i))
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    mrq.mrq_search_batch_device(h, dq, p, d_ids, d_dist, None, stream.cuda_stream)
                    b.record(stream)
                    ev.append((a, b))
                torch.cuda.synchronize()
                ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
                pt = {"K": K, "mode": mode, "tau_schedule": tau, "nprobe": npb, "eps0": e0, "m": mm,
                      "resid_scale": rs, "ms": round(ms, 4),
                      "qps": round(nq / (ms * 1e-3), 1), "recall10": round(bench.recall_at_k(ids, gt10, 10), 4),
                      "f1_per_q": round(st.stage1_pass / nq, 1), "f2_per_q": round(st.stage2_pass / nq, 1),
                      "exact_per_q": round(st.exact / nq, 1), "scanned_per_q": round(st.scanned / nq, 1)}
                if gtK is not None and K > 10:
                    pt["recall%d" % K] = round(bench.recall_at_k(ids, gtK, K), 4)
                out["points"].append(pt)
                print(json.dumps(pt), file=sys.stderr, flush=True)
    mrq.mrq_free(h)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

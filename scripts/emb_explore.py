"""Embedding-shaped workload (BASELINE.json configs[4]: N = 5M, Q = 10k,
D = 1536, d = 256 | 512, k = 16384) on one GPU: the QPS-recall grid over
nprobe, mode, tau schedule and the Chebyshev multiplier m (Eq.7).
The index comes from the GPU builder (mrq_build_gpu); recall against the
committed fp64 ground truth (scripts/gt_gpu.py, cross-checked against
oracle.bruteforce).  One JSON line per point on stdout.
  python scripts/emb_explore.py --d 512 > gpurun_out/emb_explore.jsonl
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=512)
    ap.add_argument("--grid", default="full")
    args = ap.parse_args()
    import torch
    import synth
    import paper_2411_06158_b200 as m
    cfg = synth.config_by_name("emb")
    t = time.time()
    X, Q = synth.generate(cfg, device="cuda")
    print(json.dumps({"event": "generated", "s": round(time.time() - t, 1)}), flush=True)
    bfile = "/tmp/mrq_emb_d%d.mrqb" % args.d
    t = time.time()
    binfo = m.mrq_build_gpu(X, args.d, cfg.k, bfile, device=0)
    print(json.dumps({"event": "built", "s": round(time.time() - t, 1), **binfo}), flush=True)
    h = m.mrq_index_load(bfile, X, args.d, device=0)
    gt = np.load(os.path.join(ROOT, "data", "emb", "gt_k10.npy"))
    dev = torch.device("cuda", 0)
    nq, K = Q.shape[0], 10
    dq = torch.from_numpy(Q).to(dev)
    ids = torch.empty((nq, K), dtype=torch.int64, device=dev)
    dist = torch.empty((nq, K), dtype=torch.float32, device=dev)
    s = torch.cuda.Stream(dev)

    def point(npb, mode="FULL", tau="LOOSE", mm=4.0, eps0=1.9, rs=2.0):
        p = m.SearchParams.make(K=K, nprobe=npb, mode=mode, tau_schedule=tau, m=mm, eps0=eps0, resid_scale=rs,
                                seed_lists=2)
        st = m.Stats()
        m.mrq_search_batch_device(h, dq, p, ids, dist, st, s.cuda_stream)
        torch.cuda.synchronize()
        f = ids.cpu().numpy()
        rc = sum(len(set(a.tolist()) & set(b.tolist())) for a, b in zip(f, gt)) / gt.size
        evs = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            m.mrq_search_batch_device(h, dq, p, ids, dist, None, s.cuda_stream)
            b.record(s)
            evs.append((a, b))
        torch.cuda.synchronize()
        ms = float(np.median([a.elapsed_time(b) for a, b in evs]))
        out = {"d": args.d, "nprobe": npb, "mode": mode, "tau": tau, "m": mm, "eps0": eps0, "rscale": rs,
               "recall10": round(rc, 4), "ms": round(ms, 3), "qps": round(nq / ms * 1e3, 1),
               "f1_per_q": round(st.stage1_pass / nq, 1), "f2_per_q": round(st.stage2_pass / nq, 1),
               "exact_per_q": round(st.exact / nq, 1), "scanned_per_q": round(st.scanned / nq, 1),
               "stage_ms": {k: round(getattr(st, k), 3) for k in ("ms_probe", "ms_seed", "ms_scan", "ms_head",
                                                                 "ms_topk")}}
        print(json.dumps(out), flush=True)
        return out

    if args.grid == "quick":   # np = 16 with both query-order keys (mrq_debug_set qorder = 1 | 2)
        for qo in (1, 2):
            m.mrq_debug_set(h, "qorder", qo)
            print(json.dumps({"event": "qorder", "value": qo}), flush=True)
            point(16, mode="EXACT")
            for mm in (8.0, 16.0):
                point(16, "FULL", "LOOSE", mm)
            point(16, "FULL", "TIGHT", 16.0)
        m.mrq_free(h)
        return
    for npb in (16, 32, 64, 128):
        point(npb, mode="EXACT")
    for npb in (16, 32, 64):
        for mm in (4.0, 8.0, 16.0, 32.0):
            point(npb, "FULL", "LOOSE", mm)
        point(npb, "FULL", "TIGHT", 16.0)
        point(npb, "STAGE1_ONLY", "LOOSE", 16.0)
    m.mrq_free(h)


if __name__ == "__main__":
    main()

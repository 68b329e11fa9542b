"""Upper-bound experiment for a chunked, multi-stream search (GPU box):
C independent index handles over the same base, each searching 1/C of the
query batch on its own stream, against one handle searching all of it.

  python scripts/concurrency_probe.py [config] [C,...]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2411_06158_b200 as m  # noqa: E402


def main():
    import torch
    cfgname = sys.argv[1] if len(sys.argv) > 1 else "deep"
    Cs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,3,4").split(",")]
    d = {"deep": 64, "sift": 64, "gist": 128, "tiny": 16}[cfgname]
    cfg = synth.config_by_name(cfgname)
    X, Q = synth.generate(cfg, device="cuda")
    path = os.path.join(ROOT, "data", cfgname, "build_d%d.mrqb" % d)
    H = [m.mrq_index_load(path, X, d, device=0) for _ in range(max(Cs))]
    nq = Q.shape[0]
    dq = torch.as_tensor(Q).cuda().contiguous() if not isinstance(Q, torch.Tensor) else Q.contiguous()
    K = 10
    p = m.SearchParams.make(K=K, nprobe=16, tau_schedule="LOOSE", seed_lists=2, seed_mult=2)
    ids = torch.empty((nq, K), dtype=torch.int64, device="cuda")
    dist = torch.empty((nq, K), dtype=torch.float32, device="cuda")
    prio = os.environ.get("PRIO")
    streams = [torch.cuda.Stream(priority=(-1 if (prio and i % 2 == 0) else 0)) for i in range(max(Cs))]
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for C in Cs:
        bounds = [nq * i // C for i in range(C + 1)]
        views = [(dq[bounds[i]:bounds[i + 1]], ids[bounds[i]:bounds[i + 1]], dist[bounds[i]:bounds[i + 1]])
                 for i in range(C)]
        main_s = torch.cuda.current_stream()
        times = []
        for rep in range(12):
            flush.fill_(rep & 255)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(main_s)
            for i in range(C):
                streams[i].wait_stream(main_s)
            for i in range(C):
                q_, i_, d_ = views[i]
                m.mrq_search_batch_device(H[i], q_, p, i_, d_, None, streams[i].cuda_stream)
            for i in range(C):
                main_s.wait_stream(streams[i])
            b.record(main_s)
            torch.cuda.synchronize()
            if rep >= 4:
                times.append(a.elapsed_time(b))
        print("C=%d chunks: %.4f ms median (min %.4f) -> %.2fM QPS" %
              (C, float(np.median(times)), min(times), nq / np.median(times) / 1e3), flush=True)
    for h in H:
        m.mrq_free(h)


if __name__ == "__main__":
    main()

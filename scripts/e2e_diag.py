"""Where the host-buffer (e2e) search time goes, Deep-shaped batch (GPU box):
the full mrq_search_batch call vs its parts (H2D of the queries, the device
search, D2H of ids + distances), wall clock, medians of 20."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2411_06158_b200 as m  # noqa: E402
from paper_2411_06158_b200 import mrq  # noqa: E402


def med(f, n=20):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize()
        t = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    return 1e3 * float(np.median(ts))


cfg = synth.config_by_name("deep")
X, Q = synth.generate(cfg, device="cuda")
h = mrq.mrq_index_load(os.path.join(ROOT, "data", "deep", "build_d64.mrqb"), X, 64)
nq, K = Q.shape[0], 10
p = mrq.SearchParams.make(K=K, nprobe=16, tau_schedule="LOOSE", seed_lists=2, seed_mult=2)
hq = torch.from_numpy(Q).pin_memory()
hi = torch.empty((nq, K), dtype=torch.int64).pin_memory()
hd = torch.empty((nq, K), dtype=torch.float32).pin_memory()
dq = hq.cuda()
di = torch.empty((nq, K), dtype=torch.int64, device="cuda")
dd = torch.empty((nq, K), dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
for _ in range(3):
    mrq.mrq_search_batch(h, hq.numpy(), p, with_stats=False, out_ids=hi.numpy(), out_dist=hd.numpy())
    mrq.mrq_search_batch_device(h, dq, p, di, dd, None, s.cuda_stream)
print("host call (H2D + search + D2H + sync): %.3f ms" % med(
    lambda: mrq.mrq_search_batch(h, hq.numpy(), p, with_stats=False, out_ids=hi.numpy(), out_dist=hd.numpy())))
print("device call + sync:                    %.3f ms" % med(
    lambda: mrq.mrq_search_batch_device(h, dq, p, di, dd, None, s.cuda_stream)))
print("H2D %d B (pinned):                 %.3f ms" % (Q.nbytes, med(lambda: dq.copy_(hq, non_blocking=True))))
print("D2H %d B (pinned):                  %.3f ms" % (hi.numel() * 12, med(
    lambda: (hi.copy_(di, non_blocking=True), hd.copy_(dd, non_blocking=True)))))
print("python wrapper + ctypes, nq = 0:       %.3f ms" % med(
    lambda: mrq.mrq_search_batch(h, hq.numpy()[:0], p, with_stats=False)))
flush = torch.empty(512 << 18, dtype=torch.float32, device="cuda")   # 512 MB (> L2), as bench.py


def flushed(f):
    def g():
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t = time.perf_counter()
        f()
        torch.cuda.synchronize()
        return time.perf_counter() - t
    return 1e3 * float(np.median([g() for _ in range(20)]))


print("host call after an L2 flush:           %.3f ms" % flushed(
    lambda: mrq.mrq_search_batch(h, hq.numpy(), p, with_stats=False, out_ids=hi.numpy(), out_dist=hd.numpy())))
print("device call + sync after an L2 flush:  %.3f ms" % flushed(
    lambda: mrq.mrq_search_batch_device(h, dq, p, di, dd, None, s.cuda_stream)))
mrq.mrq_free(h)

"""Probe-stage diagnostics on a workload (GPU box): per-stage times of a few
searches and the fused probe's append statistics (thresholds, appended
values per row, margin-set sizes).

  BOUND_T=32,64,128 python scripts/probe_diag.py [config] [nprobe]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2411_06158_b200 as m  # noqa: E402


def parts(nq, k, G=148):
    """mrq_probe_tc_parts: parts per query row of the fused probe."""
    mb_n, nt = (nq + 127) // 128, (k + 255) // 256
    U = mb_n * nt
    G = max(1, min(G, U, 7 * mb_n))

    def u0(i):
        return i * U // G

    def owner(u):
        i = u * G // U
        while i + 1 < G and u0(i + 1) <= u:
            i += 1
        while i > 0 and u0(i) > u:
            i -= 1
        return i
    return 2 * max(owner((mb + 1) * nt - 1) - owner(mb * nt) + 1 for mb in range(mb_n))


def main():
    cfgname = sys.argv[1] if len(sys.argv) > 1 else "deep"
    nprobe = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    d = {"deep": 64, "sift": 64, "gist": 128, "tiny": 16}[cfgname]
    cfg = synth.config_by_name(cfgname)
    t = time.time()
    X, Q = synth.generate(cfg, device="cuda")
    print("generated in %.1fs" % (time.time() - t), flush=True)
    gx = m.Index(os.path.join(ROOT, "data", cfgname, "build_d%d.mrqb" % d), X, d)
    nq = Q.shape[0]
    P = parts(nq, gx.info["k"])
    for kv in filter(None, os.environ.get("SET", "").split(",")):   # SET=name=value,... (mrq_debug_set)
        k_, v_ = kv.split("=")
        m.mrq_debug_set(gx.h, k_, int(v_))
    import torch
    torch.cuda.profiler.start()   # ncu --profile-from-start off: only the searches below are profiled
    for T in [int(x) for x in os.environ.get("BOUND_T", "64").split(",")]:
        try:
            m.mrq_debug_set(gx.h, "probe_bound_T", T)
        except Exception:   # noqa: BLE001
            pass
        print("== probe_bound_T", T)
        for _ in range(4):
            _, _, st = gx.search(Q, K=10, nprobe=nprobe, tau_schedule="LOOSE", seed_lists=2, seed_mult=int(os.environ.get("SEED_MULT", "3")))
            print("probe %.4f gemm %.4f finish %.4f total %.4f" % (st.ms_probe, st.ms_probe_gemm,
                                                                  st.ms_probe - st.ms_probe_gemm, st.ms_total),
                  flush=True)
        ncand = gx.fetch("probe_ncand", "u32")
        print("margin set per row: mean %.1f max %d" % (ncand.mean(), ncand.max()))
        try:
            ccnt = gx.fetch("probe_ccnt", "u32")[:nq * P]
            tot = ccnt.reshape(nq, P).astype(np.int64).sum(1)
            print("parts per row %d; appended per row: mean %.1f p50 %d p99 %d max %d; part max %d" %
                  (P, tot.mean(), np.percentile(tot, 50), np.percentile(tot, 99), tot.max(), ccnt.max()))
        except Exception as e:   # noqa: BLE001
            print("no probe_ccnt:", e)
    torch.cuda.profiler.stop()
    gx.close()


if __name__ == "__main__":
    main()

"""GPU <-> oracle parity, stage by stage, through the C ABI (-m gpu).

Both sides read the same oracle build file (BASELINE.json north_star) and the
same seeded base/queries.  Bar: codes, bit-planes,
probe lists, flag sets (F1, F2, S0, S1) and returned ids are compared
bit-exactly; because both sides follow the canonical fp64 order, the fp64
intermediates (q_p, constants, dis', LB1, tau0, tau1, exact distances) are
also compared bit-exactly, which is stricter than north_star's 1e-4
relative distance tolerance (asserted as well, separately).
"""
import os

import numpy as np
import pytest

import oracle
import synth
from oracle import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _gpu():
    import paper_2411_06158_b200 as m
    return m


CASES = {
    # name: (config, N, Q, D, d, k, nprobe list, committed build file or None)
    "tiny": ("tiny", None, None, None, 16, 16, (1, 4, 16), "data/tiny/build_d16.mrqb"),
    "sift50k": ("sift", 50_000, 64, 128, 64, 256, (8, 32), None),
    "deep_d48": ("deep", 20_000, 48, 96, 48, 64, (5, 16), None),
    "gist_small": ("gist", 8_000, 24, 960, 128, 32, (4,), None),
    "gist_d256": ("gist", 6_000, 16, 960, 256, 24, (3, 24), None),        # W = 8 code words
    "emb_d512": ("emb", 5_000, 12, 1536, 512, 16, (2, 16), None),         # W = 16, D = 1536
    # k = 2048, Q = 300: the tcgen05 probe's 8 column tiles per 128-query block
    # are split over several CTAs ("parts"), 3 query blocks, a ragged last one
    "sift_k2048": ("sift", 100_000, 300, 128, 64, 2048, (16, 40), None),
    # d = D: no residual (tails of width 0, eps_r = 0), one ragged code word
    "tiny_dD": ("tiny", 4_000, 40, 24, 24, 8, (2, 8), None),
}


@pytest.fixture(scope="module", params=list(CASES))
def case(request, tmp_path_factory):
    name = request.param
    cfgname, N, Q, D, d, k, nps, bfile = CASES[name]
    cfg = synth.config_by_name(cfgname)
    X, Qv = synth.generate(cfg, N=N, Q=Q, D=D)
    if bfile:
        path = os.path.join(ROOT, bfile)
        bf = B.read(path)
    else:
        bf = B.build(X, d, k)
        path = str(tmp_path_factory.mktemp("bf") / (name + ".mrqb"))
        B.write(path, bf)
    ox = oracle.Index(bf, X)
    m = _gpu()
    gx = m.Index(path, X, d)
    yield dict(name=name, X=X, Q=Qv, bf=bf, ox=ox, gx=gx, d=d, nprobe=nps, m=m)
    gx.close()


def _slot_to_id(gx):
    return gx.fetch("ids", "u32").astype(np.int64)


def test_encode_bit_exact(case):
    """a0: Alg.1 L3-L8 on the GPU equals the oracle bit for bit."""
    gx, ox, d = case["gx"], case["ox"], case["d"]
    ids = _slot_to_id(gx)
    npad = gx.info["npad"]
    W = (d + 31) // 32
    valid = ids != 0xFFFFFFFF
    sid = ids[valid]
    codes = gx.fetch("codes", "u32").reshape(W, npad)[:, valid].T
    assert np.array_equal(codes, ox.code[sid])
    for nm, ref in (("f1", ox.f1), ("f2", ox.f2), ("f3", ox.f3), ("xr2", ox.xr2f)):
        got = gx.fetch(nm, "f32")[valid]
        assert np.array_equal(got.view(np.uint32), ref[sid].view(np.uint32)), nm
    heads = gx.fetch("heads", "f32").reshape(npad, d)[valid]
    assert np.array_equal(heads, ox.head[sid])
    D = ox.D
    if D > d:
        tails = gx.fetch("tails", "f32").reshape(npad, D - d)[valid]
        assert np.array_equal(tails, ox.tail[sid])
    # inverted lists: same members, ascending ids inside each list (A-28)
    off = gx.fetch("list_off", "u32").astype(np.int64)
    size = gx.fetch("list_size", "u32").astype(np.int64)
    for c in range(ox.k):
        got = ids[off[c]:off[c] + size[c]]
        assert np.array_equal(got, ox.list_ids[ox.list_off[c]:ox.list_off[c + 1]])
        assert off[c] % 4 == 0
    assert np.array_equal(gx.fetch("Rc", "f64").reshape(ox.k, d), ox.Rc)


def _search_both(case, nprobe, K=10, mode="FULL", tau="TIGHT", **kw):
    gx, ox, Q = case["gx"], case["ox"], case["Q"]
    m = case["m"]
    m.mrq_debug_set(gx.h, "dump_dis", 1)
    gi, gd, gst = gx.search(Q, K=K, nprobe=nprobe, mode=mode, tau_schedule=tau, **kw)
    oi, od, ost, dp = ox.search(Q, K=K, nprobe=nprobe, mode=mode, tau_schedule=tau, dump=True, **kw)
    return gi, gd, gst, oi, od, ost, dp


def _segments(gx, nq, cnt_name, pos_name, extra=None):
    off = gx.fetch("f1_off", "u64").astype(np.int64)
    cnt = gx.fetch(cnt_name, "u32").astype(np.int64)
    pos = gx.fetch(pos_name, "u32").astype(np.int64)
    ex = gx.fetch(extra, "f64") if extra else None
    ids = _slot_to_id(gx)
    out = []
    for q in range(nq):
        sl = pos[off[q]:off[q] + cnt[q]]
        v = ex[off[q]:off[q] + cnt[q]] if ex is not None else None
        out.append((ids[sl], v))
    return out


@pytest.mark.parametrize("tau", ["TIGHT", "LOOSE"])
@pytest.mark.parametrize("seed_lists,seed_mult", [(1, 2), (2, 3), (4, 4)])   # (2, 3): bench.py's operating point
def test_stagewise_parity(case, tau, seed_lists, seed_mult):
    gx, ox, Q = case["gx"], case["ox"], case["Q"]
    nq, D, d = Q.shape[0], ox.D, case["d"]
    for npb in case["nprobe"]:
        gi, gd, gst, oi, od, ost, dp = _search_both(case, npb, tau=tau, seed_lists=seed_lists, seed_mult=seed_mult)
        npe = min(npb, ox.k)
        # a1 query projection, residual constants
        assert np.array_equal(gx.fetch("qp", "f64").reshape(nq, D), dp["qp"])
        assert np.array_equal(gx.fetch("qr2", "f64"), dp["qr2"])
        assert np.array_equal(gx.fetch("eps_r", "f64"), dp["eps_r"])
        # a2 probe: identical lists in identical order, bit-exact ||q_d - c||^2
        assert np.array_equal(gx.fetch("probe", "u32").reshape(nq, npe).astype(np.int64), dp["probe"])
        assert np.array_equal(gx.fetch("probe_qn2", "f64").reshape(nq, npe), dp["probe_qn2"])
        # a3 quantization: bit-planes reproduce the oracle's levels; constants bit-exact
        W = (d + 31) // 32
        planes = gx.fetch("planes", "u32").reshape(nq, npe, 4, W)
        j = np.arange(d)
        lev = np.zeros((nq, npe, d), np.int64)
        for b in range(4):
            lev += (((planes[:, :, b, j // 32] >> (j % 32).astype(np.uint32)) & 1).astype(np.int64)) << b
        assert np.array_equal(lev, dp["levels"].astype(np.int64))
        qc = gx.fetch("qconst", "f64").reshape(nq, npe, 8)[:, :, :5]
        assert np.array_equal(qc, dp["qconst"])
        # a5 scan: dis' and LB1 of every candidate bit-exact (and within 1e-4 rel), tau0, F1 sets
        off = gx.fetch("f1_off", "u64").astype(np.int64)
        dis = gx.fetch("dbg_dis", "f64")
        lb1 = gx.fetch("dbg_lb1", "f64")
        for q in range(nq):
            n = dp["scan_cnt"][q]
            assert off[q + 1] - off[q] == n
            assert np.array_equal(dis[off[q]:off[q] + n], dp["scan_dis"][q, :n])
            assert np.array_equal(lb1[off[q]:off[q] + n], dp["scan_lb1"][q, :n])
            rel = np.abs(dis[off[q]:off[q] + n] - dp["scan_dis"][q, :n]) / np.maximum(np.abs(dp["scan_dis"][q, :n]), 1e-30)
            assert np.all(rel <= 1e-4)
        assert np.array_equal(gx.fetch("tau0", "f64"), dp["tau0"])
        f1 = _segments(gx, nq, "f1_cnt", "f1_pos")
        for q in range(nq):
            assert sorted(f1[q][0].tolist()) == sorted(dp["f1_ids"][q, :dp["f1_cnt"][q]].tolist())
        # a4 seeds
        s0c = gx.fetch("s0_cnt", "u32")
        Kp = 10 * seed_mult
        s0p = gx.fetch("s0_pos", "u32").reshape(nq, Kp)
        ids = _slot_to_id(gx)
        for q in range(nq):
            assert s0c[q] == dp["s0_cnt"][q]
            assert sorted(ids[s0p[q, :s0c[q]]].tolist()) == sorted(dp["s0_ids"][q, :s0c[q]].tolist())
        # a6 stage 2: tau1 and F2 sets
        assert np.array_equal(gx.fetch("tau1", "f64"), dp["tau1"])
        f2 = _segments(gx, nq, "f2_cnt", "f2_pos", "f2_exact")
        for q in range(nq):
            oid = dp["f2_ids"][q, :dp["f2_cnt"][q]]
            oex = dp["f2_exact"][q, :dp["f2_cnt"][q]]
            gid, gex = f2[q]
            assert sorted(gid.tolist()) == sorted(oid.tolist())
            # a7 exact distances bit-exact
            o = dict(zip(oid.tolist(), oex.tolist()))
            assert all(o[i] == v for i, v in zip(gid.tolist(), gex.tolist()))
        # a8 top-K: identical ids and fp32 distances
        assert np.array_equal(gi, oi)
        assert np.array_equal(gd.view(np.uint32), od.view(np.uint32))
        assert gst.scanned == ost["scanned"]
        assert gst.stage1_pass == ost["f1"] and gst.stage2_pass == ost["f2"] and gst.exact == ost["exact"]


@pytest.mark.parametrize("mode", ["STAGE1_ONLY", "EXACT"])
def test_modes_parity(case, mode):
    npb = case["nprobe"][-1]
    gi, gd, gst, oi, od, ost, dp = _search_both(case, npb, mode=mode)
    assert np.array_equal(gi, oi)
    assert np.array_equal(gd.view(np.uint32), od.view(np.uint32))
    assert gst.exact == ost["exact"]


@pytest.mark.parametrize("K", [1, 100])
def test_k_edge_parity(case, K):
    gi, gd, gst, oi, od, ost, dp = _search_both(case, case["nprobe"][0], K=K)
    assert np.array_equal(gi, oi)
    assert np.array_equal(gd.view(np.uint32), od.view(np.uint32))


def test_probe_all_lists_and_padding(case):
    """nprobe = k (every list) and K larger than the candidate count (-1/+inf padding)."""
    ox = case["ox"]
    k = min(ox.k, 1024)
    gi, gd, gst, oi, od, ost, dp = _search_both(case, k, K=10)
    assert np.array_equal(gi, oi)
    small = case["Q"][:3]
    for mode in ("EXACT", "FULL"):
        g = case["gx"].search(small, K=1024, nprobe=1, mode=mode)
        o = ox.search(small, K=1024, nprobe=1, mode=mode)
        assert np.array_equal(g[0], o[0])
        assert np.array_equal(g[1].view(np.uint32), o[1].view(np.uint32))
        pad = g[0] < 0
        assert pad.any() and np.all(np.isinf(g[1][pad]))


def test_empty_batch_and_errors(case):
    m, gx = case["m"], case["gx"]
    ids, dist, st = gx.search(np.zeros((0, case["ox"].D), np.float32), K=10, nprobe=4)
    assert ids.shape == (0, 10)
    with pytest.raises(m.MRQError) as e:
        gx.search(case["Q"][:2], K=0, nprobe=4)
    assert e.value.code == -1
    with pytest.raises(m.MRQError) as e:
        gx.search(case["Q"][:2], K=10, nprobe=case["ox"].k + 1)
    assert e.value.code == -1


def test_probe_tensor_core_screen_bound(case):
    """The tcgen05 3xTF32 screen a_c = ||c||^2 - 2<q_d, c> stays within the proven
    delta_q = kappa (||q_d|| + max||c||)^2 of the exact key, and
    the CUDA-core screen gives the same probe lists (both are rescored exactly)."""
    gx, bf = case["gx"], case["bf"]
    d, k = case["d"], bf.k
    Q = case["Q"]
    np_ = min(case["nprobe"][-1], k)
    m = case["m"]
    m.mrq_debug_set(gx.h, "probe_unfused", 1)     # the screen goes to HBM ("approx") for inspection
    g1 = gx.search(Q, K=10, nprobe=np_)
    approx = gx.fetch("approx", "f32").reshape(Q.shape[0], k).astype(np.float64)
    qp = gx.fetch("qp", "f64").reshape(Q.shape[0], -1)[:, :d]
    C = bf.C.astype(np.float64)
    key = (C * C).sum(1)[None, :] - 2.0 * qp @ C.T
    cmax = np.sqrt((C * C).sum(1).max())
    kappa = 2.0 ** -20 + 3 * d * 2.0 ** -23      # 3xTF32 screen (mrq_probe_tc.cu header)
    bound = kappa * (np.sqrt((qp * qp).sum(1)) + cmax) ** 2
    err = np.abs(approx - key)
    assert np.all(err <= bound[:, None]), float((err / bound[:, None]).max())
    probe_tc = gx.fetch("probe", "u32").copy()
    m.mrq_debug_set(gx.h, "cuda_core_probe", 1)
    g2 = gx.search(Q, K=10, nprobe=np_)
    m.mrq_debug_set(gx.h, "cuda_core_probe", 0)
    assert np.array_equal(probe_tc, gx.fetch("probe", "u32"))
    assert np.array_equal(g1[0], g2[0]) and np.array_equal(g1[1], g2[1])
    m.mrq_debug_set(gx.h, "probe_unfused", 0)     # fused screen + running top-np (np <= 16, np <= 64)
    for npb in sorted({1, min(np_, 16), min(16, k), min(24, k), min(64, k)}):
        m.mrq_debug_set(gx.h, "probe_unfused", 1)
        gu = gx.search(Q, K=10, nprobe=npb)
        pu = gx.fetch("probe", "u32").copy()
        m.mrq_debug_set(gx.h, "probe_unfused", 0)
        gf = gx.search(Q, K=10, nprobe=npb)
        assert np.array_equal(pu, gx.fetch("probe", "u32")), npb
        assert np.array_equal(gu[0], gf[0]) and np.array_equal(gu[1], gf[1])


def test_graph_replay_identical(case):
    """Repeated searches replay a captured CUDA graph (search_dispatch); every
    replay, and a parameter change (re-capture), gives the graph-free result."""
    m, gx, Q = case["m"], case["gx"], case["Q"]
    npb = case["nprobe"][-1]
    m.mrq_debug_set(gx.h, "graphs", 0)
    ref = {}
    for tau in ("TIGHT", "LOOSE"):
        ref[tau] = m.mrq_search_batch(gx.h, Q, m.SearchParams.make(K=10, nprobe=npb, tau_schedule=tau),
                                      with_stats=False)[:2]
    m.mrq_debug_set(gx.h, "graphs", 1)
    for tau in ("TIGHT", "LOOSE", "TIGHT"):
        for _ in range(3):   # plain run, capture, replay
            ids, dist, _ = m.mrq_search_batch(gx.h, Q, m.SearchParams.make(K=10, nprobe=npb, tau_schedule=tau),
                                              with_stats=False)
            assert np.array_equal(ids, ref[tau][0]) and np.array_equal(dist, ref[tau][1])


def test_host_resident_tails_identical(case):
    """MRQ_LOAD_TAILS_HOST (the memory-limited setting of P:296):
    tails in mapped pinned host memory give the oracle's results bit for bit
    (and the HBM-resident run's counters)."""
    m, gx, ox, Q = case["m"], case["gx"], case["ox"], case["Q"]
    gh = m.Index(gx.build_file, case["X"], case["d"], tails_host=True)
    try:
        for tau in ("TIGHT", "LOOSE"):
            a = gx.search(Q, K=10, nprobe=case["nprobe"][-1], tau_schedule=tau)
            b = gh.search(Q, K=10, nprobe=case["nprobe"][-1], tau_schedule=tau)
            o = ox.search(Q, K=10, nprobe=case["nprobe"][-1], tau_schedule=tau)
            assert np.array_equal(b[0], o[0]) and np.array_equal(b[1].view(np.uint32), o[1].view(np.uint32))
            assert b[2].exact == o[2]["exact"] and b[2].stage2_pass == o[2]["f2"]
            assert a[2].exact == b[2].exact and a[2].stage2_pass == b[2].stage2_pass
    finally:
        gh.close()


def test_query_order_invariance(case):
    """The list-locality processing order (a permutation of the queries: 1 =
    key from three principal coordinates, k_qorder; 2 = key of the nearest
    probed list, k_cand_count + k_offsets_order, the default) changes no
    result: ids, distances, tau0/tau1 and every survivor count equal the
    identity order's, for both schedules and K = 1 / 10 / 100; the order is a
    permutation, sorted by its key, and the mode-2 key is the locality key of
    probe[q][0] (one key per list, every key < 4096)."""
    m, gx, Q = case["m"], case["gx"], case["Q"]
    npb = case["nprobe"][-1]
    nq = Q.shape[0]
    try:
        for tau in ("TIGHT", "LOOSE"):
            for K in (1, 10, 100):
                res = []
                for on in (0, 1, 2):
                    m.mrq_debug_set(gx.h, "qorder", on)
                    ids, dist, st = gx.search(Q, K=K, nprobe=npb, tau_schedule=tau)
                    res.append((ids, dist, st, gx.fetch("tau0", "f64").copy(), gx.fetch("tau1", "f64").copy()))
                    if on:
                        order = gx.fetch("qorder", "u32")[:nq].astype(np.int64)
                        key = gx.fetch("qkey", "u16")[:nq].astype(np.int64)
                        assert np.array_equal(np.sort(order), np.arange(nq))
                        assert np.all(np.diff(key[order]) >= 0) and key.max() < 4096
                    if on == 2:
                        top1 = gx.fetch("probe", "u32").reshape(nq, -1)[:, 0].astype(np.int64)
                        for c in np.unique(top1):          # one key per list
                            assert len(np.unique(key[top1 == c])) == 1
                a = res[0]
                for b in res[1:]:
                    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
                    assert np.array_equal(a[3], b[3]) and np.array_equal(a[4], b[4])
                    for f in ("scanned", "stage1_pass", "stage2_pass", "exact", "seeds"):
                        assert getattr(a[2], f) == getattr(b[2], f), f
    finally:
        m.mrq_debug_set(gx.h, "qorder", 2)


def test_nocorr_parity(case):
    """mode NOCORR: the K smallest (dis', id) over every
    probed candidate, distance = fp32(dis'); ids and distances bit-exact."""
    gx, ox, Q = case["gx"], case["ox"], case["Q"]
    for npb in case["nprobe"]:
        for K in (1, 10, 100):
            gi, gd, gst = gx.search(Q, K=K, nprobe=npb, mode="NOCORR")
            oi, od, ost = ox.search(Q, K=K, nprobe=npb, mode="NOCORR")
            assert np.array_equal(gi, oi), (npb, K)
            assert np.array_equal(gd.view(np.uint32), od.view(np.uint32)), (npb, K)
            assert gst.scanned == ost["scanned"] and gst.stage1_pass == 0 and gst.exact == 0


def test_graph_replay_survives_scratch_growth(case):
    """A, A (captured), a larger B (scratch reallocated), A
    again must not replay a graph holding freed scratch pointers; every call
    equals the graph-free result."""
    m, gx, Q = case["m"], case["gx"], case["Q"]
    npb = case["nprobe"][0]
    k = case["ox"].k
    QA = Q[: max(1, Q.shape[0] // 3)]
    QB = np.concatenate([Q, Q, Q], 0)
    pa = m.SearchParams.make(K=10, nprobe=npb)
    pb = m.SearchParams.make(K=100, nprobe=min(k, max(npb * 2, npb + 1)))
    m.mrq_debug_set(gx.h, "graphs", 0)
    ra = m.mrq_search_batch(gx.h, QA, pa, with_stats=False)[:2]
    rb = m.mrq_search_batch(gx.h, QB, pb, with_stats=False)[:2]
    m.mrq_debug_set(gx.h, "graphs", 1)
    for qq, pp, ref in ((QA, pa, ra), (QA, pa, ra), (QA, pa, ra), (QB, pb, rb), (QA, pa, ra), (QA, pa, ra),
                        (QB, pb, rb), (QB, pb, rb), (QA, pa, ra)):
        ids, dist, _ = m.mrq_search_batch(gx.h, qq, pp, with_stats=False)
        assert np.array_equal(ids, ref[0]) and np.array_equal(dist, ref[1])


def test_close_twice_and_reload(case):
    """Index.close is idempotent, mrq_free(NULL) is a no-op, and a reloaded
    index gives the same results."""
    m, Q = case["m"], case["Q"]
    a = m.Index(case["gx"].build_file, case["X"], case["d"])
    ia, da, _ = a.search(Q, K=10, nprobe=case["nprobe"][0])
    a.close()
    a.close()
    m.mrq_free(None)
    b = m.Index(case["gx"].build_file, case["X"], case["d"])
    ib, db, _ = b.search(Q, K=10, nprobe=case["nprobe"][0])
    b.close()
    assert np.array_equal(ia, ib) and np.array_equal(da, db)


def test_binding_shape_errors(case):
    import torch
    m, gx, Q = case["m"], case["gx"], case["Q"]
    with pytest.raises(m.MRQError) as e:
        gx.search(Q[:, :-1], K=10, nprobe=2)
    assert e.value.code == -2
    dq = torch.from_numpy(Q).cuda()
    ids = torch.empty((Q.shape[0], 10), dtype=torch.int64, device="cuda")
    dist = torch.empty((Q.shape[0], 10), dtype=torch.float32, device="cuda")
    p = m.SearchParams.make(K=10, nprobe=2)
    with pytest.raises(m.MRQError):
        m.mrq_search_batch_device(gx.h, dq.double(), p, ids, dist)
    with pytest.raises(m.MRQError):
        m.mrq_search_batch_device(gx.h, dq, p, ids[:-1], dist)
    with pytest.raises(m.MRQError):
        m.mrq_search_batch_device(gx.h, dq, m.SearchParams.make(K=10, nprobe=2, seed_mult=1000), ids, dist)
    m.mrq_search_batch_device(gx.h, dq, p, ids, dist)
    torch.cuda.synchronize()


def test_probe_overflow_and_sync_fallbacks(case):
    """Rarely-taken paths give the default results bit for bit: the fused
    probe's candidate-buffer overflow (probe_capp = 1: every centroid is
    rescored) and the candidate scratch sized by the exact device total
    (cand_budget_mb = 0: one D2H + stream sync instead of the host bound)."""
    m, gx, ox, Q = case["m"], case["gx"], case["ox"], case["Q"]
    npb = min(case["nprobe"][0], 16)
    ref = gx.search(Q, K=10, nprobe=npb)
    ref_probe = gx.fetch("probe", "u32").copy()
    oi, od, _ = ox.search(Q, K=10, nprobe=npb)
    assert np.array_equal(ref[0], oi)
    try:
        m.mrq_debug_set(gx.h, "probe_capp", 1)
        a = gx.search(Q, K=10, nprobe=npb)
        assert np.array_equal(gx.fetch("probe", "u32"), ref_probe)
        assert np.array_equal(a[0], ref[0]) and np.array_equal(a[1], ref[1])
        m.mrq_debug_set(gx.h, "probe_capp", 256)
        m.mrq_debug_set(gx.h, "cand_budget_mb", 0)
        for tau in ("TIGHT", "LOOSE"):
            b = gx.search(Q, K=10, nprobe=npb, tau_schedule=tau)
            o = ox.search(Q, K=10, nprobe=npb, tau_schedule=tau)
            assert np.array_equal(b[0], o[0]) and np.array_equal(b[1].view(np.uint32), o[1].view(np.uint32))
    finally:
        m.mrq_debug_set(gx.h, "probe_capp", 256)
        m.mrq_debug_set(gx.h, "cand_budget_mb", 8192)


def test_probe_shared_bound_exact(case):
    """The fused probe's parts share their running np-th smallest (a per-row
    bound): with and without sharing the probe lists and their
    qn2 equal the oracle's exact top-np for every query, at every nprobe of
    the case (the multi-part rows of sift_k2048 included)."""
    m, gx, ox, Q = case["m"], case["gx"], case["ox"], case["Q"]
    try:
        for share in (1, 0):
            m.mrq_debug_set(gx.h, "probe_share", share)
            for npb in case["nprobe"]:
                m.mrq_debug_set(gx.h, "dump_dis", 1)
                gx.search(Q, K=10, nprobe=npb)
                oi, od, ost, dp = ox.search(Q, K=10, nprobe=npb, dump=True)
                npr = min(npb, ox.k)
                nq = Q.shape[0]
                got = gx.fetch("probe", "u32").reshape(nq, npr).astype(np.int64)
                assert np.array_equal(got, dp["probe"]), (share, npb)
                assert np.array_equal(gx.fetch("probe_qn2", "f64").reshape(nq, npr), dp["probe_qn2"]), (share, npb)
                assert np.array_equal(gx.search(Q, K=10, nprobe=npb)[0], oi)
    finally:
        m.mrq_debug_set(gx.h, "probe_share", 1)
        m.mrq_debug_set(gx.h, "dump_dis", 0)


def test_head_sketch_prefilter_exact(case):
    """The int8 head-sketch pre-pass of the stage-2 gather (LOOSE)
    prunes with a proven lower bound of the canonical HEAD, so F2 (as a set,
    with bit-exact exact distances), tau1, the top-K and every counter equal
    the oracle's; the pre-pass must actually prune (survivors < |F1|)."""
    m, gx, ox, Q = case["m"], case["gx"], case["ox"], case["Q"]
    nq = Q.shape[0]
    pruned = 0
    for npb in case["nprobe"]:
        m.mrq_debug_set(gx.h, "dump_dis", 0)
        m.mrq_debug_set(gx.h, "sketch", 1)
        gi, gd, gst = gx.search(Q, K=10, nprobe=npb, tau_schedule="LOOSE")
        surv = gx.fetch("surv_cnt", "u32").astype(np.int64)
        f1c = gx.fetch("f1_cnt", "u32").astype(np.int64)
        f2 = _segments(gx, nq, "f2_cnt", "f2_pos", "f2_exact")
        oi, od, ost, dp = ox.search(Q, K=10, nprobe=npb, tau_schedule="LOOSE", dump=True)
        assert np.array_equal(gi, oi) and np.array_equal(gd.view(np.uint32), od.view(np.uint32))
        assert (gst.stage1_pass, gst.stage2_pass, gst.exact) == (ost["f1"], ost["f2"], ost["exact"])
        assert np.array_equal(gx.fetch("tau1", "f64"), dp["tau1"])
        for q in range(nq):
            oid = dp["f2_ids"][q, :dp["f2_cnt"][q]]
            oex = dict(zip(oid.tolist(), dp["f2_exact"][q, :dp["f2_cnt"][q]].tolist()))
            gid, gex = f2[q]
            assert sorted(gid.tolist()) == sorted(oid.tolist())
            assert all(oex[i] == v for i, v in zip(gid.tolist(), gex.tolist()))
        assert np.all(surv <= f1c) and np.all(surv >= dp["f2_cnt"])
        pruned += int((f1c - surv).sum())
        m.mrq_debug_set(gx.h, "sketch", 0)
        hi, hd, hst = gx.search(Q, K=10, nprobe=npb, tau_schedule="LOOSE")
        m.mrq_debug_set(gx.h, "sketch", 1)
        assert np.array_equal(hi, gi) and np.array_equal(hd, gd) and hst.exact == gst.exact
    assert pruned > 0


@pytest.mark.parametrize("K", [1, 10, 32])
def test_head_topk_fused_equals_oracle(case, K):
    """Stage 2 + exact re-rank + top-K fused in one kernel (k_head_topk: every
    schedule without S1, K <= 32) returns the oracle's ids and distances and
    F2 counts, and the same as the unfused kernels (k_head_b + k_topk_w)."""
    m, gx, ox, Q = case["m"], case["gx"], case["ox"], case["Q"]
    m.mrq_debug_set(gx.h, "dump_dis", 0)
    for mode, tau in (("FULL", "LOOSE"), ("STAGE1_ONLY", "TIGHT"), ("EXACT", "TIGHT")):
        for npb in case["nprobe"]:
            m.mrq_debug_set(gx.h, "fuse_topk", 1)
            gi, gd, gst = gx.search(Q, K=K, nprobe=npb, mode=mode, tau_schedule=tau)
            oi, od, ost = ox.search(Q, K=K, nprobe=npb, mode=mode, tau_schedule=tau)
            assert np.array_equal(gi, oi), (mode, npb)
            assert np.array_equal(gd.view(np.uint32), od.view(np.uint32)), (mode, npb)
            assert gst.exact == ost["exact"]
            if mode == "FULL":
                assert gst.stage2_pass == ost["f2"]
            m.mrq_debug_set(gx.h, "fuse_topk", 0)
            hi, hd, hst = gx.search(Q, K=K, nprobe=npb, mode=mode, tau_schedule=tau)
            assert np.array_equal(hi, gi) and np.array_equal(hd.view(np.uint32), gd.view(np.uint32))
            assert (hst.stage2_pass, hst.exact) == (gst.stage2_pass, gst.exact)
    m.mrq_debug_set(gx.h, "fuse_topk", 1)


def test_exact_mode_any_code_length():
    """mode EXACT reads no code, so any d loads and searches (the d = D index
    of the Exp-2 ablation, with D = 960 > 512): ids and
    distances equal the oracle's; the MRQ modes reject such d with EINVAL."""
    m = _gpu()
    import tempfile
    cfg = synth.config_by_name("gist")
    X, Qv = synth.generate(cfg, N=3_000, Q=20, D=960)
    bf = B.build(X, 960, 12)
    path = os.path.join(tempfile.mkdtemp(), "gist_dD.mrqb")
    B.write(path, bf)
    ox = oracle.Index(bf, X)
    gx = m.Index(path, X, 960)
    try:
        for npb in (1, 4, 12):
            gi, gd, gst = gx.search(Qv, K=10, nprobe=npb, mode="EXACT")
            oi, od, ost = ox.search(Qv, K=10, nprobe=npb, mode="EXACT")
            assert np.array_equal(gi, oi) and np.array_equal(gd.view(np.uint32), od.view(np.uint32)), npb
            assert gst.scanned == ost["scanned"] and gst.exact == ost["exact"]
        for mode in ("FULL", "STAGE1_ONLY", "NOCORR"):
            with pytest.raises(m.MRQError) as e:
                gx.search(Qv, K=10, nprobe=4, mode=mode)
            assert e.value.code == -1
    finally:
        gx.close()


@pytest.mark.parametrize("lm,qg", [(2, 16), (1, 1), (1, 3), (1, 16)])
def test_list_major_scan_equals_oracle(case, lm, qg):
    """The list-major scan (the (query, list) pairs grouped by
    list, a 128-slot tile evaluated against a chunk of its list's queries,
    per-query appends by atomics; lm = 2: the integer inner products S and
    <a, b> of a tile x 8 pairs on the tensor cores, lm = 1: AND+POPC on the
    CUDA cores with qg pairs per unit) produces the oracle's F1 sets (TIGHT:
    f1_pos holds all of F1), the oracle's F2 sets and top-K, and for LOOSE
    sketch survivors between F2 and F1 -- the same as the query-major scan.
    qg = 1 / 3 splits the lists' pairs over many work units."""
    m, gx, ox, Q = case["m"], case["gx"], case["ox"], case["Q"]
    nq, d = Q.shape[0], case["d"]
    if d > 128:
        pytest.skip("list-major scan is for d <= 128")
    m.mrq_debug_set(gx.h, "dump_dis", 0)
    m.mrq_debug_set(gx.h, "scan_lm_qg", qg)
    try:
        for npb in case["nprobe"]:
            oi, od, ost, dp = ox.search(Q, K=10, nprobe=npb, tau_schedule="TIGHT", dump=True)
            m.mrq_debug_set(gx.h, "scan_lm", lm)
            gi, gd, gst = gx.search(Q, K=10, nprobe=npb, tau_schedule="TIGHT")
            assert np.array_equal(gi, oi) and np.array_equal(gd.view(np.uint32), od.view(np.uint32)), npb
            assert (gst.scanned, gst.stage1_pass, gst.stage2_pass) == (ost["scanned"], ost["f1"], ost["f2"])
            f1 = _segments(gx, nq, "f1_cnt", "f1_pos")
            for q in range(nq):
                assert sorted(f1[q][0].tolist()) == sorted(dp["f1_ids"][q, :dp["f1_cnt"][q]].tolist()), (npb, q)
            oi, od, ost, dp = ox.search(Q, K=10, nprobe=npb, tau_schedule="LOOSE", dump=True)
            gi, gd, gst = gx.search(Q, K=10, nprobe=npb, tau_schedule="LOOSE")
            assert np.array_equal(gi, oi) and np.array_equal(gd.view(np.uint32), od.view(np.uint32)), npb
            assert (gst.stage1_pass, gst.stage2_pass, gst.exact) == (ost["f1"], ost["f2"], ost["exact"])
            f2 = _segments(gx, nq, "f2_cnt", "f2_pos")
            for q in range(nq):
                assert sorted(f2[q][0].tolist()) == sorted(dp["f2_ids"][q, :dp["f2_cnt"][q]].tolist()), (npb, q)
            if gst.sketch_pass != gst.stage1_pass:   # the sketch ran: survivors between F2 and F1
                surv = gx.fetch("surv_cnt", "u32").astype(np.int64)
                f1c = gx.fetch("f1_cnt", "u32").astype(np.int64)
                assert np.all(surv <= f1c) and np.all(surv >= dp["f2_cnt"])
                assert np.array_equal(f1c, dp["f1_cnt"].astype(np.int64))
            m.mrq_debug_set(gx.h, "scan_lm", 0)
            hi, hd, hst = gx.search(Q, K=10, nprobe=npb, tau_schedule="LOOSE")
            assert np.array_equal(hi, gi) and np.array_equal(hd.view(np.uint32), gd.view(np.uint32))
            assert (hst.stage1_pass, hst.stage2_pass, hst.exact) == (gst.stage1_pass, gst.stage2_pass, gst.exact)
    finally:
        m.mrq_debug_set(gx.h, "scan_lm", 0)
        m.mrq_debug_set(gx.h, "scan_lm_qg", 16)

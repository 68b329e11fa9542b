"""Multi-rank path.

CPU (-m "not gpu"): the list -> rank plan through the C ABI (host code, no
GPU), on two gloo ranks, and the host all-gather plumbing the virtual-rank
GPU test uses.  GPU (-m gpu): two ranks of a world-2 index as two threads on
one GPU exchanging through the host callback (their kernels never wait on
one another: the exchange blocks on the host) give exactly the world-1
result; a world-1 index forced through the exchange + merge path does too.
"""
import os
import socket
import threading

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    import paper_2411_06158_b200 as m
    from paper_2411_06158_b200 import _build
    _build.build()
    return m


def _sift_like_sizes(k=4096, seed=0):
    rng = np.random.default_rng(seed)
    return rng.gamma(2.0, 122.0, size=k).astype(np.uint32) + 1


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_plan_partition_and_balance(world):
    m = _lib()
    sizes = _sift_like_sizes()
    owner = m.mrq_shard_plan(sizes, world)
    assert owner.shape == sizes.shape and owner.max() < world
    load = np.bincount(owner, weights=sizes.astype(np.float64), minlength=world)
    assert load.sum() == sizes.sum()                      # a partition of all lists
    # greedy LPT: every rank within one (largest) list of the mean
    assert load.max() - load.min() <= sizes.max()
    assert np.array_equal(owner, m.mrq_shard_plan(sizes, world))   # deterministic


def test_shard_plan_ties_and_degenerate():
    m = _lib()
    owner = m.mrq_shard_plan(np.array([5, 5, 5, 5], np.uint32), 2)
    assert owner.tolist() == [0, 1, 0, 1]                  # ties: list id, then least-loaded rank
    assert m.mrq_shard_plan(np.array([7], np.uint32), 4).tolist() == [0]
    with pytest.raises(m.MRQError):
        m.mrq_shard_plan(np.array([1, 2], np.uint32), 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, ROOT)
    import paper_2411_06158_b200 as m
    # every rank derives the plan from the same build-file list sizes
    from oracle import build as B
    bf = B.read(os.path.join(ROOT, "data", "tiny", "build_d16.mrqb"))
    sizes = np.bincount(bf.assign, minlength=bf.k).astype(np.uint32)
    owner = m.mrq_shard_plan(sizes, world)
    plans = [None] * world
    dist.all_gather_object(plans, owner.tolist())
    mine = set(np.nonzero(owner == rank)[0].tolist())
    owned = [None] * world
    dist.all_gather_object(owned, sorted(mine))
    # host all-gather plumbing of the library's exchange callback: rank-major bytes
    payload = bytes([rank]) * 24 * 3
    got = [None] * world
    dist.all_gather_object(got, payload)
    cb_out = b"".join(got)
    out[rank] = (plans, owned, cb_out, int(sizes.sum()))
    dist.destroy_process_group()


def test_shard_plan_two_gloo_ranks():
    world = 2
    port = _free_port()
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.start_processes(_gloo_worker, args=(world, port, out), nprocs=world, start_method="spawn")
    plans0, owned0, cb0, total = out[0]
    plans1, owned1, cb1, _ = out[1]
    assert plans0[0] == plans0[1] == plans1[0] == plans1[1]          # identical plan on every rank
    assert set(owned0[0]).isdisjoint(owned0[1])
    assert sorted(owned0[0] + owned0[1]) == list(range(len(plans0[0])))
    assert cb0 == cb1 == bytes([0]) * 72 + bytes([1]) * 72


# ------------------------------------------------------------------- GPU

class _ThreadExchange:
    """Rank-major all-gather among `world` threads of one process."""

    def __init__(self, world):
        self.world = world
        self.buf = [None] * world
        self.bar = threading.Barrier(world)

    def fn(self, rank):
        def f(b):
            self.buf[rank] = b
            self.bar.wait()
            out = b"".join(self.buf)
            self.bar.wait()
            return out
        return f


_ORC = {}


def _oracle_tiny(X):
    """The oracle index of the committed Tiny build file (test infrastructure)."""
    if "ix" not in _ORC:
        import oracle
        from oracle import build as B
        _ORC["ix"] = oracle.Index(B.read(os.path.join(ROOT, "data", "tiny", "build_d16.mrqb")), X)
    return _ORC["ix"]


def _tiny():
    import synth
    cfg = synth.config_by_name("tiny")
    X, Q = synth.generate(cfg)
    return X, Q, os.path.join(ROOT, "data", "tiny", "build_d16.mrqb")


@pytest.mark.gpu
@pytest.mark.parametrize("tau", ["TIGHT", "LOOSE"])
def test_forced_exchange_equals_fast_path(tau):
    m = _lib()
    X, Q, bfile = _tiny()
    a = m.Index(bfile, X, 16)
    ia, da, sa = a.search(Q, K=10, nprobe=4, tau_schedule=tau)
    t0a, t1a = a.fetch("tau0", "f64").copy(), a.fetch("tau1", "f64").copy()
    m.mrq_debug_set(a.h, "force_exchange", 1)
    ib, db, sb = a.search(Q, K=10, nprobe=4, tau_schedule=tau)
    assert np.array_equal(ia, ib) and np.array_equal(da, db)
    assert np.array_equal(t0a, a.fetch("tau0", "f64")) and np.array_equal(t1a, a.fetch("tau1", "f64"))
    assert (sa.scanned, sa.stage1_pass, sa.stage2_pass, sa.exact) == (sb.scanned, sb.stage1_pass, sb.stage2_pass,
                                                                      sb.exact)
    a.close()


@pytest.mark.gpu
@pytest.mark.parametrize("world,K", [(2, 10), (3, 10), (2, 100)])
@pytest.mark.parametrize("tau,mode", [("TIGHT", "FULL"), ("LOOSE", "FULL"), ("TIGHT", "STAGE1_ONLY"),
                                      ("TIGHT", "EXACT"), ("TIGHT", "NOCORR")])
def test_virtual_ranks_equal_single_gpu(world, K, tau, mode):
    m = _lib()
    X, Q, bfile = _tiny()
    ref = m.Index(bfile, X, 16)
    ir, dr, sr = ref.search(Q, K=K, nprobe=4, tau_schedule=tau, mode=mode)
    t0r, t1r = ref.fetch("tau0", "f64").copy(), ref.fetch("tau1", "f64").copy()
    ref.close()
    ex = _ThreadExchange(world)
    idx = [m.Index(bfile, X, 16, rank=r, world=world, host_allgather=ex.fn(r)) for r in range(world)]
    res = [None] * world

    def run(r):
        res[r] = idx[r].search(Q, K=K, nprobe=4, tau_schedule=tau, mode=mode)

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(120)
    oi, od, ost = _oracle_tiny(X).search(Q, K=K, nprobe=4, tau_schedule=tau, mode=mode)
    for r in range(world):
        ids, dd, st = res[r]
        assert np.array_equal(ids, ir), r                  # every rank holds the merged result
        assert np.array_equal(dd, dr), r
        # ... which is the oracle's result queue (Alg.2 L15-L16)
        assert np.array_equal(ids, oi), r
        assert np.array_equal(dd.view(np.uint32), od.view(np.uint32)), r
        assert np.array_equal(idx[r].fetch("tau0", "f64"), t0r)
        assert np.array_equal(idx[r].fetch("tau1", "f64"), t1r)
    tot = lambda f: sum(getattr(res[r][2], f) for r in range(world))  # noqa: E731
    assert tot("scanned") == sr.scanned == ost["scanned"]
    assert tot("stage1_pass") == sr.stage1_pass                           # F1 as a set: sizes add up
    assert tot("stage2_pass") == sr.stage2_pass
    if mode in ("FULL", "STAGE1_ONLY"):      # the oracle's EXACT/NOCORR modes run no stages
        assert tot("stage1_pass") == ost["f1"] and tot("stage2_pass") == ost["f2"]
    for x in idx:
        x.close()


@pytest.mark.gpu
def test_nccl_one_rank_exchange_equals_fast_path():
    """The NCCL transport itself (dlopen'ed libnccl, ncclCommInitRank,
    ncclAllGather on the search stream) on a one-rank communicator: the
    sharded path through NCCL gives the single-GPU result bit for bit."""
    m = _lib()
    X, Q, bfile = _tiny()
    ref = m.Index(bfile, X, 16)
    ir, dr, _ = ref.search(Q, K=10, nprobe=4)
    ref.close()
    uid = m.mrq_nccl_unique_id()
    assert len(uid) == 128
    a = m.Index(bfile, X, 16, rank=0, world=1, nccl_unique_id=uid)
    m.mrq_debug_set(a.h, "force_exchange", 1)
    for tau in ("TIGHT", "LOOSE"):
        ia, da, _ = a.search(Q, K=10, nprobe=4, tau_schedule=tau)
        oi, od, _ = _oracle_tiny(X).search(Q, K=10, nprobe=4, tau_schedule=tau)
        assert np.array_equal(ia, oi) and np.array_equal(da.view(np.uint32), od.view(np.uint32)), tau
        if tau == "TIGHT":
            assert np.array_equal(ia, ir) and np.array_equal(da, dr)
    a.close()


def _nccl_worker(rank, world, uid, tau, out):
    import sys
    sys.path.insert(0, ROOT)
    import paper_2411_06158_b200 as m
    X, Q, bfile = _tiny()
    ix = m.Index(bfile, X, 16, rank=rank, world=world, device=rank, nccl_unique_id=uid)
    ids, dist, st = ix.search(Q, K=10, nprobe=4, tau_schedule=tau)
    out[rank] = (ids.tolist(), dist.view(np.uint32).tolist(), st.scanned, st.stage1_pass, st.stage2_pass)
    ix.close()


@pytest.mark.gpu
@pytest.mark.parametrize("tau", ["TIGHT", "LOOSE"])
def test_two_process_nccl_merge_equals_oracle(tau):
    """Two processes, one GPU each, lists sharded by mrq_shard_plan, the
    decision-T seed sets and the per-rank top-K exchanged with ncclAllGather
    (DESIGN.md §6): every rank returns the oracle's result queue
    and the per-rank survivor counts add up to the oracle's.  Needs 2 GPUs
    (the gpurun box has one: skipped there; the virtual-rank test covers the
    exchange logic on one GPU)."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    m = _lib()
    uid = m.mrq_nccl_unique_id()
    world = 2
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.start_processes(_nccl_worker, args=(world, uid, tau, out), nprocs=world, start_method="spawn")
    X, Q, _ = _tiny()
    oi, od, ost = _oracle_tiny(X).search(Q, K=10, nprobe=4, tau_schedule=tau)
    for r in range(world):
        ids, dist, *_ = out[r]
        assert np.array_equal(np.array(ids), oi)
        assert np.array_equal(np.array(dist, np.uint32), od.view(np.uint32))
    assert sum(out[r][2] for r in range(world)) == ost["scanned"]
    assert sum(out[r][3] for r in range(world)) == ost["f1"]
    assert sum(out[r][4] for r in range(world)) == ost["f2"]

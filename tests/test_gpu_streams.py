"""Row f2 on the GPU (multi-stream ranks, time-ordered memory) through the C ABI, bit-exact
against the oracle: random multi-stream graphs, the overlapped-gradient-reduce shape of the
dense configs, per-op start/finish, time-ordered peaks and the critical path."""
import os

import numpy as np
import pytest

import oracle
import workloads as w

pytestmark = pytest.mark.gpu
NPROC = os.cpu_count() or 1


@pytest.fixture(scope="module")
def prism():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_15617_b200 as P

    P.build_library()
    P.use_torch_allocator()
    return P


def _graph(P, tm):
    import torch

    return P.Graph(tm, stream=torch.cuda.current_stream().cuda_stream)


def _check(P, tm, S, node_dur=None, ranks=16):
    g = _graph(P, tm)
    if node_dur is not None:
        g.set_durations(node_dur=node_dur)
    it = g.replay(S, amp_q16=6554, kind_mask=7)
    assert g.last_algo() in ("cells", "ranks")  # "ranks": S = 1 on a graph that drew no side stream
    ref = oracle.replay(tm, S, amp_q16=6554, kind_mask=7, node_dur=node_dur, times=True, threads=min(NPROC, S))
    assert np.array_equal(it, ref["iter"]), (it[:4], ref["iter"][:4])
    for k in sorted({0, S - 1}):
        assert np.array_equal(g.peak_memory_at(k), ref["peak"][k])
    assert np.array_equal(g.peak_memory(), ref["peak"][0])
    rp = g.export("rank_ptr")
    W = tm.topo.world
    for r in (range(W) if W <= ranks else np.random.default_rng(0).choice(W, ranks, replace=False)):
        for k in sorted({0, S - 1}):
            st, fi, _ = g.query_rank(int(r), k)
            a, b = rp[r], rp[r + 1]
            assert np.array_equal(fi, ref["finish"][k, a:b]) and np.array_equal(st, ref["start"][k, a:b]), (r, k)
    return g


@pytest.mark.parametrize("seed", range(24))
def test_random_multistream(prism, seed):
    tm = w.random_templates(seed, max_world=32, max_ops=40, streams=[2, 3, 4][seed % 3])
    d = np.random.default_rng(seed).integers(0, 1000, tm.n_nodes) if seed % 2 else None
    _check(prism, tm, [1, 5, 33, 64][seed % 4], node_dur=d)


def test_hand_examples(prism):
    b = w._StageBuilder()
    b.compute(100, alloc=10)
    b.compute(100, free=10)
    b.compute(50, stream=1, alloc=7, free=7)
    tm = w.assemble(w.Topology(1, 1, 1), [b.array()], [1000])
    g = _graph(prism, tm)
    assert g.replay(1).tolist() == [200]
    assert g.peak_memory().tolist() == [1017]  # time order sees the side buffer overlap
    st, fi, _ = g.query_rank(0, 0)
    assert st.tolist() == [0, 100, 0] and fi.tolist() == [100, 200, 50]


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_overlap_grad_reduce_scaled(prism, name):
    _check(prism, w.overlap_grad_reduce(w.scaled(name)), 64)


@pytest.mark.parametrize("seed", range(10))
def test_multistream_critical_path(prism, seed):
    tm = w.random_templates(seed, max_world=32, max_ops=40, streams=2)
    d = np.random.default_rng(seed).integers(0, 500, tm.n_nodes)
    g = _graph(prism, tm)
    g.set_durations(node_dur=d)
    g.replay(3, amp_q16=6554, kind_mask=7)
    for k in (0, 2):
        path, T = g.critical_path(k)
        rpath, rT = oracle.critical_path(tm, k, amp_q16=6554, kind_mask=7, node_dur=d)
        assert T == rT and np.array_equal(path, rpath)


def test_time_ordered_equals_program_order_single_stream(prism):
    tm = w.scaled("C3")
    g = _graph(prism, tm)
    g.replay(8, amp_q16=6554, kind_mask=7)
    assert np.array_equal(g.peak_memory_at(5), g.peak_memory())


def test_multistream_full_size_c2(prism):
    """The overlapped C2 (1024 ranks, one rank per warp) at S = 64: sampled scenarios' iteration
    times and scenario 0's time-ordered peaks equal the oracle's."""
    tm = w.overlap_grad_reduce(w.config("C2"))
    g = _graph(prism, tm)
    it = g.replay(64, amp_q16=6554, kind_mask=7)
    for k in (0, 63):
        r = oracle.replay(tm, 1, scen_first=k, amp_q16=6554, kind_mask=7, peaks=(k == 0))
        assert it[k] == r["iter"][0]
        if k == 0:
            assert np.array_equal(g.peak_memory(), r["peak"][0])


@pytest.mark.slow
def test_multistream_full_size_c5(prism):
    """The 8192-rank C5 with overlapped gradient buckets (TP cells + per-rank stream / event
    state): sampled scenarios' iteration times equal the oracle's."""
    tm = w.overlap_grad_reduce(w.config("C5"))
    g = _graph(prism, tm)
    it = g.replay(64, amp_q16=6554, kind_mask=7)
    for k in (0, 63):
        assert it[k] == oracle.replay(tm, 1, scen_first=k, amp_q16=6554, kind_mask=7, peaks=False)["iter"][0]

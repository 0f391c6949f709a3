"""Rows f1 / f3 / f4 on the GPU through the C ABI, bit-exact against the oracle: replays with
per-node (measured) durations, label overrides, per-rank compute slowdown, per-node memory deltas
(MoE-imbalance shape) and the critical path."""
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


def _check(P, tm, S, node_dur, algo="auto", times=True, node_alloc=None, node_free=None, **extra):
    g = _graph(P, tm)
    g.set_durations(node_dur=node_dur, node_alloc=node_alloc, node_free=node_free, **extra)
    it = g.replay(S, amp_q16=6554, kind_mask=7, algo=algo)
    d = node_dur if not extra else oracle.whatif_durations(tm, node_dur=node_dur, **{
        {"rank_slow_q16": "rank_factor_q16"}.get(k, k): v for k, v in extra.items()})
    ref = oracle.replay(tm, S, amp_q16=6554, kind_mask=7, node_dur=d, node_alloc=node_alloc,
                        node_free=node_free, times=times, threads=min(NPROC, S))
    assert np.array_equal(it, ref["iter"]), (it[:4], ref["iter"][:4])
    assert np.array_equal(g.peak_memory(), ref["peak"][0])
    if times:
        rp = g.export("rank_ptr")
        W = tm.topo.world
        for r in (range(W) if W <= 32 else np.random.default_rng(0).choice(W, 32, replace=False)):
            st, fi, _ = g.query_rank(int(r), S - 1)
            a, b = rp[r], rp[r + 1]
            assert np.array_equal(fi, ref["finish"][S - 1, a:b]) and np.array_equal(st, ref["start"][S - 1, a:b])
    return g, ref


@pytest.mark.parametrize("algo", ["cells", "levels"])
@pytest.mark.parametrize("seed", range(16))
def test_measured_durations_random(prism, seed, algo):
    tm = w.random_templates(seed, max_world=32, max_ops=40)
    if algo == "cells" and tm.topo.tp > 8:
        pytest.skip("cells need tp <= 8")
    d = np.random.default_rng(seed).integers(0, 2000, tm.n_nodes)
    _check(prism, tm, [1, 5, 33, 64][seed % 4], d, algo=algo)


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_measured_durations_configs(prism, name):
    """f1: per-node 'measured' durations = the model +-5 % jitter per node (slice-fill shape)."""
    tm = w.scaled(name)
    nt = oracle.node_table(tm)
    rng = np.random.default_rng(7)
    d = (nt["dur"] * rng.integers(95, 106, tm.n_nodes)) // 100
    _check(prism, tm, 64, d)


def test_calibration_fig5_and_identity(prism):
    """S:318 on the GPU: the receive is shifted after the send; template durations given as
    node_dur reproduce the plain replay."""
    b0 = w._StageBuilder(); b0.compute(12); b0.p2p(w.SEND_NEXT, 0)
    b1 = w._StageBuilder(); b1.compute(3); b1.p2p(w.RECV_PREV, 0)
    tm = w.assemble(w.Topology(1, 2, 1), [b0.array(), b1.array()], [0, 0])
    g = _graph(prism, tm)
    g.set_durations(node_dur=[12, 0, 3, 0])
    assert g.replay(1).tolist() == [12]
    st, fi, _ = g.query_rank(1, 0)
    assert st.tolist() == [0, 12] and fi.tolist() == [3, 12]
    tm = w.scaled("C2")
    g = _graph(prism, tm)
    a = g.replay(64, amp_q16=6554, kind_mask=7)
    g.set_durations(node_dur=oracle.node_table(tm)["dur"])
    assert np.array_equal(g.replay(64, amp_q16=6554, kind_mask=7), a)
    g.set_durations()
    assert np.array_equal(g.replay(64, amp_q16=6554, kind_mask=7), a)


def test_whatif_labels_and_fault_injection(prism):
    tm = w.scaled("C5")
    nt = oracle.node_table(tm)
    labs = sorted(set(int(l) for l, k in zip(nt["label"], nt["kind"]) if k == 0))[:40]
    ov = {l: 777 + i for i, l in enumerate(labs)}
    f = np.full(tm.topo.world, 65536, np.int32)
    f[5] = int(1.12 * 65536)
    f[17] = 3 * 65536
    _check(prism, tm, 33, None, label_dur=ov, rank_slow_q16=f)
    g = _graph(prism, tm)
    with pytest.raises(prism.PrismError) as e:
        g.set_durations(label_dur={0xDEADBEEF: 5})
    assert e.value.name == "PRISM_E_UNKNOWN_LABEL"


def test_moe_memory_deltas(prism):
    """f4 shape: per-node activation sizes scaled per EP rank; peaks equal the oracle's and a
    running total below zero is refused."""
    tm = w.scaled("C4")
    nt = oracle.node_table(tm)
    ex_alloc = np.zeros(tm.n_nodes, np.int64)
    ex_free = np.zeros(tm.n_nodes, np.int64)
    # rebuild alloc/free from the templates, scaled by (1 + rank % 3) / 2 per rank
    t = tm.topo
    n = 0
    for r in range(t.world):
        s = (r // t.tp) % t.pp
        T = tm.stage(s)
        k = 1 + r % 3
        ex_alloc[n:n + len(T)] = T["mem_alloc"] * k // 2
        ex_free[n:n + len(T)] = T["mem_free"] * k // 2
        n += len(T)
    _check(prism, tm, 16, None, node_alloc=ex_alloc, node_free=ex_free, times=False)
    g = _graph(prism, tm)
    bad = ex_free.copy()
    bad[np.argmax(bad)] += 1 << 40
    with pytest.raises(prism.PrismError) as e:
        g.set_durations(node_alloc=ex_alloc, node_free=bad)
    assert e.value.name == "PRISM_E_NEGATIVE_MEMORY"


@pytest.mark.parametrize("seed", range(20))
def test_critical_path_random(prism, seed):
    tm = w.random_templates(seed, max_world=32, max_ops=40)
    d = np.random.default_rng(seed).integers(0, 500, tm.n_nodes)
    g = _graph(prism, tm)
    g.set_durations(node_dur=d)
    S = 5
    g.replay(S, amp_q16=6554, kind_mask=7)
    for k in (0, S - 1):
        path, T = g.critical_path(k)
        rpath, rT = oracle.critical_path(tm, k, amp_q16=6554, kind_mask=7, node_dur=d)
        assert T == rT and np.array_equal(path, rpath)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_critical_path_configs(prism, name):
    tm = w.config(name) if name == "C1" else w.scaled(name)
    g = _graph(prism, tm)
    g.replay(3, amp_q16=6554, kind_mask=7)
    for k in (0, 2):
        path, T = g.critical_path(k)
        rpath, rT = oracle.critical_path(tm, k, amp_q16=6554, kind_mask=7)
        assert T == rT and np.array_equal(path, rpath), (name, k, len(path), len(rpath))


@pytest.mark.parametrize("seed", range(3))
def test_moe_imbalance_fig3(prism, seed):
    """f4: the Fig. 3 br profile on the C4-shaped MoE graph: per-node expert / A2A
    durations and activation sizes; iteration times and every rank's peak equal the oracle's."""
    import workloads.moe as M

    tm = w.scaled("C4")
    s = M.derive_schedule(M.FIG3_PROFILE, 32, tm.topo.ep, seed=seed)
    d, a, f = M.moe_overrides(tm, s)
    g, ref = _check(prism, tm, 33, d, node_alloc=a, node_free=f)
    base = oracle.replay(tm, 1)
    assert ref["peak"][0].max() > base["peak"][0].max()  # imbalance raises the worst rank's peak

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


def test_memory_deltas(prism):
    """Per-node activation sizes scaled per rank; peaks equal the oracle's and a running total below
    zero is refused (device-side validation) with the previous overrides kept."""
    tm = w.scaled("C4")
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
    g, ref = _check(prism, tm, 16, None, node_alloc=ex_alloc, node_free=ex_free, times=False)
    bad = ex_free.copy()
    bad[np.argmax(bad)] += 1 << 40
    with pytest.raises(prism.PrismError) as e:
        g.set_durations(node_alloc=ex_alloc, node_free=bad)
    assert e.value.name == "PRISM_E_NEGATIVE_MEMORY"
    assert np.array_equal(g.peak_memory(), ref["peak"][0])  # the previous overrides stand
    neg = ex_alloc.copy()
    neg[3] = -1
    with pytest.raises(prism.PrismError) as e:
        g.set_durations(node_alloc=neg, node_free=ex_free)
    assert e.value.name == "PRISM_E_INVALID_ARG"


@pytest.mark.parametrize("big", [False, True])
@pytest.mark.parametrize("seed", range(20))
def test_critical_path_random(prism, seed, big):
    """big: durations in multiples of 2^36 ns with many ties, so T >= 2^38 and the group pass takes
    its unpacked two-pass form (ready time, then the lowest member at it)."""
    tm = w.random_templates(seed, max_world=32, max_ops=40)
    rng = np.random.default_rng(seed)
    d = rng.integers(0, 4, tm.n_nodes) << 36 if big else rng.integers(0, 500, tm.n_nodes)
    g = _graph(prism, tm)
    g.set_durations(node_dur=d)
    S = 5
    g.replay(S, amp_q16=6554, kind_mask=7)
    for k in (0, S - 1):
        path, T = g.critical_path(k)
        rpath, rT = oracle.critical_path(tm, k, amp_q16=6554, kind_mask=7, node_dur=d)
        assert T == rT and np.array_equal(path, rpath)
        assert not big or T >= 1 << 38 or len(path) < 4


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_critical_path_configs(prism, name):
    tm = w.config(name) if name == "C1" else w.scaled(name)
    g = _graph(prism, tm)
    g.replay(3, amp_q16=6554, kind_mask=7)
    for k in (0, 2):
        path, T = g.critical_path(k)
        rpath, rT = oracle.critical_path(tm, k, amp_q16=6554, kind_mask=7)
        assert T == rT and np.array_equal(path, rpath), (name, k, len(path), len(rpath))


def _moe_inputs(tm, seed, events=32):
    import workloads.moe as M

    s = M.derive_schedule(M.FIG3_PROFILE, events, tm.topo.ep, seed=seed)
    return M.op_events(tm, events), M.br_q16(s)


@pytest.mark.parametrize("seed", range(3))
def test_moe_imbalance_fig3(prism, seed):
    """f4 (App. F mock router): the Fig. 3 br profile on the C4-shaped MoE
    graph through prism_set_moe_load, against the oracle's own plain-loop br scaling
    (oracle.moe_load) replayed by the DES: iteration times, per-op times, every rank's peak."""
    tm = w.scaled("C4")
    ev, br = _moe_inputs(tm, seed)
    g = _graph(prism, tm)
    g.set_moe_load(ev, br)
    S = 33
    it = g.replay(S, amp_q16=6554, kind_mask=7)
    d, a, f = oracle.moe_load(tm, ev, br)
    ref = oracle.replay(tm, S, amp_q16=6554, kind_mask=7, node_dur=d, node_alloc=a, node_free=f, times=True,
                        threads=min(NPROC, S))
    assert np.array_equal(it, ref["iter"])
    assert np.array_equal(g.peak_memory(), ref["peak"][0])
    rp = g.export("rank_ptr")
    for r in np.random.default_rng(seed).choice(tm.topo.world, 24, replace=False):
        st, fi, _ = g.query_rank(int(r), S - 1)
        assert np.array_equal(fi, ref["finish"][S - 1, rp[r]:rp[r + 1]])
        assert np.array_equal(st, ref["start"][S - 1, rp[r]:rp[r + 1]])
    base = oracle.replay(tm, 1)
    assert ref["peak"][0].max() > base["peak"][0].max()  # imbalance raises the worst rank's peak
    g.set_moe_load(None)  # cleared: the template graph again
    assert np.array_equal(g.replay(2, amp_q16=6554, kind_mask=7), oracle.replay(tm, 2, amp_q16=6554, kind_mask=7,
                                                                              peaks=False)["iter"])


@pytest.mark.parametrize("scale", [1, 2, 6, 7])
def test_moe_load_composes_with_overrides(prism, scale):
    """MoE load on top of measured durations, then label overrides and a slowed rank (include/
    prism.h order: base -> br -> label -> rank slowdown), either call first."""
    tm = w.scaled("C4")
    ev, br = _moe_inputs(tm, 5, events=7)
    rng = np.random.default_rng(scale)
    base = oracle.node_table(tm)["dur"] * rng.integers(90, 111, tm.n_nodes) // 100
    lab = {int(l): 1234 for l in np.unique(tm.ops["label"])[:3]}
    f = np.full(tm.topo.world, 65536, np.int32)
    f[3] = 2 * 65536
    d, a, fr = oracle.moe_load(tm, ev, br, scale, node_dur=base)
    d = oracle.whatif_durations(tm, node_dur=d, label_dur=lab, rank_factor_q16=f)
    ref = oracle.replay(tm, 5, amp_q16=6554, kind_mask=7, node_dur=d, node_alloc=a, node_free=fr,
                        threads=min(NPROC, 5))
    for order in (0, 1):
        g = _graph(prism, tm)
        if order == 0:
            g.set_moe_load(ev, br, scale)
            g.set_durations(node_dur=base, label_dur=lab, rank_slow_q16=f)
        else:
            g.set_durations(node_dur=base, label_dur=lab, rank_slow_q16=f)
            g.set_moe_load(ev, br, scale)
        assert np.array_equal(g.replay(5, amp_q16=6554, kind_mask=7), ref["iter"])
        assert np.array_equal(g.peak_memory(), ref["peak"][0])


def test_moe_load_errors(prism):
    tm = w.scaled("C4")
    ev, br = _moe_inputs(tm, 0, events=32)
    g = _graph(prism, tm)
    with pytest.raises(prism.PrismError):
        g.set_moe_load(np.full_like(ev, br.shape[0]), br)  # event outside [-1, n_events)
    bad = br.copy()
    bad[0, 0] = -5
    with pytest.raises(prism.PrismError):
        g.set_moe_load(ev, bad)
    # scaling frees but not allocations drives the running total negative (br > 1 on some rank)
    with pytest.raises(prism.PrismError) as e:
        g.set_moe_load(ev, np.full_like(br, 2 * 65536), 1 | 4)
    assert e.value.name == "PRISM_E_NEGATIVE_MEMORY"


@pytest.mark.slow
def test_moe_fig3_full_c4(prism):
    """Full-size C4 (2048 ranks, EP 64) under the Fig. 3 profile, as bench.py's f4 row runs it."""
    tm = w.config("C4")
    ev, br = _moe_inputs(tm, 0, events=64)
    g = _graph(prism, tm)
    g.set_moe_load(ev, br)
    it = g.replay(64, amp_q16=6554, kind_mask=7)
    d, a, f = oracle.moe_load(tm, ev, br)
    ref = oracle.replay(tm, 64, amp_q16=6554, kind_mask=7, node_dur=d, node_alloc=a, node_free=f, threads=NPROC)
    assert np.array_equal(it, ref["iter"]) and np.array_equal(g.peak_memory(), ref["peak"][0])


def test_moe_two_rank_golden(prism):
    """The hand-worked two-rank example (tests/golden/moe_two_rank_example.txt) on the GPU."""
    from test_moe_router import _golden, _two_rank_templates
    import workloads.moe as M

    G = _golden()
    tm = _two_rank_templates()
    g = _graph(prism, tm)
    g.set_moe_load(M.op_events(tm, 1), np.array([G["br_q16"]], np.int32))
    assert g.replay(1)[0] == G["iter"][0]
    assert g.peak_memory().tolist() == G["peak"]
    assert g.query_rank(0)[1].tolist() == G["finish_rank0"] and g.query_rank(1)[1].tolist() == G["finish_rank1"]


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_device_arrays_equal_host_arrays(prism, name):
    """prism_set_durations with per-node arrays already on the GPU (a CUDA int64 tensor, copied
    device to device) replays exactly as the same values from host memory, and as the oracle."""
    import torch

    tm = w.scaled(name)
    nt = oracle.node_table(tm)
    rng = np.random.default_rng(11)
    d = (nt["dur"] * rng.integers(90, 111, tm.n_nodes)) // 100
    al = rng.integers(0, 1000, tm.n_nodes)  # every node frees what it allocated: totals stay >= 0
    fr = al.copy()
    g_host, ref = _check(prism, tm, 33, d, node_alloc=al, node_free=fr, times=False)
    g = _graph(prism, tm)
    g.set_durations(node_dur=torch.from_numpy(np.ascontiguousarray(d, np.int64)).cuda(),
                    node_alloc=torch.from_numpy(np.ascontiguousarray(al, np.int64)).cuda(),
                    node_free=torch.from_numpy(np.ascontiguousarray(fr, np.int64)).cuda())
    it = g.replay(33, amp_q16=6554, kind_mask=7)
    assert np.array_equal(it, ref["iter"])
    assert np.array_equal(g.peak_memory(), ref["peak"][0])
    with pytest.raises(ValueError):
        g.set_durations(node_dur=torch.zeros(3, dtype=torch.int64, device="cuda"))
    with pytest.raises(ValueError):
        g.set_durations(node_dur=torch.zeros(tm.n_nodes, dtype=torch.int32, device="cuda"))

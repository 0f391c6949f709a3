"""Row f2 (multi-stream ranks, time-ordered memory; P:699 overlapped gradient communication,
P:1729 "P2P Overlap" rows): the oracle pinned by hand-computed schedules, the program-order vs
time-order memory example, and brute-force path enumeration on random multi-stream graphs."""
import numpy as np
import pytest

import oracle
from oracle import brute
import workloads as w


def _path_length(tm, path, d):
    """Critical-path length: compute spans add their duration, sync nodes their group's (Z2)."""
    ex = oracle.expand(tm)
    nt = oracle.node_table(tm)
    grp = {}
    for gi in range(ex["groups"]):
        mem = ex["mem"][ex["ptr"][gi]:ex["ptr"][gi + 1]]
        for m in mem:
            grp.setdefault(int(m), []).append(max(int(d[x]) for x in mem))
    return sum(int(d[n]) if nt["kind"][n] == 0 else max(grp[int(n)]) for n in path)


def _one_rank(ops):
    b = w._StageBuilder()
    for kw in ops:
        b.compute(**kw)
    return w.assemble(w.Topology(1, 1, 1), [b.array()], [1000])


def test_two_streams_run_concurrently():
    tm = _one_rank([dict(dur=100), dict(dur=200), dict(dur=150, stream=1)])
    r = oracle.replay(tm, 1, times=True)
    assert r["start"][0].tolist() == [0, 100, 0] and r["iter"][0] == 300


def test_event_wait():
    tm = _one_rank([dict(dur=100, record=0), dict(dur=200), dict(dur=150, stream=1, wait=0)])
    r = oracle.replay(tm, 1, times=True)
    assert r["start"][0].tolist() == [0, 100, 100] and r["iter"][0] == 300
    # a wait on a slot never recorded before it is satisfied at once (CUDA event semantics)
    tm = _one_rank([dict(dur=50, stream=1, wait=3), dict(dur=100, record=3)])
    assert oracle.replay(tm, 1, times=True)["start"][0].tolist() == [0, 0]


def test_time_ordered_memory():
    """+alloc at start / -free at finish in (time, event index) order: a buffer on a side stream
    that overlaps the main stream's activation adds to the peak; program order would not see it."""
    ops = [dict(dur=100, alloc=10), dict(dur=100, free=10), dict(dur=50, stream=1, alloc=7, free=7)]
    assert oracle.replay(_one_rank(ops), 1)["peak"][0].tolist() == [1000 + 17]
    ops[2]["wait"] = 0
    ops[1]["record"] = 0  # now the side buffer lives after the activation is freed
    assert oracle.replay(_one_rank(ops), 1)["peak"][0].tolist() == [1000 + 10]


def test_overlapped_grad_reduce_closed_form():
    """Megatron-style overlap on one DP pair: each backward span k (stream 0, 1000 ns) records an
    event; a 300 ns DP all-reduce bucket on stream 1 waits for it; OPT waits for the last bucket.
    Buckets are shorter than backward spans, so each bucket ends 300 ns after its span and
    T = 3 * 1000 + 300 + 500 (OPT)."""
    stages = []
    b = w._StageBuilder()
    for k in range(3):
        b.compute(1000, record=k)
        b.coll(w.ROLE_DP, w.COLL_AR, 300, stream=1, wait=k, record=4 + k % 2)
    b.compute(500, wait=4 + 2 % 2)
    tm = w.assemble(w.Topology(1, 1, 2), [b.array()], [0])
    r = oracle.replay(tm, 1, times=True)
    assert r["iter"][0] == 3000 + 300 + 500
    assert r["iter"][0] == brute.iteration_time(tm)[0]


@pytest.mark.parametrize("seed", range(24))
def test_random_multistream_brute_force(seed):
    tm = w.random_templates(seed, max_world=8, max_ops=10, streams=2)
    d = np.random.default_rng(seed).integers(0, 300, tm.n_nodes)
    T, fin = brute.iteration_time(tm, d)
    r = oracle.replay(tm, 1, node_dur=d, times=True)
    assert r["iter"][0] == T and r["finish"][0].tolist() == fin


@pytest.mark.parametrize("seed", range(8))
def test_random_multistream_critical_path_tight(seed):
    tm = w.random_templates(seed, max_world=8, max_ops=12, streams=3)
    d = np.random.default_rng(seed).integers(0, 300, tm.n_nodes)
    path, T = oracle.critical_path(tm, 0, node_dur=d)
    assert _path_length(tm, path, d) == T == brute.iteration_time(tm, d)[0]


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_overlap_grad_reduce_never_slower(name):
    """Moving the gradient buckets onto a side stream only removes ordering constraints (each
    bucket waits for an earlier backward span instead of the last), so the overlapped iteration
    is never longer than the serial one; per-rank memory events stay non-negative in time order."""
    tm = w.scaled(name)
    ov = w.overlap_grad_reduce(tm)
    a = oracle.replay(tm, 3, amp_q16=6554, kind_mask=7)
    b = oracle.replay(ov, 3, amp_q16=6554, kind_mask=7)
    assert (b["iter"] <= a["iter"]).all()
    if name != "C4":  # C4's iteration ends with ZeRO-1 all-gathers the overlap cannot shorten
        assert (b["iter"] < a["iter"]).any()


def test_overlap_tiny_brute_force():
    tm = w.uniform_pipeline(1, 2, 2, 2, dp_ar_ns=300)
    b = w._StageBuilder()
    for k in range(3):
        b.compute(100 * (k + 1), record=k)
    for k in range(3):
        b.coll(w.ROLE_DP, w.COLL_AR, 50 + k, stream=1, wait=k)
    b.compute(10, stream=0)
    tm = w.assemble(w.Topology(1, 1, 2), [b.array()], [0])
    assert oracle.replay(tm, 1)["iter"][0] == brute.iteration_time(tm)[0] == 600 + 52

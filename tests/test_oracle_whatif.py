"""Rows f1 (inter-slice calibration) and f3 (what-if attribution, fault injection): the oracle
pinned against SPEC worked examples, closed-form / brute-force values and exact properties.

The engine is the same ASAP replay as rows a6-a8 with per-node durations (oracle.replay node_dur):
calibration = replay of the timed graph filled slice by slice; what-if = replay with
label overrides and per-rank compute slowdown."""
import numpy as np
import pytest

import oracle
from oracle import brute
import workloads as w


def _two_stage_send_recv(send_at: int, recv_local: int):
    """SPEC S:318 (Fig. 5 of the paper): a send on stage 0 after `send_at` ns of work,
    its matched receive on stage 1 after `recv_local` ns."""
    b0 = w._StageBuilder()
    b0.compute(send_at, w.make_label("SPAN"))
    b0.p2p(w.SEND_NEXT, 0, w.make_label("P2P"))
    b1 = w._StageBuilder()
    b1.compute(recv_local, w.make_label("SPAN"))
    b1.p2p(w.RECV_PREV, 0, w.make_label("P2P"))
    return w.assemble(w.Topology(1, 2, 1), [b0.array(), b1.array()], [0, 0])


# ------------------------------------------------------------------ f1: calibration
def test_spec_fig5_receive_shifted_after_send():
    """send (slice 0) ends at t=12, matched recv (slice 1) locally at t=3 -> recv start 12."""
    tm = _two_stage_send_recv(12, 3)
    nt = oracle.node_table(tm)
    local = oracle.slice_local_finish(tm, nt["dur"], [[0], [1]])
    assert local.tolist() == [12, 12, 3, 3]  # slice-local: the receive 'happens' at 3
    r = oracle.replay(tm, 1, node_dur=nt["dur"], times=True)
    recv = 3  # node order: stage-0 span, send, stage-1 span, recv
    assert r["start"][0][recv] == 12 and r["finish"][0][recv] == 12
    assert r["iter"][0] == 12


def test_spec_single_node():
    """one node of duration 5 -> start 0, makespan 5."""
    b = w._StageBuilder()
    b.compute(5)
    tm = w.assemble(w.Topology(1, 1, 1), [b.array()], [0])
    r = oracle.replay(tm, 1, node_dur=np.array([5]), times=True)
    assert r["start"][0].tolist() == [0] and r["iter"][0] == 5


@pytest.mark.parametrize("name", ["C1", "C2", "C4"])
def test_calibration_with_exact_durations_is_the_full_schedule(name):
    """Acceptance S:646 analogue: slice-filled durations equal to the model (jitter 0) calibrate to
    exactly the full-concurrency schedule."""
    tm = w.config(name) if name == "C1" else w.scaled(name)
    nt = oracle.node_table(tm)
    a = oracle.replay(tm, 1, times=True)
    b = oracle.replay(tm, 1, node_dur=nt["dur"], times=True)
    assert np.array_equal(a["start"], b["start"]) and np.array_equal(a["finish"], b["finish"])


def test_calibration_necessity():
    """Acceptance S:647 analogue (P:1694-1696 '>10%'): on a 4-slice pipeline (one stage per slice)
    the concatenated slice-local timestamps miss the pipeline's cross-stage waits by > 5%; the
    calibrated makespan is the schedule's, error 0."""
    tm = w.uniform_pipeline(1, 4, 1, 8, dp_ar_ns=-1, opt_ns=-1)
    nt = oracle.node_table(tm)
    local = oracle.slice_local_finish(tm, nt["dur"], [[s] for s in range(4)])
    T = oracle.replay(tm, 1, node_dur=nt["dur"])["iter"][0]
    assert T == (8 + 4 - 1) * (1000 + 2000)  # 1F1B closed form (m+p-1)(f+b)
    assert int(local.max()) == 8 * (1000 + 2000)  # slice-local: no bubble is ever seen
    assert abs(int(local.max()) - T) / T > 0.05


@pytest.mark.parametrize("seed", range(8))
def test_calibration_idempotent(seed):
    """calibrate(calibrate(g)) = calibrate(g): re-feeding every node's calibrated duration
    (finish - start; a sync node's is its group's shared duration, Z2) reproduces the schedule."""
    tm = w.random_templates(seed, max_world=12, max_ops=14)
    rng = np.random.default_rng(seed)
    d = rng.integers(0, 500, tm.n_nodes)
    a = oracle.replay(tm, 1, node_dur=d, times=True)
    d2 = a["finish"][0] - a["start"][0]
    b = oracle.replay(tm, 1, node_dur=d2, times=True)
    assert np.array_equal(a["start"], b["start"]) and np.array_equal(a["finish"], b["finish"])


@pytest.mark.parametrize("seed", range(12))
def test_per_node_durations_brute_force(seed):
    """Random per-node (measured) durations on tiny random graphs: DES == path enumeration."""
    tm = w.random_templates(seed, max_world=8, max_ops=10)
    d = np.random.default_rng(100 + seed).integers(0, 300, tm.n_nodes)
    T, fin = brute.iteration_time(tm, d)
    r = oracle.replay(tm, 1, node_dur=d, times=True)
    assert r["iter"][0] == T and r["finish"][0].tolist() == fin


# ------------------------------------------------------------------ f3: what-if, fault injection
def _path_length(tm, path, d):
    """Sum over the critical path: a compute node contributes its duration, a sync node its
    group's (the max of the members' durations, Z2)."""
    ex = oracle.expand(tm)
    nt = oracle.node_table(tm)
    grp_of = {}
    for gi in range(ex["groups"]):
        mem = ex["mem"][ex["ptr"][gi]:ex["ptr"][gi + 1]]
        gd = max(int(d[m]) for m in mem)
        for m in mem:
            grp_of.setdefault(int(m), []).append(gd)
    return sum(int(d[n]) if nt["kind"][n] == 0 else max(grp_of[int(n)]) for n in path)


@pytest.mark.parametrize("seed", range(10))
def test_critical_path_is_tight(seed):
    """The critical path's summed durations equal the makespan (critical-path length =
    makespan of the ASAP schedule), against brute force."""
    tm = w.random_templates(seed, max_world=8, max_ops=12)
    d = np.random.default_rng(seed).integers(0, 300, tm.n_nodes)
    path, T = oracle.critical_path(tm, 0, node_dur=d)
    assert T == brute.iteration_time(tm, d)[0]
    assert _path_length(tm, path, d) == T


def test_whatif_identity_and_unknown_label():
    tm = w.config("C1")
    assert np.array_equal(oracle.whatif_durations(tm), oracle.node_table(tm)["dur"])
    with pytest.raises(oracle.OracleError) as e:
        oracle.whatif_durations(tm, label_dur={0xDEAD: 1})
    assert e.value.name == "UNKNOWN_LABEL"


def test_whatif_halve_forward_pp1():
    """halving every forward compute in a PP=1 workload lowers the makespan by exactly the
    summed savings on the critical path."""
    tm = w.uniform_pipeline(2, 1, 2, 6, f_ns=1001, b_ns=2000)
    nt = oracle.node_table(tm)
    fwd = {int(l): int(dd) // 2 for l, dd, k in zip(nt["label"], nt["dur"], nt["kind"])
           if k == 0 and (int(l) >> 24) in (w.OPCODES["ATTN_F"], w.OPCODES["MLP_F"], w.OPCODES["LAYER_F"])}
    path, T = oracle.critical_path(tm, 0)
    d2 = oracle.whatif_durations(tm, label_dur=fwd)
    saved = sum(int(nt["dur"][n] - d2[n]) for n in path if nt["kind"][n] == 0)
    assert saved > 0
    assert oracle.replay(tm, 1, node_dur=d2)["iter"][0] == T - saved


@pytest.mark.parametrize("seed", range(6))
def test_whatif_off_critical_node_leaves_makespan(seed):
    """shortening a node that is off the critical path leaves the makespan unchanged (the
    path keeps its length and the makespan cannot grow)."""
    tm = w.random_templates(seed + 40, max_world=16, max_ops=20)
    nt = oracle.node_table(tm)
    path, T = oracle.critical_path(tm, 0)
    # compute spans only: a sync node's duration also shapes its group's (Z2: max over members)
    off = [n for n in range(tm.n_nodes) if n not in set(path.tolist()) and nt["dur"][n] > 0 and nt["kind"][n] == 0]
    if not off:
        pytest.skip("every node is critical")
    d = nt["dur"].copy()
    for n in off[:5]:
        d[n] = d[n] * 9 // 10
    assert oracle.replay(tm, 1, node_dur=d)["iter"][0] == T


def test_fault_inject_identity_and_growth():
    """factor 1.0 -> identical; slowing a critical pipeline rank grows the makespan
    (value from brute force); a rank with slack absorbs its slowdown while its own finish grows."""
    tm = w.uniform_pipeline(1, 3, 1, 2, dp_ar_ns=-1, opt_ns=-1)
    W = tm.topo.world
    one = np.full(W, 65536)
    assert np.array_equal(oracle.whatif_durations(tm, rank_factor_q16=one), oracle.node_table(tm)["dur"])
    f = one.copy()
    f[1] = int(1.12 * 65536)
    d = oracle.whatif_durations(tm, rank_factor_q16=f)
    T0 = oracle.replay(tm, 1)["iter"][0]
    T1 = oracle.replay(tm, 1, node_dur=d)["iter"][0]
    assert T1 > T0 and T1 == brute.iteration_time(tm, d)[0]
    # slack: a rank whose compute is tiny next to the rank it waits on
    b0 = w._StageBuilder(); b0.compute(100); b0.p2p(w.SEND_NEXT, 0)
    b1 = w._StageBuilder(); b1.compute(10); b1.p2p(w.RECV_PREV, 0); b1.compute(5)
    tm2 = w.assemble(w.Topology(1, 2, 1), [b0.array(), b1.array()], [0, 0])
    f2 = np.array([65536, 4 * 65536])
    d2 = oracle.whatif_durations(tm2, rank_factor_q16=f2)
    a = oracle.replay(tm2, 1)
    b = oracle.replay(tm2, 1, node_dur=d2)
    assert b["iter"][0] > a["iter"][0]  # its trailing span grows 5 -> 20
    assert b["rank_end"][0][0] == a["rank_end"][0][0] == 100  # the send side keeps its finish

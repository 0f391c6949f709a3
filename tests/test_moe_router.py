"""Row f4 inputs: the MoE mock router's balance-ratio schedule (Appendix F; Fig. 3
caption statistics) pinned to SPEC S:535-603's worked examples and properties, and its
effect on the oracle's replay / peak memory."""
import os

import numpy as np
import pytest

import oracle
import workloads as w
import workloads.moe as M


def test_stats_worked_examples():
    assert M.stats(np.ones(16)) == M.BrProfile(1, 1, 1, 0, 1, 0)
    s = M.stats([1, 3])
    assert (s.br_avg, s.br_std, s.br_med) == (2, 1, 2)


def test_br_to_counts_examples():
    assert M.br_to_counts([1] * 8, 128).tolist() == [16] * 8
    assert M.br_to_counts([2, 0, 1, 1], 16).tolist() == [8, 0, 4, 4]
    rng = np.random.default_rng(0)
    for _ in range(50):  # always sums to the total under normalisation
        row = rng.uniform(0.1, 3, 16)
        assert M.br_to_counts(row, 4096).sum() == 4096


def test_fig3_round_trip_and_degenerate():
    s = M.derive_schedule(M.FIG3_PROFILE, 32, 64, seed=3)
    assert s.shape == (32, 64) and M.within(M.stats(s), M.FIG3_PROFILE)
    assert (M.derive_schedule(M.UNIFORM, 4, 4) == 1).all()
    with pytest.raises(M.InfeasibleProfile):
        M.derive_schedule(M.BrProfile(1, 1, 1, 0.5, 1, 0), 4, 4)


@pytest.mark.parametrize("seed", range(6))
def test_round_trip_random_profiles(seed):
    rng = np.random.default_rng(seed)
    mn = rng.uniform(0.2, 1.0)
    mx = mn + rng.uniform(0.5, 2.5)
    med = rng.uniform(mn + 0.3 * (mx - mn), mn + 0.5 * (mx - mn))
    p = M.BrProfile(mn, mx, med + rng.uniform(0, 0.1) * (mx - mn), rng.uniform(0.1, 0.25) * (mx - mn), med,
                    rng.uniform(0, 0.6))
    assert M.within(M.stats(M.derive_schedule(p, 16, 32, seed)), p)


def _golden():
    out = {}
    for line in open(os.path.join(os.path.dirname(__file__), "golden", "moe_two_rank_example.txt")):
        if "=" in line and not line.startswith("#"):
            k, v = line.split("=")
            out[k.strip()] = [int(x) for x in v.split()]
    return out


def _two_rank_templates():
    """The hand-worked example's templates (tests/golden/moe_two_rank_example.txt)."""
    b = w._StageBuilder()
    b.compute(1000, w.make_label("EXPERT_F", 0, 0), alloc=100)
    b.coll(w.ROLE_EP, w.COLL_A2A, 300, label=w.make_label("EP_A2A", 0, 0), alloc=40, free=40)
    b.compute(2000, w.make_label("EXPERT_B", 0, 0), free=100)
    b.compute(10, w.make_label("OPT"))
    return w.Templates(w.Topology(1, 1, 2, 2), b.array(), np.array([0, 4], np.int64), np.zeros(1, np.int64))


def test_moe_load_hand_worked_example():
    """oracle.moe_load + replay against the hand-worked two-rank example (App. F)."""
    G = _golden()
    tm = _two_rank_templates()
    ev = M.op_events(tm, 1)
    assert ev.tolist() == [0, 0, 0, -1]
    br = np.array([G["br_q16"]], np.int32)
    d, a, f = oracle.moe_load(tm, ev, br)
    assert d.tolist() == G["dur_rank0"] + G["dur_rank1"]
    assert a.tolist() == G["alloc_rank0"] + G["alloc_rank1"]
    assert f.tolist() == G["free_rank0"] + G["free_rank1"]
    r = oracle.replay(tm, 1, node_dur=d, node_alloc=a, node_free=f, times=True)
    assert r["finish"][0].tolist() == G["finish_rank0"] + G["finish_rank1"]
    assert r["iter"][0] == G["iter"][0] and r["peak"][0].tolist() == G["peak"]
    # only durations scale: same times, template peaks
    d1, a1, f1 = oracle.moe_load(tm, ev, br, 1)
    r1 = oracle.replay(tm, 1, node_dur=d1, node_alloc=a1, node_free=f1)
    assert r1["iter"][0] == G["iter"][0] and r1["peak"][0].tolist() == G["peak_uniform"]
    u = oracle.moe_load(tm, ev, np.full((1, 2), 65536, np.int32))
    ru = oracle.replay(tm, 1, node_dur=u[0], node_alloc=u[1], node_free=u[2])
    assert ru["iter"][0] == G["iter_uniform"][0] and ru["peak"][0].tolist() == G["peak_uniform"]


def test_moe_load_floor_and_zero():
    """Q16 floor (reading Z8's rounding, R7) and br = 0: a rank that receives no tokens does no
    routed work and holds no routed buffers."""
    tm = _two_rank_templates()
    ev = M.op_events(tm, 1)
    d, a, f = oracle.moe_load(tm, ev, np.array([[65537, 0]], np.int32))
    assert d[:3].tolist() == [1000 * 65537 // 65536, 300 * 65537 // 65536, 2000 * 65537 // 65536]
    assert d[4:].tolist() == [0, 0, 0, 10] and a[4:].tolist() == [0, 0, 0, 0]
    r = oracle.replay(tm, 1, node_dur=d, node_alloc=a, node_free=f)
    assert r["iter"][0] == 1000 + 300 + 2000 + 10  # the busy rank decides T; the A2A waits for it


def test_uniform_schedule_is_the_template_graph():
    tm = w.scaled("C4")
    ev = M.op_events(tm, 4)
    d, a, f = oracle.moe_load(tm, ev, M.br_q16(np.ones((4, tm.topo.ep))))
    nt = oracle.node_table(tm)
    assert np.array_equal(d, nt["dur"])
    base = oracle.replay(tm, 2, amp_q16=6554, kind_mask=7)
    ov = oracle.replay(tm, 2, amp_q16=6554, kind_mask=7, node_dur=d, node_alloc=a, node_free=f)
    assert np.array_equal(base["iter"], ov["iter"]) and np.array_equal(base["peak"], ov["peak"])


def test_routed_ops_are_the_expert_and_a2a_ops():
    """op_events marks exactly the EXPERT_F / EXPERT_B / EP all-to-all template ops, and the
    forward and backward ops of one (layer, microbatch) share one gating event."""
    tm = w.scaled("C4")
    ev = M.op_events(tm, 1 << 20)
    code = tm.ops["label"].astype(np.int64) >> 24
    routed = np.isin(code, [w.OPCODES["EXPERT_F"], w.OPCODES["EXPERT_B"], w.OPCODES["EP_A2A"]])
    assert ((ev >= 0) == routed).all() and routed.any()
    key = tm.ops["label"].astype(np.int64) & 0xFFFFFF
    for k in np.unique(key[routed]):
        assert len(np.unique(ev[routed & (key == k)])) == 1


def test_peak_memory_monotone_in_br():
    """heavier routing never lowers a rank's peak (activations scale with br, frees match)."""
    tm = w.scaled("C4")
    s = M.derive_schedule(M.FIG3_PROFILE, 16, tm.topo.ep, seed=1)
    ev = M.op_events(tm, 16)
    peaks = []
    for bump in (0.0, 0.1, 0.5):
        d, a, f = oracle.moe_load(tm, ev, M.br_q16(s + bump))
        peaks.append(oracle.replay(tm, 1, node_dur=d, node_alloc=a, node_free=f)["peak"][0])
    assert (peaks[1] >= peaks[0]).all() and (peaks[2] >= peaks[1]).all() and (peaks[2] > peaks[0]).any()
    # and the imbalanced iteration is never shorter than the balanced one at the same mean load
    d0, _, _ = oracle.moe_load(tm, ev, M.br_q16(np.full_like(s, s.min())))
    d1, _, _ = oracle.moe_load(tm, ev, M.br_q16(s))
    assert oracle.replay(tm, 1, node_dur=d1)["iter"][0] >= oracle.replay(tm, 1, node_dur=d0)["iter"][0]

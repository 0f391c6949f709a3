"""Pins for the CPU oracle (tests/ is the only place it is exercised against the paper).

Each test fixes the oracle to something other than itself: values the paper/SPEC print for a
worked example (tests/golden/), closed forms of the 1F1B / interleaved pipeline and ring
all-reduce, invariants of the ASAP schedule, and brute-force path enumeration on tiny graphs.
"""
import itertools
import os

import numpy as np
import pytest

import oracle
from oracle import brute
import workloads as w

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _tm(topo, stage_ops, static=None):
    stages = []
    for ops in stage_ops:
        b = w._StageBuilder()
        for o in ops:
            kind = o[0]
            if kind == "c":
                b.compute(o[1], alloc=o[2] if len(o) > 2 else 0, free=o[3] if len(o) > 3 else 0)
            elif kind == "coll":
                b.coll(o[1], o[2], o[3])
            elif kind == "p2p":
                b.op(w.KIND_P2P, o[2], mask=o[1])
        stages.append(b.array() if ops else np.zeros(0, w.OP_DTYPE))
    return w.assemble(topo, stages, static or [0] * topo.pp)


# ------------------------------------------------------------------ hash (reading Z8) pins
def test_splitmix64_published_vector():
    rows = [l.split() for l in open(os.path.join(GOLD, "splitmix64_seed0.txt")) if l[0] != "#"]
    for i, hexv in rows:
        x = (int(i) * 0x9E3779B97F4A7C15) % 2**64
        assert oracle.splitmix64(x) == int(hexv, 16)


def test_perturb_identities_and_bounds():
    rng = np.random.default_rng(1)
    for _ in range(2000):
        d = int(rng.integers(0, 2**40))
        uid = int(rng.integers(0, 2**63))
        k = int(rng.integers(1, 64))
        amp = int(rng.integers(0, 65536))
        assert oracle.perturb(d, uid, 0, 0x5EED, amp) == d          # scenario 0 unperturbed
        assert oracle.perturb(d, uid, k, 0x5EED, 0) == d            # zero amplitude
        v = oracle.perturb(d, uid, k, 0x5EED, amp)
        # delta in [-amp, amp]  =>  floor(d (65536-amp)/65536) <= v <= floor(d (65536+amp)/65536)
        assert (d * (65536 - amp)) >> 16 <= v <= (d * (65536 + amp)) >> 16
    # delta is (close to) uniform on [-amp, amp]: mean ~ 0, both extremes reachable
    amp = 3
    ds = [oracle.perturb(65536, u, 5, 0x5EED, amp) - 65536 for u in range(4000)]
    assert set(ds) == {-3, -2, -1, 0, 1, 2, 3}
    assert abs(np.mean(ds)) < 0.15


# ------------------------------------------------------------------ SPEC worked examples
def test_spec_examples():
    one = w.Topology(1, 1, 1)
    assert oracle.replay(_tm(one, [[("c", 5)]]))["iter"][0] == 5
    r = oracle.replay(_tm(one, [[("c", 5)]]), times=True)
    assert r["start"][0, 0] == 0 and r["finish"][0, 0] == 5
    assert oracle.replay(_tm(w.Topology(1, 2, 1), [[("c", 3)], [("c", 7)]]))["iter"][0] == 7
    assert oracle.replay(_tm(one, [[("c", 3), ("c", 7)]]))["iter"][0] == 10
    assert oracle.replay(_tm(one, [[]]))["iter"][0] == 0
    # S:319 (Fig. 5): the send finishes at 12, the matched receive is locally ready at 3
    tm = _tm(w.Topology(1, 2, 1), [[("c", 12), ("p2p", w.SEND_NEXT, 0)],
                                   [("c", 3), ("p2p", w.RECV_PREV, 0)]])
    r = oracle.replay(tm, times=True)
    assert r["start"][0, 3] == 12 and r["finish"][0, 3] == 12 and r["iter"][0] == 12


def test_group_counts_tp2pp2dp2():
    """tp=2, pp=2, dp=2 -> 4 TP groups of 2, 4 DP groups of 2 (and, with one op of each
    role per stage, the closed-form counts of row a2 for EP / EDP as well)."""
    for tp, pp, dp, ep in [(2, 2, 2, 1), (2, 2, 4, 2), (1, 3, 4, 4), (3, 2, 6, 3)]:
        topo = w.Topology(tp, pp, dp, ep)
        ops = [("coll", w.ROLE_TP, 0, 1), ("coll", w.ROLE_DP, 0, 1), ("coll", w.ROLE_EP, 3, 1),
               ("coll", w.ROLE_EDP, 1, 1), ("coll", w.ROLE_WORLD, 5, 1)]
        ex = oracle.expand(_tm(topo, [ops] * pp))
        sizes = np.diff(ex["ptr"])
        role = (ex["uid"] >> np.uint64(56)).astype(int)
        count = {r: int((role == r).sum()) for r in range(1, 6)}
        assert count == {1: pp * dp, 2: tp * pp, 3: tp * pp * dp // ep, 4: tp * pp * ep, 5: 1}
        for r, n in [(1, tp), (2, dp), (3, ep), (4, dp // ep), (5, tp * pp * dp)]:
            assert set(sizes[role == r].tolist()) == {n}
        # members by brute-force coordinate enumeration (TP group = same (pp, dp))
        W = tp * pp * dp
        coords = {r: (r % tp, (r // tp) % pp, r // (tp * pp)) for r in range(W)}
        per_rank = len(ops)
        for g in np.nonzero(role == 1)[0]:
            mem = ex["mem"][ex["ptr"][g]:ex["ptr"][g + 1]] // per_rank
            assert len({coords[int(m)][1:] for m in mem}) == 1


# ------------------------------------------------------------------ pipeline closed forms
@pytest.mark.parametrize("f,b", [(1, 1), (1, 2), (3, 5)])
def test_1f1b_closed_form(f, b):
    """(m + p - 1)(f + b): the textbook 1F1B bubble with free P2P (SURVEY §8.2 pins)."""
    for p in range(1, 7):
        for m in range(1, 10):
            tm = w.uniform_pipeline(1, p, 1, m, f_ns=f, b_ns=b, dense_tp_layout=False,
                                    dp_ar_ns=-1, opt_ns=-1)
            assert oracle.replay(tm)["iter"][0] == (m + p - 1) * (f + b), (p, m)


def test_1f1b_p2_with_p2p_cost():
    """p = 2 with per-message cost c: (m + 1)(f + b + c)."""
    for m in range(1, 12):
        for f, b, c in itertools.product([1, 2, 5], [1, 3, 4], [0, 1, 7, 13]):
            tm = w.uniform_pipeline(1, 2, 1, m, f_ns=f, b_ns=b, p2p_c=c, dense_tp_layout=False,
                                    dp_ar_ns=-1, opt_ns=-1)
            assert oracle.replay(tm)["iter"][0] == (m + 1) * (f + b + c)


def test_interleaved_closed_form():
    """Interleaved 1F1B with free P2P: (m v + p - 1)(f_c + b_c)."""
    for p in (2, 3, 4):
        for v in (2, 3):
            for m in (p, 2 * p, 3 * p):
                tm = w.uniform_pipeline(1, p, 1, m, vpp=v, f_ns=2, b_ns=3, dense_tp_layout=False,
                                        dp_ar_ns=-1, opt_ns=-1)
                assert oracle.replay(tm)["iter"][0] == (m * v + p - 1) * 5, (p, v, m)


def test_c1_closed_form():
    """BASELINE.json C1 (TP2 PP2 DP2, 4 layers, m=4, uniform costs): f = 4400, b = 8400,
    T = (m+p-1)(f+b) + DP AR + OPT = 64,800 ns; with c = 50: (m+1)(f+b+c) + 800 = 65,050 ns.
    Peaks: static + min(p-s, m) * 4 MiB."""
    r = oracle.replay(w.config("C1"))
    assert r["iter"][0] == 64_800
    r50 = oracle.replay(w.config("C1", p2p_c=50))
    assert r50["iter"][0] == 65_050
    peak = r["peak"][0]
    for rank in range(8):
        stage = (rank // 2) % 2
        assert peak[rank] == (1 << 30) + min(2 - stage, 4) * 4 * (1 << 20)
    assert set(peak.tolist()) == {1_082_130_432, 1_077_936_128}


def test_ring_allreduce_cost_model():
    """p = 1, DP ring all-reduce: T = m (f + b) + 2 (n - 1)(alpha + ceil(ceil(B/n) 1000 / beta))
    ((K-1) reduce rounds + (K-1) broadcast rounds, each moving B/K)."""
    for n in (2, 4, 8, 16):
        for B in (1, 1000, 10**6, 123_456_789):
            dur = w.coll_ns(w.COLL_AR, n, B, list(range(0, 8 * n, 8)))  # inter-node tier
            steps, per = 2 * (n - 1), -(-B // n)
            assert dur == steps * (15_000 + -(-per * 1000 // 50_000))
            tm = w.uniform_pipeline(1, 1, n, 3, f_ns=10, b_ns=20, dense_tp_layout=False,
                                    dp_ar_ns=dur, opt_ns=0)
            assert oracle.replay(tm)["iter"][0] == 3 * 30 + dur


def test_memory_closed_forms():
    """1F1B: peak_s = static + min(p - s, m) A; interleaved: static + min(nw_s + 1, m v) A with
    nw_s = min((p-s-1) 2 + (v-1) p, m v) (S:174 '(warmup+1) live activations')."""
    A = 1000
    for p in range(1, 8):
        for m in range(1, 12):
            tm = w.uniform_pipeline(1, p, 1, m, dense_tp_layout=False, act_bytes=A, static_bytes=7,
                                    dp_ar_ns=-1, opt_ns=-1)
            pk = oracle.replay(tm)["peak"][0]
            assert pk.tolist() == [7 + min(p - s, m) * A for s in range(p)]
    for p in range(2, 6):
        for v in (2, 3):
            for m in (p, 2 * p, 3 * p):
                tm = w.uniform_pipeline(1, p, 1, m, vpp=v, dense_tp_layout=False, act_bytes=A,
                                        static_bytes=0, dp_ar_ns=-1, opt_ns=-1)
                pk = oracle.replay(tm)["peak"][0]
                exp = [min(min((p - s - 1) * 2 + (v - 1) * p, m * v) + 1, m * v) * A for s in range(p)]
                assert pk.tolist() == exp, (p, v, m)


# ------------------------------------------------------------------ brute force
@pytest.mark.parametrize("seed", range(40))
def test_brute_force_random_tiny(seed):
    tm = w.random_templates(seed, max_world=6, max_ops=6, max_dur=20)
    if tm.n_nodes > 40:
        pytest.skip("too large for path enumeration")
    T, fin = brute.iteration_time(tm)
    r = oracle.replay(tm, times=True)
    assert r["iter"][0] == T
    assert r["finish"][0].tolist() == fin


def test_brute_force_1f1b_demo():
    """1F1B demo (PP=2, GA=2, all durations 10, comm 1) -> exhaustive enumeration."""
    tm = w.uniform_pipeline(1, 2, 1, 2, f_ns=10, b_ns=10, p2p_c=1, dense_tp_layout=False,
                            dp_ar_ns=-1, opt_ns=-1)
    T, fin = brute.iteration_time(tm)
    assert oracle.replay(tm)["iter"][0] == T == 3 * (10 + 10 + 1)


# ------------------------------------------------------------------ invariants
def _check_invariants(tm, r, k=0):
    ex = oracle.expand(tm)
    st, fi = r["start"][k], r["finish"][k]
    # (i) collective members share start and finish (single-group nodes)
    ngroups = np.zeros(tm.n_nodes, np.int64)
    for g in range(ex["groups"]):
        mem = ex["mem"][ex["ptr"][g]:ex["ptr"][g + 1]]
        ngroups[mem] += 1
    for g in range(ex["groups"]):
        mem = ex["mem"][ex["ptr"][g]:ex["ptr"][g + 1]]
        single = mem[ngroups[mem] == 1]
        if len(single) > 1:
            assert len(set(st[single].tolist())) == 1
            assert len(set(fi[single].tolist())) == 1
    return ngroups


def test_invariants_random_and_scaled():
    for seed in range(30):
        tm = w.random_templates(seed, max_world=16, max_ops=30)
        r = oracle.replay(tm, 3, amp_q16=6554, kind_mask=7, times=True)
        ng = _check_invariants(tm, r, 2)
        # chain invariants per rank
        N = tm.n_nodes
        comp = ng == 0
        for k in range(3):
            st, fi = r["start"][k], r["finish"][k]
            assert (fi >= st).all()
            # walk ranks
            off = 0
            for rank in range(tm.topo.world):
                s = (rank // tm.topo.tp) % tm.topo.pp if tm.topo.rank_order == 0 else rank // (tm.topo.tp * tm.topo.dp)
                L = len(tm.stage(s))
                for i in range(off, off + L):
                    prev = fi[i - 1] if i > off else 0
                    if comp[i]:
                        assert st[i] == prev
                    else:
                        assert st[i] >= prev
                off += L
            assert off == N
            assert r["iter"][k] == (fi.max() if N else 0)


def test_dp_replicas_identical_uniform():
    """with unperturbed costs, DP replicas replay bit-identically."""
    tm = w.scaled("C2")
    r = oracle.replay(tm, times=True, peaks=True)
    t = tm.topo
    per = tm.n_nodes // t.dp
    fi = r["finish"][0].reshape(t.dp, per)
    assert (fi == fi[0]).all()
    assert tm.n_nodes == t.dp * per                   # (iv) node count = dp x replica nodes


def test_monotone_and_off_critical_path():
    """(vi) monotone in any duration; (viii) stretching a node with slack leaves T alone."""
    tm = w.uniform_pipeline(1, 3, 1, 4, f_ns=10, b_ns=20, p2p_c=3, dense_tp_layout=False,
                            dp_ar_ns=-1, opt_ns=-1)
    base = oracle.replay(tm, times=True)
    T0 = base["iter"][0]
    rng = np.random.default_rng(0)
    for _ in range(20):
        i = int(rng.integers(0, len(tm.ops)))
        t2 = w.Templates(tm.topo, tm.ops.copy(), tm.tmpl_ptr, tm.static_mem)
        t2.ops["dur_ns"][i] += int(rng.integers(1, 50))
        assert oracle.replay(t2)["iter"][0] >= T0
    # (viii) S:496: a node with slack. Stage 1's compute (3 ns) waits for the send that stage 0
    # finishes at 10, so it has 7 ns of slack: stretching it by up to 7 keeps T, by 8 adds 1.
    t = w.Topology(1, 2, 1)
    for extra, T in [(0, 15), (7, 15), (8, 16)]:
        tm2 = _tm(t, [[("c", 10), ("p2p", w.SEND_NEXT, 0), ("c", 5)],
                      [("c", 3 + extra), ("p2p", w.RECV_PREV, 0), ("c", 5)]])
        assert oracle.replay(tm2)["iter"][0] == T


def test_relabel_invariance():
    """Reading Z1: T does not depend on the rank numbering; per-rank results permute."""
    for name in ("C1",):
        tm = w.config(name)
        r0 = oracle.replay(tm, 2, amp_q16=0)
        t2 = w.Templates(w.Topology(tm.topo.tp, tm.topo.pp, tm.topo.dp, 1, 1, w.ORDER_MEGATRON),
                         tm.ops, tm.tmpl_ptr, tm.static_mem)
        r1 = oracle.replay(t2, 2, amp_q16=0)
        assert (r0["iter"] == r1["iter"]).all()
        assert sorted(r0["peak"][0].tolist()) == sorted(r1["peak"][0].tolist())


# ------------------------------------------------------------------ error behaviour
def test_errors():
    t = w.Topology(1, 2, 1)
    # send/send with rendezvous semantics: a cycle
    dead = _tm(t, [[("p2p", w.SEND_NEXT, 1), ("p2p", w.RECV_NEXT, 1)],
                   [("p2p", w.SEND_PREV, 1), ("p2p", w.RECV_PREV, 1)]])
    with pytest.raises(oracle.OracleError) as e:
        oracle.replay(dead)
    assert e.value.name == "DEADLOCK"
    with pytest.raises(oracle.OracleError) as e:
        oracle.expand(dead)
    assert e.value.name == "DEADLOCK"
    # the same pair in the right order is fine
    ok = _tm(t, [[("p2p", w.SEND_NEXT, 1), ("p2p", w.RECV_NEXT, 1)],
                 [("p2p", w.RECV_PREV, 1), ("p2p", w.SEND_PREV, 1)]])
    assert oracle.replay(ok)["iter"][0] == 2
    unmatched = _tm(t, [[("p2p", w.SEND_NEXT, 1)], [("c", 1)]])
    with pytest.raises(oracle.OracleError) as e:
        oracle.replay(unmatched)
    assert e.value.name == "TEMPLATE_MISMATCH"
    world_mismatch = _tm(t, [[("coll", w.ROLE_WORLD, 0, 1)], [("c", 1)]])
    with pytest.raises(oracle.OracleError) as e:
        oracle.replay(world_mismatch)
    assert e.value.name == "TEMPLATE_MISMATCH"
    neg = _tm(w.Topology(1, 1, 1), [[("c", 1, 5, 0), ("c", 1, 0, 6)]])
    with pytest.raises(oracle.OracleError) as e:
        oracle.replay(neg)
    assert e.value.name == "NEGATIVE_MEMORY"
    with pytest.raises(oracle.OracleError) as e:
        oracle.replay(_tm(w.Topology(1, 1, 3, 2), [[("c", 1)]]))
    assert e.value.name == "INVALID_SPEC"

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


GOLD_K = 0x9E3779B97F4A7C15
MIX_K = 0xBF58476D1CE4E5B9
M64 = 2**64 - 1


def test_perturb_worked_examples():
    """Reading Z8 composed with SplitMix64's published outputs (tests/golden/splitmix64_seed0.txt):
    the seed is chosen so that x = seed ^ k*G ^ uid*M is 0, G or 2G, i.e. h is published output
    1, 2 or 3; the rest is worked by hand (Z8 worked examples):
      h = 0xE220A8397B1DCDAF, h>>40 = 14819496, mod 13109 = 6326, delta = -228,
          d = 10^6 -> 10^6 * 65308 >> 16 = 996520                        (amp 6554)
      h = 0x6E789E6AA1B965F4, h>>40 = 7239838, mod 201 = 19, delta = -81,
          d = 4400 -> 4400 * 65455 >> 16 = 4394                           (amp 100)
      h = 0x06C45D188009454F, h>>40 = 443485, mod 131071 = 50272, delta = -15263,
          d = 2^40 -> 2^24 * 50273 = 843440979968                         (amp 65535)
    A k / uid mix-up, a different shift of h or a wrong delta offset all miss these."""
    cases = [  # (k, uid, x target, amp, d, expected d')
        (1, 1, 0, 6554, 10**6, 996520),
        (2, (5 << 32) | 7, GOLD_K, 100, 4400, 4394),
        (63, (6 << 56) | (12345 << 24) | 9, (2 * GOLD_K) & M64, 65535, 2**40, 843440979968),
    ]
    for k, uid, x, amp, d, want in cases:
        seed = x ^ ((k * GOLD_K) & M64) ^ ((uid * MIX_K) & M64)  # input chosen, not an expected value
        assert oracle.perturb(d, uid, k, seed, amp) == want, (k, uid)


def _golden_levels():
    rows, kv = [], {}
    for line in open(os.path.join(GOLD, "levels_hand.txt")):
        if not line.strip() or line.startswith("#"):
            continue
        p = line.split()
        if p[0] == "A":
            rows.append((int(p[1]), int(p[2]), int(p[3])))
        else:
            kv[p[0]] = [int(x) for x in p[1:]]
    return rows, kv


def test_levels_hand_worked():
    """Row a5 (reading R2) against tests/golden/levels_hand.txt, derived by hand."""
    rows, kv = _golden_levels()
    ex = oracle.expand(w.uniform_pipeline(1, 2, 2, 2))
    got = sorted((int(ex["mem"][ex["ptr"][g]]), int(ex["mem"][ex["ptr"][g] + 1]), int(ex["level"][g]))
                 for g in range(ex["groups"]))
    assert got == sorted(rows) and ex["levels"] == kv["A_levels"][0]
    c1 = oracle.expand(w.config("C1"))
    assert c1["levels"] == kv["C1_levels"][0]
    role = (c1["uid"] >> np.uint64(56)).astype(int)
    dp = [int(g) for g in np.nonzero(role == w.ROLE_DP)[0]]
    per_rank = c1["nodes"] // 8
    by_stage = {}
    for g in dp:  # stage of a DP group = stage of its members (TP_PP_DP rank order)
        r = int(c1["mem"][c1["ptr"][g]]) // per_rank
        by_stage.setdefault((r // 2) % 2, set()).add(int(c1["level"][g]))
    assert by_stage == {0: {kv["C1_dp_levels"][0]}, 1: {kv["C1_dp_levels"][1]}}


# ------------------------------------------------------------------ SPEC worked examples
def _spec_golden():
    """tests/golden/spec_worked_examples.txt: name -> {key: value} (values as printed by SPEC)."""
    out = {}
    for line in open(os.path.join(GOLD, "spec_worked_examples.txt")):
        if line.startswith("#") or not line.strip():
            continue
        name, _src, *kv = line.split()
        out[name] = dict(x.split("=") for x in kv)
    return out


def test_spec_examples():
    G = _spec_golden()
    T = lambda name: int(G[name]["T"])
    one = w.Topology(1, 1, 1)
    assert oracle.replay(_tm(one, [[("c", 5)]]))["iter"][0] == T("single_node_5")
    r = oracle.replay(_tm(one, [[("c", 5)]]), times=True)
    assert r["start"][0, 0] == int(G["one_node_start0"]["start"]) and r["finish"][0, 0] == T("one_node_start0")
    assert oracle.replay(_tm(w.Topology(1, 2, 1), [[("c", 3)], [("c", 7)]]))["iter"][0] == T("two_independent_3_7")
    assert oracle.replay(_tm(one, [[("c", 3), ("c", 7)]]))["iter"][0] == T("chain_3_7")
    assert oracle.replay(_tm(one, [[]]))["iter"][0] == T("empty_graph")
    # S:319 (Fig. 5): the send finishes at 12, the matched receive is locally ready at 3
    tm = _tm(w.Topology(1, 2, 1), [[("c", 12), ("p2p", w.SEND_NEXT, 0)],
                                   [("c", 3), ("p2p", w.RECV_PREV, 0)]])
    r = oracle.replay(tm, times=True)
    want = int(G["fig5_send12_recv3"]["recv_start"])
    assert r["start"][0, 3] == want and r["finish"][0, 3] == want and r["iter"][0] == want
    # pp=2, ga=2 1F1B stage orders
    order = {s: ",".join(f"{it[0]}{it[1] + 1}" for it in w.schedule_1f1b(2, s, 2) if it[0] != "P") for s in (0, 1)}
    assert order[0] == G["pp2_ga2_stage_orders"]["stage0"] and order[1] == G["pp2_ga2_stage_orders"]["stage1"]
    # tp=2 pp=2 dp=2 -> 4 TP, 4 DP groups (one op of each role per stage)
    ex = oracle.expand(_tm(w.Topology(2, 2, 2), [[("coll", w.ROLE_TP, 0, 1), ("coll", w.ROLE_DP, 0, 1)]] * 2))
    role = (ex["uid"] >> np.uint64(56)).astype(int)
    want = G["tp2pp2dp2_group_counts"]
    assert int((role == 1).sum()) == int(want["TP"]) and int((role == 2).sum()) == int(want["DP"])


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
        # every role's member sets = the classes of ranks sharing the role's fixed coordinates
        # (row a2): DP = same (tp, pp); EP = same (tp, pp, edp = dp // ep), ep_i = dp % ep varies;
        # EDP = same (tp, pp, ep_i); WORLD = everyone
        key = {2: lambda c: (c[0], c[1]), 3: lambda c: (c[0], c[1], c[2] // ep),
               4: lambda c: (c[0], c[1], c[2] % ep), 5: lambda c: ()}
        for rr, f in key.items():
            want = {}
            for r, c in coords.items():
                want.setdefault(f(c), set()).add(r)
            got = [frozenset(int(m) // per_rank for m in ex["mem"][ex["ptr"][g]:ex["ptr"][g + 1]])
                   for g in np.nonzero(role == rr)[0]]
            assert sorted(map(sorted, got)) == sorted(map(sorted, want.values())), (tp, pp, dp, ep, rr)
            if rr == 3:  # an EP group spans ep consecutive dp coordinates (ep carved out of dp)
                for m in got:
                    assert sorted(coords[r][2] % ep for r in m) == list(range(ep))


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


# ------------------------------------------------------------------ fixed-point cross-check
@pytest.mark.parametrize("seed", range(12))
def test_fixed_point_matches_des_random(seed):
    """a Bellman-Ford-style fixed point on the weighted DAG equals the DES on
    medium random graphs (far beyond path enumeration), per node."""
    tm = w.random_templates(seed, max_world=24, max_ops=30)
    T, fin = brute.fixed_point(tm)
    r = oracle.replay(tm, times=True)
    assert T == r["iter"][0] and fin == r["finish"][0].tolist()


@pytest.mark.parametrize("name", ["C1"])
def test_fixed_point_matches_des_configs(name):
    tm = w.config(name)
    T, fin = brute.fixed_point(tm)
    r = oracle.replay(tm, times=True)
    assert T == r["iter"][0] == 64800 and fin == r["finish"][0].tolist()
    tm = w.uniform_pipeline(2, 3, 2, 6, vpp=3, p2p_c=7)  # interleaved, P2P cost
    T, fin = brute.fixed_point(tm)
    assert fin == oracle.replay(tm, times=True)["finish"][0].tolist()

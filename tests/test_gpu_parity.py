"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Integer times and bytes => the bar is bit-exact equality everywhere (north_star).
"""
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


# ------------------------------------------------------------------ rows a1-a5: the CSR DAG
def _check_csr(P, tm):
    g = _graph(P, tm)
    st = g.stats()
    ex = oracle.expand(tm)
    assert (st["nodes"], st["groups"], st["memberships"], st["levels"]) == (
        ex["nodes"], ex["groups"], ex["memberships"], ex["levels"])
    # node SoA: every rank holds its stage template (rank-major, program order)
    rank_ptr = g.export("rank_ptr")
    node_rank = g.export("node_rank")
    dur = g.export("node_dur")
    alloc, free = g.export("node_alloc"), g.export("node_free")
    t = tm.topo
    for r in range(t.world):
        s = (r // t.tp) % t.pp if t.rank_order == 0 else r // (t.tp * t.dp)
        a, b = rank_ptr[r], rank_ptr[r + 1]
        tmpl = tm.stage(s)
        assert b - a == len(tmpl)
        assert (node_rank[a:b] == r).all()
        assert (dur[a:b] == tmpl["dur_ns"]).all()
        assert (alloc[a:b] == tmpl["mem_alloc"]).all() and (free[a:b] == tmpl["mem_free"]).all()
    # groups: same uid set, same members / duration / level per uid
    uid = g.export("grp_uid")
    gptr = g.export("grp_ptr")
    mem = g.export("grp_mem")
    gdur = g.export("grp_dur")
    glvl = g.export("grp_level")
    assert len(set(uid.tolist())) == len(uid)
    o_index = {int(u): i for i, u in enumerate(ex["uid"])}
    assert set(o_index) == set(int(u) for u in uid)
    for i, u in enumerate(uid):
        j = o_index[int(u)]
        mine = np.sort(mem[gptr[i]:gptr[i + 1]])
        theirs = ex["mem"][ex["ptr"][j]:ex["ptr"][j + 1]]
        assert np.array_equal(mine, theirs), (hex(int(u)), mine, theirs)
        assert gdur[i] == ex["dur"][j] and glvl[i] == ex["level"][j]
    assert (np.diff(glvl) >= 0).all()  # sorted by level (frontier tiles are contiguous)
    # node -> group lists are the inverse of group -> members
    ngptr = g.export("node_gptr")
    ngrp = g.export("node_grp")
    for n in range(0, st["nodes"], max(1, st["nodes"] // 500)):
        for h in ngrp[ngptr[n]:ngptr[n + 1]]:
            assert n in mem[gptr[h]:gptr[h + 1]]
    g.close()


@pytest.mark.parametrize("name", ["C1", "C2s", "C3s", "C4s", "C5s"])
def test_csr_configs(prism, name):
    tm = w.config(name) if name == "C1" else w.scaled(name[:2])
    _check_csr(prism, tm)


@pytest.mark.parametrize("seed", range(12))
def test_csr_random(prism, seed):
    _check_csr(prism, w.random_templates(seed, max_world=32, max_ops=40))


# ------------------------------------------------------------------ rows a6-a9: replay + memory
def _check_replay(P, tm, S, amp=6554, mask=7, times=True, seed=0x5EED, algo="auto"):
    g = _graph(P, tm)
    it = g.replay(S, seed=seed, amp_q16=amp, kind_mask=mask, record=True, algo=algo)
    if algo != "auto":
        assert g.last_algo() == algo
    ref = oracle.replay(tm, S, seed=seed, amp_q16=amp, kind_mask=mask, times=times,
                        threads=min(NPROC, S))
    assert np.array_equal(it, ref["iter"]), (it[:8], ref["iter"][:8])
    assert np.array_equal(g.peak_memory(), ref["peak"][0])
    if times:
        W = tm.topo.world
        ranks = range(W) if W <= 64 else np.random.default_rng(0).choice(W, 64, replace=False)
        for k in sorted({0, min(1, S - 1), S - 1}):
            for r in ranks:
                st, fi, coords = g.query_rank(int(r), k)
                rp = g.export("rank_ptr")
                a, b = rp[r], rp[r + 1]
                assert np.array_equal(fi, ref["finish"][k, a:b]), (k, r)
                assert np.array_equal(st, ref["start"][k, a:b]), (k, r)
    g.close()
    return it


@pytest.mark.parametrize("algo", ["levels", "cells"])
@pytest.mark.parametrize("seed", range(40))
def test_replay_random(prism, seed, algo):
    tm = w.random_templates(seed, max_world=32, max_ops=40)
    S = [1, 2, 3, 5, 17, 33, 64, 70][seed % 8]
    if algo == "cells" and tm.topo.tp > 8:
        pytest.skip("cells need tp <= 8")
    _check_replay(prism, tm, S, algo=algo)


def test_c1_closed_form_gpu(prism):
    assert _check_replay(prism, w.config("C1"), 1, amp=0)[0] == 64_800
    assert _check_replay(prism, w.config("C1", p2p_c=50), 1, amp=0)[0] == 65_050
    g = _graph(prism, w.config("C1"))
    pk = g.peak_memory()
    assert sorted(set(pk.tolist())) == [1_077_936_128, 1_082_130_432]


@pytest.mark.parametrize("algo", ["levels", "cells"])
@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_replay_scaled_configs(prism, name, algo):
    _check_replay(prism, w.scaled(name), 64, times=True, algo=algo)


@pytest.mark.parametrize("algo", ["levels", "cells"])
def test_fin_array_all_nodes(prism, algo):
    """Every node-scenario finish of the recorded replay equals the oracle (scenario-fastest)."""
    tm = w.scaled("C3")
    g = _graph(prism, tm)
    S = 64
    g.replay(S, amp_q16=6554, kind_mask=7, algo=algo)
    fin = g.export("fin", scen_pad=64).reshape(-1, 64)
    ref = oracle.replay(tm, S, amp_q16=6554, kind_mask=7, times=True, threads=NPROC)
    assert np.array_equal(fin[:, :S].T, ref["finish"])


def test_deterministic_and_record_off(prism):
    tm = w.scaled("C2")
    g = _graph(prism, tm)
    a = g.replay(64, amp_q16=6554, kind_mask=7)
    b = g.replay(64, amp_q16=6554, kind_mask=7)
    c = g.replay(64, amp_q16=6554, kind_mask=7, record=False)
    d = g.replay(64, amp_q16=6554, kind_mask=7, record=False, algo="levels")
    e = g.replay(130, amp_q16=6554, kind_mask=7, algo="cells")  # 3 scenario chunks
    assert np.array_equal(a, b) and np.array_equal(a, c) and np.array_equal(a, d)
    assert np.array_equal(e[:64], a)
    g.replay(64, amp_q16=6554, kind_mask=7, record=False)
    with pytest.raises(prism.PrismError) as e:
        g.query_rank(0, 0)
    assert e.value.name == "PRISM_E_NOT_REPLAYED"


def test_edge_cases(prism):
    # all-empty templates
    tm = w.assemble(w.Topology(2, 2, 2), [np.zeros(0, w.OP_DTYPE)] * 2, [5, 6])
    g = _graph(prism, tm)
    assert g.replay(3).tolist() == [0, 0, 0]
    assert g.peak_memory().tolist() == [5, 5, 6, 6, 5, 5, 6, 6]
    # one stage empty, the other compute only; amplitude maximum
    b = w._StageBuilder()
    for d in (0, 1, 2**40):
        b.compute(d)
    tm = w.assemble(w.Topology(1, 2, 3), [b.array(), np.zeros(0, w.OP_DTYPE)], [0, 0])
    _check_replay(prism, tm, 9, amp=65535)
    with pytest.raises(prism.PrismError) as e:
        g.query_rank(99, 0)
    assert e.value.name == "PRISM_E_UNKNOWN_RANK"


@pytest.mark.parametrize("algo", ["levels", "cells"])
def test_world_collectives_large_groups(prism, algo):
    """WORLD collectives (one group spanning every rank) and EP/EDP groups."""
    for seed in range(100, 110):
        tm = w.random_templates(seed, max_world=64, max_ops=60)
        _check_replay(prism, tm, 64, times=False, algo=algo if tm.topo.tp <= 8 else "auto")


@pytest.mark.slow
@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_full_size(prism, name):
    """BASELINE.json full sizes in the bench launch configuration (auto schedule = the cell kernel,
    S = 64, +-10% jitter): all 64 iteration times, every rank's last finish in the first and last
    scenario, and every rank's peak equal the oracle's (the oracle on all host threads)."""
    tm = w.config(name)
    g = _graph(prism, tm)
    S = 64
    it = g.replay(S, amp_q16=6554, kind_mask=7)
    pk = g.peak_memory()
    ref = oracle.replay(tm, S, amp_q16=6554, kind_mask=7, peaks=False, threads=NPROC)
    assert np.array_equal(it, ref["iter"]), name
    assert np.array_equal(pk, oracle.replay(tm, 1)["peak"][0])
    for k in (0, S - 1):
        for rk in range(tm.topo.world):
            _, fi, _ = g.query_rank(rk, k)
            assert (fi[-1] if len(fi) else 0) == ref["rank_end"][k, rk], (name, k, rk)
    g.close()


@pytest.mark.slow
def test_full_size_c5_per_op_times(prism):
    """C5 at full size in the bench launch configuration (S = 64, cell kernel): every op's start and
    finish of sampled ranks (all stages, both scenario chunks) equal the oracle's, scenario by
    scenario (the oracle's per-node times of all 64 scenarios would take 18 GB: single scenarios)."""
    tm = w.config("C5")
    g = _graph(prism, tm)
    S = 64
    g.replay(S, amp_q16=6554, kind_mask=7)
    assert g.last_algo() == "cells"
    rp = g.export("rank_ptr")
    rng = np.random.default_rng(64)
    ranks = sorted(set(rng.choice(tm.topo.world, 12, replace=False).tolist()) | {0, tm.topo.world - 1})
    for k in (0, 37, 63):
        ref = oracle.replay(tm, 1, scen_first=k, amp_q16=6554, kind_mask=7, times=True, peaks=False)
        for r in ranks:
            st, fi, _ = g.query_rank(r, k)
            a, b = rp[r], rp[r + 1]
            assert np.array_equal(st, ref["start"][0, a:b]) and np.array_equal(fi, ref["finish"][0, a:b]), (k, r)
    g.close()


def test_wide_tp_uses_levels(prism):
    """tp > 8 has no cell-kernel instantiation: the auto schedule falls back to one launch per
    frontier level, bit-exact as well; a multi-stream graph with tp > 8 is refused."""
    tm = w.uniform_pipeline(16, 2, 2, 4, p2p_c=30)
    it = _check_replay(prism, tm, 33, times=True)
    g = _graph(prism, tm)
    g.replay(2)
    assert g.last_algo() == "levels"
    ov = w.overlap_grad_reduce(tm)
    g2 = _graph(prism, ov)
    with pytest.raises(prism.PrismError):
        g2.replay(2)


def test_scenario_offset(prism):
    """prism_scenarios.first: a batch replays scenarios first .. first+n-1 of the sweep."""
    tm = w.scaled("C2")
    g = _graph(prism, tm)
    full = g.replay(40, amp_q16=6554, kind_mask=7)
    part = g.replay(13, amp_q16=6554, kind_mask=7, first=27)
    assert np.array_equal(part, full[27:40])
    ref = oracle.replay(tm, 5, scen_first=100, amp_q16=6554, kind_mask=7, threads=NPROC)
    assert np.array_equal(g.replay(5, amp_q16=6554, kind_mask=7, first=100, algo="levels"), ref["iter"])
    assert np.array_equal(g.replay(5, amp_q16=6554, kind_mask=7, first=100, algo="cells"), ref["iter"])
    st, fi, _ = g.query_rank(3, 4)
    r2 = oracle.replay(tm, 1, scen_first=104, amp_q16=6554, kind_mask=7, times=True)
    rp = g.export("rank_ptr")
    assert np.array_equal(st, r2["start"][0, rp[3]:rp[4]]) and np.array_equal(fi, r2["finish"][0, rp[3]:rp[4]])


@pytest.mark.parametrize("seed", range(30))
def test_single_scenario_rank_kernel_random(prism, seed):
    """S = 1 on the lane = rank kernel (PRISM_ALGO_RANKS): perturbed (first > 0) and unperturbed,
    with and without per-node durations."""
    tm = w.random_templates(seed, max_world=64, max_ops=40)
    if tm.topo.tp & (tm.topo.tp - 1):
        pytest.skip("the rank kernel needs tp a power of two")
    g = _graph(prism, tm)
    first = [0, 1, 9][seed % 3]
    it = g.replay(1, amp_q16=6554, kind_mask=7, first=first, algo="ranks")
    assert g.last_algo() == "ranks"
    ref = oracle.replay(tm, 1, scen_first=first, amp_q16=6554, kind_mask=7, times=True)
    assert np.array_equal(it, ref["iter"])
    rp = g.export("rank_ptr")
    for r in range(tm.topo.world):
        st, fi, _ = g.query_rank(r, 0)
        assert np.array_equal(fi, ref["finish"][0, rp[r]:rp[r + 1]]) and np.array_equal(st, ref["start"][0, rp[r]:rp[r + 1]])
    if seed % 2:
        d = np.random.default_rng(seed).integers(0, 700, tm.n_nodes)
        g.set_durations(node_dur=d)
        it = g.replay(1, amp_q16=6554, kind_mask=7, first=first)
        assert g.last_algo() == "ranks"
        assert np.array_equal(it, oracle.replay(tm, 1, scen_first=first, amp_q16=6554, kind_mask=7, node_dur=d)["iter"])


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_single_scenario_rank_kernel_configs(prism, name):
    tm = w.config(name) if name == "C1" else w.scaled(name)
    g = _graph(prism, tm)
    for first in (0, 5):
        it = g.replay(1, amp_q16=6554, kind_mask=7, first=first)
        assert g.last_algo() == "ranks"
        ref = oracle.replay(tm, 1, scen_first=first, amp_q16=6554, kind_mask=7)
        assert np.array_equal(it, ref["iter"])
        path, T = g.critical_path(0)
        rpath, rT = oracle.critical_path(tm, first, amp_q16=6554, kind_mask=7)
        assert T == rT and np.array_equal(path, rpath)


@pytest.mark.slow
def test_single_scenario_full_size_c5(prism):
    tm = w.config("C5")
    g = _graph(prism, tm)
    it = g.replay(1, amp_q16=6554, kind_mask=7, first=3)
    assert g.last_algo() == "ranks"
    assert it[0] == oracle.replay(tm, 1, scen_first=3, amp_q16=6554, kind_mask=7, peaks=False)["iter"][0]


@pytest.mark.slow
@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_single_scenario_full_size_configs(prism, name):
    """One perturbed scenario of the full-size configs (segment path for C2 / C3, the cell kernel
    for C4's EP-CTA plan): T and every rank's last finish against the oracle."""
    tm = w.config(name)
    g = _graph(prism, tm)
    it = g.replay(1, amp_q16=6554, kind_mask=7, first=5)
    assert g.last_algo() == ("cells" if name == "C4" else "ranks")
    ref = oracle.replay(tm, 1, scen_first=5, amp_q16=6554, kind_mask=7, threads=NPROC)
    assert it[0] == ref["iter"][0]
    rp = g.export("rank_ptr")
    W = tm.topo.world
    for r in np.random.default_rng(5).choice(W, 48, replace=False):
        st, fi, _ = g.query_rank(int(r), 0)
        assert fi[-1] == ref["rank_end"][0, r], (name, r)
    assert np.array_equal(g.peak_memory(), ref["peak"][0])  # program order: any scenario's


# ------------------------------------------------------------------ asynchronous build pipeline
def test_async_builds_pipelined(prism):
    """Ten graphs built back to back with asynchronous builds on one stream (more than the four
    pinned staging buffers of the build upload, so the ring wraps while earlier uploads may still
    be queued behind a long replay), replayed in reverse order and destroyed out of order: every
    result equals the oracle's (a staging buffer reused before its copy completed would corrupt a
    graph's tables)."""
    import torch

    sh = torch.cuda.current_stream().cuda_stream
    big = prism.Graph(w.scaled("C5", 16), stream=sh, asynchronous=True)
    it_dev = torch.zeros(64, dtype=torch.int64, device="cuda")
    big.replay_async(it_dev.data_ptr(), 64, amp_q16=6554, kind_mask=7)  # keeps the stream busy
    tms = [w.random_templates(100 + i, max_world=32, max_ops=40) for i in range(10)]
    graphs = [prism.Graph(tm, stream=sh, asynchronous=True) for tm in tms]
    for i in reversed(range(10)):
        S = [1, 3, 17, 64][i % 4]
        it = graphs[i].replay(S, amp_q16=6554, kind_mask=7)
        ref = oracle.replay(tms[i], S, amp_q16=6554, kind_mask=7, times=False, threads=min(NPROC, S))
        assert np.array_equal(it, ref["iter"]), i
        assert np.array_equal(graphs[i].peak_memory(), ref["peak"][0]), i
        if i % 3 == 0:
            graphs[i].close()
    for g in graphs:
        g.close()
    big.close()


@pytest.mark.parametrize("ep", [1, 8])
def test_tp1_8192_ranks_on_cells(prism, ep):
    """TP = 1 at 8192 ranks (the paper's S.A/S.C/S.D shapes): one-rank cells cannot
    all be co-resident, so the replay runs replica cells (8 DP replicas per warp; EP CTAs when ep
    allows) instead of dropping to the level-by-level path; bit-exact against the oracle."""
    tm = w.uniform_pipeline(1, 8, 1024, 4, f_ns=700, b_ns=1300, p2p_c=40, dense_tp_layout=False)
    if ep > 1:
        t = tm.topo
        tm = w.Templates(w.Topology(t.tp, t.pp, t.dp, ep, t.vpp, t.rank_order), tm.ops, tm.tmpl_ptr, tm.static_mem)
    g = _graph(prism, tm)
    it = g.replay(64, amp_q16=6554, kind_mask=7)
    assert g.last_algo() == "cells"
    ref = oracle.replay(tm, 64, amp_q16=6554, kind_mask=7, threads=NPROC, times=True)
    assert np.array_equal(it, ref["iter"])
    assert np.array_equal(g.peak_memory(), ref["peak"][0])
    rp = g.export("rank_ptr")
    for r in (0, 4095, 8191):
        st, fi, _ = g.query_rank(r, 63)
        assert np.array_equal(fi, ref["finish"][63, rp[r]:rp[r + 1]])

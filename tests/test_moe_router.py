"""Row f4 inputs: the MoE mock router's balance-ratio schedule (Appendix F; Fig. 3
caption statistics) pinned to SPEC S:535-603's worked examples and properties, and its
effect on the oracle's replay / peak memory."""
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


def test_uniform_schedule_is_the_template_graph():
    tm = w.scaled("C4")
    d, a, f = M.moe_overrides(tm, np.ones((4, tm.topo.ep)))
    nt = oracle.node_table(tm)
    assert np.array_equal(d, nt["dur"])
    base = oracle.replay(tm, 2, amp_q16=6554, kind_mask=7)
    ov = oracle.replay(tm, 2, amp_q16=6554, kind_mask=7, node_dur=d, node_alloc=a, node_free=f)
    assert np.array_equal(base["iter"], ov["iter"]) and np.array_equal(base["peak"], ov["peak"])


def test_peak_memory_monotone_in_br():
    """heavier routing never lowers a rank's peak (activations scale with br, frees match)."""
    tm = w.scaled("C4")
    s = M.derive_schedule(M.FIG3_PROFILE, 16, tm.topo.ep, seed=1)
    peaks = []
    for bump in (0.0, 0.1, 0.5):
        d, a, f = M.moe_overrides(tm, s + bump)
        peaks.append(oracle.replay(tm, 1, node_dur=d, node_alloc=a, node_free=f)["peak"][0])
    assert (peaks[1] >= peaks[0]).all() and (peaks[2] >= peaks[1]).all() and (peaks[2] > peaks[0]).any()
    # and the imbalanced iteration is never shorter than the balanced one at the same mean load
    d0, _, _ = M.moe_overrides(tm, np.full_like(s, s.min()))
    d1, _, _ = M.moe_overrides(tm, s)
    assert oracle.replay(tm, 1, node_dur=d1)["iter"][0] >= oracle.replay(tm, 1, node_dur=d0)["iter"][0]

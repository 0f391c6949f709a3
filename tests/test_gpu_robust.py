"""Failure is loud and recoverable (include/prism.h prism_sync / prism_debug_set): a replay the
device watchdog aborts is reported as PRISM_E_DEADLOCK by the next synchronising call, asynchronous
callers learn it through prism_sync, and the next replay of the same graph is bit-exact again (the
guard kernel resets the ready slots an aborted replay left unwritten, so no stale same-parity value
can read as valid)."""
import os

import numpy as np
import pytest

import oracle
import workloads as w

pytestmark = pytest.mark.gpu

NPROC = min(16, os.cpu_count() or 1)


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


@pytest.mark.parametrize("cfg,S", [("C2", 64), ("C4", 33), ("C2", 1)])
def test_watchdog_abort_then_exact(prism, cfg, S):
    import torch

    tm = w.scaled(cfg)
    kw = dict(amp_q16=6554, kind_mask=7)
    ref = oracle.replay(tm, S, peaks=False, threads=NPROC, **kw)
    g = _graph(prism, tm)
    assert np.array_equal(g.replay(S, **kw), ref["iter"])  # a clean replay first (parity 0 slots)
    g.debug_set("watchdog_ns", 20_000_000)  # 20 ms
    g.debug_set("stall_unit", 3)  # warp 3 never arrives: its partners must time out
    out = torch.zeros(S, dtype=torch.int64, device="cuda")
    g.replay_async(out.data_ptr(), S, seed=77, **kw)  # different seed: stale slots would differ
    with pytest.raises(prism.PrismError) as e:
        g.sync()
    assert e.value.name == "PRISM_E_DEADLOCK"
    g.sync()  # reported once
    g.debug_set("stall_unit", -1)
    for seed in (0x5EED, 77):  # both parities after the abort
        r = oracle.replay(tm, S, seed=seed, peaks=False, threads=NPROC, **kw)
        assert np.array_equal(g.replay(S, seed=seed, **kw), r["iter"])
    s0, f0, _ = g.query_rank(0, S - 1)
    r = oracle.replay(tm, S, seed=77, times=True, threads=NPROC, **kw)
    assert np.array_equal(f0, r["finish"][S - 1][: len(f0)])
    assert np.array_equal(s0, r["start"][S - 1][: len(s0)])


def test_abort_reported_by_synchronous_replay(prism):
    tm = w.scaled("C3")
    g = _graph(prism, tm)
    g.debug_set("watchdog_ns", 20_000_000)
    g.debug_set("stall_unit", 0)
    with pytest.raises(prism.PrismError) as e:
        g.replay(40, amp_q16=6554, kind_mask=7)
    assert e.value.name == "PRISM_E_DEADLOCK"
    with pytest.raises(prism.PrismError):  # no recorded replay survives an abort
        g.query_rank(0, 0)
    g.debug_set("stall_unit", -1)
    ref = oracle.replay(tm, 40, amp_q16=6554, kind_mask=7, peaks=False, threads=NPROC)
    assert np.array_equal(g.replay(40, amp_q16=6554, kind_mask=7), ref["iter"])


def test_abort_of_earlier_async_replay_is_sticky(prism):
    """An aborted replay followed by a clean one before any sync: the abort is still reported."""
    import torch

    tm = w.scaled("C2")
    g = _graph(prism, tm)
    g.debug_set("watchdog_ns", 20_000_000)
    out = torch.zeros(32, dtype=torch.int64, device="cuda")
    g.debug_set("stall_unit", 1)
    g.replay_async(out.data_ptr(), 32, amp_q16=6554, kind_mask=7)
    g.debug_set("stall_unit", -1)
    g.replay_async(out.data_ptr(), 32, amp_q16=6554, kind_mask=7)
    with pytest.raises(prism.PrismError):
        g.sync()
    ref = oracle.replay(tm, 32, amp_q16=6554, kind_mask=7, peaks=False, threads=NPROC)
    g.replay_async(out.data_ptr(), 32, amp_q16=6554, kind_mask=7)
    g.sync()
    assert np.array_equal(out.cpu().numpy(), ref["iter"])


def test_debug_set_validation(prism):
    g = _graph(prism, w.config("C1"))
    with pytest.raises(prism.PrismError):
        g.debug_set("watchdog_ns", 10)

"""The seeded input generator (workloads/): schedule fixtures and config shapes."""
import numpy as np
import pytest

import workloads as w


def _fb(sched):
    return [f"{it[0]}{it[1] + 1}" for it in sched if it[0] in "FB"]


def test_spec_s159_stage_orders():
    """pp=2, ga=2 -> stage 0 = F1,F2,B1,B2; stage 1 = F1,B1,F2,B2."""
    assert _fb(w.schedule_1f1b(2, 0, 2)) == ["F1", "F2", "B1", "B2"]
    assert _fb(w.schedule_1f1b(2, 1, 2)) == ["F1", "B1", "F2", "B2"]


@pytest.mark.parametrize("p,m,v", [(2, 4, 1), (4, 8, 1), (4, 4, 2), (4, 8, 3), (3, 6, 2), (8, 3, 1)])
def test_forward_count(p, m, v):
    """per-stage forward count = ga * max(vpp, 1); backward count equals it; every
    (microbatch, chunk) appears once forward and once backward, forward first."""
    for s in range(p):
        sch = w.schedule_interleaved(p, s, m, v) if v > 1 else w.schedule_1f1b(p, s, m)
        F = [(it[1], it[2]) for it in sch if it[0] == "F"]
        B = [(it[1], it[2]) for it in sch if it[0] == "B"]
        assert len(F) == len(B) == m * max(v, 1)
        assert sorted(F) == sorted(B) == sorted(set(F))
        for key in F:
            fi = [i for i, it in enumerate(sch) if it[0] == "F" and (it[1], it[2]) == key][0]
            bi = [i for i, it in enumerate(sch) if it[0] == "B" and (it[1], it[2]) == key][0]
            assert fi < bi


def test_interleaved_preconditions():
    with pytest.raises(ValueError):
        w.schedule_interleaved(4, 0, 6, 2)  # m % p != 0 (reading Z14)
    with pytest.raises(ValueError):
        w.schedule_interleaved(4, 0, 0, 2)


def test_message_counts_match():
    """Every SEND_NEXT of stage s has a RECV_PREV on stage s+1 (and SEND_PREV / RECV_NEXT)."""
    for p, m, v in [(4, 8, 1), (4, 8, 2), (3, 9, 3), (2, 2, 1)]:
        cnt = {}
        for s in range(p):
            sch = w.schedule_interleaved(p, s, m, v) if v > 1 else w.schedule_1f1b(p, s, m)
            for it in sch:
                if it[0] == "P":
                    for bit in (1, 2, 4, 8):
                        if it[1] & bit:
                            cnt[(s, bit)] = cnt.get((s, bit), 0) + 1
        for s in range(p):
            assert cnt.get((s, w.SEND_NEXT), 0) == cnt.get(((s + 1) % p, w.RECV_PREV), 0)
            assert cnt.get((s, w.SEND_PREV), 0) == cnt.get(((s - 1) % p, w.RECV_NEXT), 0)


def test_op_layout():
    assert w.OP_DTYPE.itemsize == 48
    offs = {n: w.OP_DTYPE.fields[n][1] for n in w.OP_DTYPE.names}
    assert offs["label"] == 8 and offs["dur_ns"] == 16 and offs["mem_free"] == 40


@pytest.mark.parametrize("name,world,lo,hi", [("C2", 1024, 2.5e6, 3.0e6), ("C3", 4096, 9e6, 12e6),
                                              ("C4", 2048, 1.8e6, 2.8e6), ("C5", 8192, 17e6, 19.5e6)])
def test_config_shapes(name, world, lo, hi):
    tm = w.config(name)
    assert tm.topo.world == world
    assert lo <= tm.n_nodes <= hi, tm.n_nodes
    assert (tm.ops["dur_ns"] >= 0).all() and (tm.ops["dur_ns"] <= 2**40).all()
    for s in range(tm.topo.pp):
        run = np.cumsum(tm.stage(s)["mem_alloc"] - tm.stage(s)["mem_free"])
        assert run.min(initial=0) >= 0 and run[-1] == 0


def test_random_templates_deterministic():
    a = w.random_templates(7)
    b = w.random_templates(7)
    assert a.topo == b.topo and (a.ops == b.ops).all()

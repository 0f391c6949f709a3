"""CPU-side checks of the C ABI: the library loads, exports every symbol include/prism.h declares,
and its host-side validation / quotient plan (row a1-a5 sizes and levels) agrees with the oracle.
No compute call is made without a GPU (build returns PRISM_E_CUDA: there is no CPU fallback)."""
import os
import re

import numpy as np
import pytest

import oracle
import paper_2605_15617_b200 as prism
import workloads as w

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for f in os.listdir(os.path.join(ROOT, "include")):
        if f.endswith(".h"):
            txt = open(os.path.join(ROOT, "include", f)).read()
            names |= set(re.findall(r"PRISM_API[^;(]*?\b(prism_\w+)\s*\(", txt))
    return names


def test_library_exports_declared_symbols():
    prism.build_library()
    L = prism.lib()
    declared = _declared()
    assert len(declared) >= 12
    for name in declared:
        assert hasattr(L, name), name
    assert set(prism.EXPORTED_SYMBOLS) == declared
    assert L.prism_abi_version() == 4
    assert L.prism_status_string(5) == b"PRISM_E_DEADLOCK"


def _cmp_plan(tm):
    p = prism.plan(tm)
    ex = oracle.expand(tm)
    for k in ("world", "nodes", "groups", "memberships", "levels", "sync_nodes", "max_group"):
        assert p[k] == ex[k], (k, p[k], ex[k])


@pytest.mark.parametrize("name", ["C1", "C2", "C4"])
def test_plan_matches_oracle_configs(name):
    _cmp_plan(w.config(name))


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_plan_matches_oracle_scaled(name):
    _cmp_plan(w.scaled(name))


@pytest.mark.parametrize("seed", range(60))
def test_plan_matches_oracle_random(seed):
    _cmp_plan(w.random_templates(seed, max_world=32, max_ops=40))


def _tm(topo, stages):
    arrs = []
    for ops in stages:
        b = w._StageBuilder()
        for o in ops:
            if o[0] == "c":
                b.compute(o[1], alloc=o[2] if len(o) > 2 else 0, free=o[3] if len(o) > 3 else 0)
            elif o[0] == "coll":
                b.coll(o[1], o[2], o[3])
            else:
                b.op(w.KIND_P2P, o[2], mask=o[1])
        arrs.append(b.array() if ops else np.zeros(0, w.OP_DTYPE))
    return w.assemble(topo, arrs, [0] * topo.pp)


ERROR_CASES = {
    "PRISM_E_DEADLOCK": (w.Topology(1, 2, 1), [[("p2p", w.SEND_NEXT, 1), ("p2p", w.RECV_NEXT, 1)],
                                                [("p2p", w.SEND_PREV, 1), ("p2p", w.RECV_PREV, 1)]]),
    "PRISM_E_TEMPLATE_MISMATCH": (w.Topology(1, 2, 1), [[("p2p", w.SEND_NEXT, 1)], [("c", 1)]]),
    "PRISM_E_NEGATIVE_MEMORY": (w.Topology(1, 1, 1), [[("c", 1, 5, 0), ("c", 1, 0, 6)]]),
    "PRISM_E_INVALID_SPEC": (w.Topology(1, 1, 3, 2), [[("c", 1)]]),
}


@pytest.mark.parametrize("name", sorted(ERROR_CASES))
def test_error_statuses_agree_with_oracle(name):
    topo, stages = ERROR_CASES[name]
    tm = _tm(topo, stages)
    with pytest.raises(prism.PrismError) as e:
        prism.plan(tm)
    assert e.value.name == name
    with pytest.raises(oracle.OracleError) as e2:
        oracle.replay(tm)
    assert "PRISM_E_" + e2.value.name == name


def test_invalid_ops_rejected():
    tm = w.config("C1")
    bad = tm.ops.copy()
    bad["dur_ns"][3] = -1
    with pytest.raises(prism.PrismError) as e:
        prism.plan(w.Templates(tm.topo, bad, tm.tmpl_ptr, tm.static_mem))
    assert e.value.name == "PRISM_E_INVALID_ARG"
    bad = tm.ops.copy()
    bad["kind"][0] = 7
    with pytest.raises(prism.PrismError):
        prism.plan(w.Templates(tm.topo, bad, tm.tmpl_ptr, tm.static_mem))


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(prism.PrismError) as e:
        prism.Graph(w.config("C1"))
    assert e.value.name == "PRISM_E_CUDA"


def test_bench_reference_arm_runs():
    """bench.py --impl reference (the CPU oracle arm) prints its JSON line on a bounded sample."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1", "--config", "C2"], capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_bench_clock_window():
    """bench.Clocks keeps the samples that arrived during the timed region (else the nearest one),
    reports the median SM clock and any throttle reason, and can be summarised twice."""
    import importlib.util
    import os

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    c = bench.Clocks(0)
    row = lambda sm, t, slow="Not Active": ["0", str(sm), "1965", "700.0", "0x0", slow, "Not Active",
                                             "Not Active", "Not Active", t]
    c.rows = [row(1000, 0.5), row(1965, 10.0), row(1950, 10.1), row(1965, 10.2, "Active"), row(900, 20.0)]
    c.mark(9.95, 10.25)
    s1 = c.summary()
    assert s1 == {"sm_mhz": 1965, "sm_max_mhz": 1965, "reasons": ["hw_slowdown"], "samples": 3}
    assert c.summary() == s1
    c.mark(30.0, 30.1)  # no sample inside: the nearest one
    assert c.summary()["samples"] == 1 and c.summary()["sm_mhz"] == 900
    c.rows = []
    assert c.summary()["reasons"] == ["unsampled"]

"""GPU: bench.py end to end on a small config — the one JSON line the driver parses, with every key
of the contract, and the same iteration times as the CPU oracle's scenario 0 (row d)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import workloads as w

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_json_contract():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "C2", "--steps", "3",
                        "--warmup", "3", "--no-cpu-baseline", "--no-f-rows"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    assert 0 < d["roofline"]["frac"] < 1
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and d["value"] > 0
    tm = w.config("C2")
    assert d["config"]["nodes"] == tm.n_nodes
    ref = oracle.replay(tm, 1, seed=0x5EED, amp_q16=6554, kind_mask=7, peaks=False, threads=os.cpu_count() or 1)
    assert d["extra"]["iteration_time_ns_scenario0"] == int(ref["iter"][0])

#!/bin/bash
# kernel change check: parity subset + bench timing ($1 = pytest files)
mkdir -p gpurun_out
timeout 1200 python -m pytest ${1:-tests/test_gpu_parity.py tests/test_gpu_robust.py} -m gpu -x -q > gpurun_out/pytest_k.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_k.log
timeout 600 python bench.py --no-f-rows --no-cpu-baseline > gpurun_out/bench_k.json 2> gpurun_out/bench_k.err
PRISM_CELL_KS=1 timeout 600 python bench.py --no-f-rows --no-cpu-baseline > gpurun_out/bench_k1.json 2>> gpurun_out/bench_k.err

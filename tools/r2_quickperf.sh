#!/bin/bash
# quick perf check: lone-warp chain, C5 and C3 (amp/rec combinations), then the GPU parity subset
mkdir -p gpurun_out
DPS=1 python tools/exp/probe_ops.py > gpurun_out/qp.log 2>&1
python tools/exp/probe_full.py >> gpurun_out/qp.log 2>&1
CONFIG=C3 python tools/exp/probe_full.py >> gpurun_out/qp.log 2>&1
CONFIG=C4 python tools/exp/probe_full.py >> gpurun_out/qp.log 2>&1
CONFIG=C2 python tools/exp/probe_full.py >> gpurun_out/qp.log 2>&1
[ -n "$NOPAR" ] && exit 0
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "random or scaled or fin_array or full_size or world or edge or determin" > gpurun_out/qp_parity.log 2>&1; echo "rc=$?" >> gpurun_out/qp_parity.log

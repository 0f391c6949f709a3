#!/bin/bash
# lookahead check: timings with PRISM_LA=0/1 (probe_full for C5 and C3), then parity
mkdir -p gpurun_out
for la in 0 1; do echo "PRISM_LA=$la"; PRISM_LA=$la python tools/exp/probe_full.py; done > gpurun_out/la_probe.log 2>&1
for la in 0 1; do echo "C3 PRISM_LA=$la"; PRISM_LA=$la CONFIG=C3 python tools/exp/probe_full.py; done >> gpurun_out/la_probe.log 2>&1
[ -n "$NOPAR" ] && exit 0
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "random or scaled or fin_array or full_size or world or edge or determin" > gpurun_out/la_parity.log 2>&1; echo "rc=$?" >> gpurun_out/la_parity.log

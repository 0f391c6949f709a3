#!/bin/bash
mkdir -p gpurun_out
for t in 0 1; do echo "PRISM_FIN_TMA=$t"; PRISM_FIN_TMA=$t python tools/exp/probe_full.py; PRISM_FIN_TMA=$t CONFIG=C4 python tools/exp/probe_full.py; PRISM_FIN_TMA=$t CONFIG=C2 python tools/exp/probe_full.py; done > gpurun_out/tma.log 2>&1
[ -n "$NOPAR" ] && exit 0
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_robust.py tests/test_gpu_shards.py tests/test_gpu_streams.py -m gpu -x -q > gpurun_out/tma_parity.log 2>&1; echo "rc=$?" >> gpurun_out/tma_parity.log

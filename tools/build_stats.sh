#!/bin/bash
# Instrumented build of the library (-DPRISM_CELL_STATS) for tools/cell_stats.py / wait_hist.py.
cd "$(dirname "$0")/../paper_2605_15617_b200"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden -shared -DPRISM_CELL_STATS -o libprism_b200_stats.so csrc/*.cu csrc/*.cpp

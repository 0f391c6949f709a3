#!/bin/bash
# ncu capture of one C5 cell-kernel launch with per-SASS-line counts (source page)
mkdir -p gpurun_out
CFG=${CFG:-C5}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cell_kernel -s 2 -c 1 -o gpurun_out/prof_src_$CFG -f python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-f-rows > gpurun_out/ncu_src_$CFG.log 2>&1
ncu -i gpurun_out/prof_src_$CFG.ncu-rep --page source --csv --print-source sass > gpurun_out/src_sass_$CFG.csv 2>gpurun_out/src_err.log
ncu -i gpurun_out/prof_src_$CFG.ncu-rep --page raw --csv > gpurun_out/raw_src_$CFG.csv 2>/dev/null

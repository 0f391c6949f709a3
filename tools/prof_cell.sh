#!/bin/bash
# ncu full capture (with source counters) of one C5 cell-kernel launch; $1 = output tag, $2 = extra bench args
mkdir -p gpurun_out
tag=${1:-cell}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cell_kernel -s 2 -c 1 -o gpurun_out/prof_$tag -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-f-rows $2 > gpurun_out/ncu_$tag.log 2>&1
ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$tag.csv 2>/dev/null
ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/raw_$tag.csv 2>/dev/null
ncu -i gpurun_out/prof_$tag.ncu-rep --page details --csv > gpurun_out/details_$tag.csv 2>/dev/null
ls -la gpurun_out

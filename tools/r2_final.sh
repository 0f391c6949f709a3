#!/bin/bash
# round-2 final evidence at HEAD: smoke (+ under ncu), -m gpu suite, C5/C4 bench lines, launch
# list, ncu --set full of one cell-kernel launch (C5, C4)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smoke_ncu.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu.log 2>&1; echo "smoke-under-ncu rc=$?" >> gpurun_out/smoke_ncu.log
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 600 python bench.py --config C4 --no-cpu-baseline --no-f-rows > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-f-rows > gpurun_out/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cell_kernel -s 2 -c 1 -o gpurun_out/prof_c5 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-f-rows > gpurun_out/ncu_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cell_kernel -s 2 -c 1 -o gpurun_out/prof_c4 -f python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-f-rows > gpurun_out/ncu_c4.log 2>&1
for t in c5 c4; do
  ncu -i gpurun_out/prof_$t.ncu-rep --page raw --csv > gpurun_out/raw_$t.csv 2>/dev/null
  ncu -i gpurun_out/prof_$t.ncu-rep --page details --csv > gpurun_out/details_$t.csv 2>/dev/null
done
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
./tools/micro/cluster_coop > gpurun_out/cluster.log 2>&1

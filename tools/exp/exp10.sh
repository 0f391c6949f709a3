mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline --no-f-rows --steps 10 > gpurun_out/exp10_bench.json 2> gpurun_out/exp10_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:expand_nodes -c 6 --csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-f-rows > gpurun_out/exp10_ncu.csv 2>&1

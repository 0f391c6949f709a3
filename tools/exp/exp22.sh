mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-f-rows > gpurun_out/exp22_ncu.csv 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/exp22.txt 2>&1

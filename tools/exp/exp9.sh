mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/exp9_pytest.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-f-rows > gpurun_out/exp9_bench.json 2> gpurun_out/exp9_bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:expand_nodes -s 2 -c 1 -o gpurun_out/prof_expand -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-f-rows > gpurun_out/exp9_ncu.log 2>&1

mkdir -p gpurun_out
timeout 300 python tools/exp/host_async.py > gpurun_out/exp11_host.txt 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/exp11_pytest.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-f-rows > gpurun_out/exp11_bench.json 2> gpurun_out/exp11_bench.err

mkdir -p gpurun_out
timeout 300 python tools/step_timeline.py > gpurun_out/exp3_steptl.txt 2>&1
timeout 300 python tools/host_overhead.py > gpurun_out/exp3_host.txt 2>&1

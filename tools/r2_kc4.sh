mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_whatif.py tests/test_gpu_robust.py tests/test_gpu_shards.py -m gpu -x -q -k "C4 or random or moe or world or watchdog or abort or sharded" > gpurun_out/pytest_rc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_rc.log
python tools/scen_scaling.py C4 > gpurun_out/scal_c4.log 2>&1
PRISM_REPLICA_CELLS=0 python tools/scen_scaling.py C4 > gpurun_out/scal_c4_off.log 2>&1
python bench.py --no-cpu-baseline --no-f-rows --steps 10 > gpurun_out/bench.json 2> gpurun_out/bench.err

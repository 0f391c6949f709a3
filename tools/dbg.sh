mkdir -p gpurun_out
timeout 600 python -X faulthandler -m pytest tests/test_gpu_robust.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/r1.log 2>&1; echo "rc=$?" >> gpurun_out/r1.log

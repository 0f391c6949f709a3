mkdir -p gpurun_out
python tools/exp/fast_sweep.py 4,32,256 > gpurun_out/exp7_sweep.txt 2>&1
for c in C4 C3 C2; do CFG=$c python tools/exp/fast_sweep.py 4,32,256 >> gpurun_out/exp7_sweep.txt 2>&1; done
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/exp7_pytest.txt 2>&1
DPS=1,2072 timeout 300 python tools/exp/probe_ops.py > gpurun_out/exp7_ops.txt 2>&1

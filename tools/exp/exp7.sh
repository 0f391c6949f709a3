mkdir -p gpurun_out
python tools/exp/fast_sweep.py 4,32,256 > gpurun_out/exp7_sweep.txt 2>&1
for c in C4 C3 C2; do CFG=$c python tools/exp/fast_sweep.py 4,32,256 >> gpurun_out/exp7_sweep.txt 2>&1; done
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/exp7_pytest.txt 2>&1
export PRISM_LIB=$PWD/paper_2605_15617_b200/libprism_b200_stats.so
DP=1 AMP=6554 REC=1 timeout 300 python tools/timeline.py > gpurun_out/exp7_tl.txt 2>&1

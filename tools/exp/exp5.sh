mkdir -p gpurun_out
python tools/exp/fast_sweep.py 4,32,256 0,0,0 > gpurun_out/exp5_sweep.txt 2>&1
CFG=C4 python tools/exp/fast_sweep.py 4,32,256 >> gpurun_out/exp5_sweep.txt 2>&1
CFG=C3 python tools/exp/fast_sweep.py 4,32,256 >> gpurun_out/exp5_sweep.txt 2>&1
CFG=C2 python tools/exp/fast_sweep.py 4,32,256 >> gpurun_out/exp5_sweep.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/exp5_parity.txt 2>&1
export PRISM_LIB=$PWD/paper_2605_15617_b200/libprism_b200_stats.so
DP=1 AMP=6554 REC=1 timeout 300 python tools/timeline.py > gpurun_out/exp5_tl.txt 2>&1

mkdir -p gpurun_out
python tools/exp/fast_sweep.py 0,0,0 4,32,256 0,32,128 16,32,128 2,16,64 4,32,512 8,64,1024 4,32,256/2,32,2048 4,32,256/2,64,4096 > gpurun_out/exp4_sweep.txt 2>&1
CFG=C4 python tools/exp/fast_sweep.py 0,0,0 4,32,256 >> gpurun_out/exp4_sweep.txt 2>&1
CFG=C2 python tools/exp/fast_sweep.py 0,0,0 4,32,256 >> gpurun_out/exp4_sweep.txt 2>&1
export PRISM_LIB=$PWD/paper_2605_15617_b200/libprism_b200_stats.so
DP=1 AMP=6554 REC=1 timeout 300 python tools/timeline.py > gpurun_out/exp4_tl.txt 2>&1
DP=64 AMP=6554 REC=1 timeout 300 python tools/timeline.py >> gpurun_out/exp4_tl.txt 2>&1

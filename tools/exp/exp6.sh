mkdir -p gpurun_out
CFG=C4 python tools/exp/fast_sweep.py 4,32,256 0,0,0 > gpurun_out/exp6_sweep.txt 2>&1
CFG=C4 PRISM_LEAN=0 python tools/exp/fast_sweep.py 4,32,256 >> gpurun_out/exp6_sweep.txt 2>&1
python tools/exp/fast_sweep.py 4,32,256 2,32,128 8,32,512 4,32,256/2,32,512 4,32,256/4,32,2048 >> gpurun_out/exp6_sweep.txt 2>&1

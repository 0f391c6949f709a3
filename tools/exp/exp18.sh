mkdir -p gpurun_out
CFG=C4 python tools/exp/fast_sweep.py 4,32,256 > gpurun_out/exp18.txt 2>&1
CFG=C4 PRISM_LEAN=2 python tools/exp/fast_sweep.py 4,32,256 >> gpurun_out/exp18.txt 2>&1

mkdir -p gpurun_out
python tools/exp/fast_sweep.py 4,32,256 4,32,256 1,32,128 8,64,512 16,32,256 4,16,128 0,0,0 4,32,256/1,32,512 4,32,256/4,64,2048 > gpurun_out/exp17.txt 2>&1
CFG=C3 python tools/exp/fast_sweep.py 4,32,256 1,32,128 8,64,512 >> gpurun_out/exp17.txt 2>&1

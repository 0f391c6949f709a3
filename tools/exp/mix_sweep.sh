mkdir -p gpurun_out
for m in 1 5 7 11 17 65 99 101 103 151 201 255 257 301 385 451 999; do printf "mix=%s " $m >> gpurun_out/mix.log; PRISM_CELL_MIX=$m python tools/poll_sweep.py C5 2,32,1024 >> gpurun_out/mix.log 2>&1; done

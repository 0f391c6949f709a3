mkdir -p gpurun_out
timeout 300 python tools/exp/probe_dp1.py > gpurun_out/exp2_probe.txt 2>&1
PROBE=6554,1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:cell_kernel -s 2 -c 1 -o gpurun_out/prof_dp1 -f python tools/exp/probe_dp1.py > gpurun_out/exp2_ncu.log 2>&1

mkdir -p gpurun_out
export PRISM_LIB=$PWD/paper_2605_15617_b200/libprism_b200_stats.so
for dp in 1 64; do
  echo "== DP=$dp AMP=6554 REC=1"; DP=$dp AMP=6554 REC=1 timeout 300 python tools/timeline.py
  echo "== DP=$dp AMP=0 REC=0"; DP=$dp AMP=0 REC=0 timeout 300 python tools/timeline.py
done > gpurun_out/exp1_timeline.txt 2>&1
unset PRISM_LIB
timeout 600 python tools/chain_probe.py > gpurun_out/exp1_chain.txt 2>&1

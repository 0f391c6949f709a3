#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/expand_lb.log
for n in 2 3 4; do
  sed -i "s/__launch_bounds__(256, [0-9]) expand_nodes_kernel/__launch_bounds__(256, $n) expand_nodes_kernel/" paper_2605_15617_b200/csrc/expand.cu
  python -c "from paper_2605_15617_b200 import build as b; b.build()" >> gpurun_out/expand_lb.log 2>&1
  echo "minblocks=$n" >> gpurun_out/expand_lb.log
  python tools/exp/expand_time.py C5 C3 >> gpurun_out/expand_lb.log 2>&1
done

#!/bin/bash
mkdir -p gpurun_out
for la in 0 1 3 8 20; do echo "PRISM_LA=$la"; PRISM_LA=$la python tools/exp/probe_full.py; done > gpurun_out/la_probe2.log 2>&1

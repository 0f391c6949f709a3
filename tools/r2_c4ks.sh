mkdir -p gpurun_out
for ks in 8 16; do PRISM_EP_CTA_KS=$ks python tools/scen_scaling.py C4 > gpurun_out/scal_c4_ks$ks.log 2>&1; done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_whatif.py tests/test_gpu_shards.py -m gpu -x -q -k "C4 or moe" > gpurun_out/pytest_rc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_rc.log

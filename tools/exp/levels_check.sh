mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_whatif.py -m gpu -x -q -k "levels or wide or random" > gpurun_out/pytest_lv.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_lv.log
python - > gpurun_out/lv_time.log 2>&1 <<'PY'
import sys; sys.path.insert(0, '.')
import torch, paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
for name in ("C2", "C5"):
    tm = w.config(name)
    g = prism.Graph(tm, stream=torch.cuda.current_stream().cuda_stream, profile=True)
    ts = []
    for _ in range(3):
        g.replay(64, amp_q16=6554, kind_mask=7, algo="levels"); ts.append(g.last_timing()["levels"])
    print(name, "levels path ms", min(ts))
PY

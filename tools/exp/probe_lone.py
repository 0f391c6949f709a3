"""Dev experiment: one lone-warp chain replay (tp=8, pp=1, dp=1, S=32, amp and record on) for an
ncu source-level capture of where a lone warp's per-op latency goes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
tm = w.uniform_pipeline(8, 1, int(os.environ.get("DP", "1")), 64, layers_per_chunk=8, dp_ar_ns=-1)
g = prism.Graph(tm, stream=torch.cuda.current_stream().cuda_stream, profile=True)
for _ in range(3):
    g.replay(32, amp_q16=6554, kind_mask=7, record=True, algo="cells")
print("ms", g.last_timing()["levels"])

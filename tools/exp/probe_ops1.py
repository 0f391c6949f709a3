"""Dev experiment: one lone warp on a chain with no cross-cell ops (tp=8, pp=1, dp=1), one
(amp, record) combination from PROBE (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
tm = w.uniform_pipeline(8, 1, 1, 64, layers_per_chunk=8, dp_ar_ns=-1)
g = prism.Graph(tm, stream=torch.cuda.current_stream().cuda_stream, profile=True)
amp, rec = (int(x) for x in os.environ.get("PROBE", "0,0").split(","))
for _ in range(4):
    g.replay(32, amp_q16=amp, kind_mask=7, record=bool(rec), algo="cells")
print(g.last_timing()["levels"])

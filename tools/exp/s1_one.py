"""Dev tool: one S = 1 replay of a config (for ncu captures of the rank kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
sh = torch.cuda.current_stream().cuda_stream
tm = w.config(sys.argv[1] if len(sys.argv) > 1 else "C5")
amp = int(sys.argv[2]) if len(sys.argv) > 2 else 0
g = prism.Graph(tm, stream=sh)
for _ in range(2):
    print(g.replay(1, record=True, algo="ranks", amp_q16=amp, kind_mask=7, first=1))
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        g.replay(1, record=True, algo="ranks", amp_q16=amp, kind_mask=7, first=1)
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12))

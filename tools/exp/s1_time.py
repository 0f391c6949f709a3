"""Dev experiment: S = 1 replay time of a config (segment path), median of 7, plus T."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
sh = torch.cuda.current_stream().cuda_stream
for name in sys.argv[1:] or ["C5"]:
    tm = w.config(name)
    g = prism.Graph(tm, stream=sh, profile=True)
    ts = []
    for _ in range(7):
        it = g.replay(1, record=True, amp_q16=6554, kind_mask=7, first=1)
        t = g.last_timing(); ts.append(t["levels"] + t.get("tail", 0) + t.get("reduce", 0))
    print(f"{name} S=1 replay ms median {sorted(ts)[3]:.4f} min {min(ts):.4f} algo {g.last_algo()} T {int(it[0])}", flush=True)
    g.close()

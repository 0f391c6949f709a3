"""Dev experiment: replay time of every BASELINE config at S = 1 (rank kernel) and S = 64 (cell
kernel), device-timed (profile graphs), median of 5."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
for name in ("C1", "C2", "C3", "C4", "C5"):
    tm = w.config(name)
    g = prism.Graph(tm, stream=torch.cuda.current_stream().cuda_stream, profile=True)
    st = g.stats()
    row = [name, st["nodes"]]
    for S in (1, 64):
        ts = []
        for _ in range(5):
            g.replay(S, amp_q16=6554 if S > 1 else 0, kind_mask=7)
            t = g.last_timing()
            ts.append(t["levels"] + t["tail"] + t["reduce"])
        ms = sorted(ts)[2]
        row += [S, g.last_algo(), round(ms, 3), round(st["nodes"] * S / ms / 1e6, 1)]
    print(*row, flush=True)
    g.close()

"""Dev experiment: device time of the expansion (rank tables + nodes + groups) of a config,
median of 9 profiled builds."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
for name in (sys.argv[1:] or ["C5"]):
    tm = w.config(name)
    ts = []
    for _ in range(9):
        g = prism.Graph(tm, stream=torch.cuda.current_stream().cuda_stream, profile=True)
        ts.append(g.last_timing()["expand"])
        g.close()
    print(name, "expand ms median", round(sorted(ts)[4], 4), "min", round(min(ts), 4), flush=True)

"""Dev tool: S = 1 replay time of each schedule (device ms, best of 5) for the configs given."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
sh = torch.cuda.current_stream().cuda_stream
for name in (sys.argv[1:] or ["C5"]):
    tm = w.config(name)
    g = prism.Graph(tm, stream=sh, profile=True)
    ref = None
    for algo in ("auto", "cells", "ranks", "levels"):
        for amp in (0, 6554):
            try:
                best = None
                for _ in range(5):
                    it = g.replay(1, record=True, algo=algo, amp_q16=amp, kind_mask=7, first=1)
                    ms = g.last_timing()["levels"]
                    best = ms if best is None else min(best, ms)
                print(name, algo, "amp", amp, "->", g.last_algo(), "%.4f ms" % best, it[0], flush=True)
            except Exception as e:
                print(name, algo, "amp", amp, "failed", e, flush=True)
    g.close()

"""Dev tool: C5 replay time vs scenario count (latency- vs throughput-bound)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
tm = w.config(sys.argv[1] if len(sys.argv) > 1 else "C5")
g = prism.Graph(tm, stream=torch.cuda.current_stream().cuda_stream, profile=True)
for S in (1, 32, 64, 96, 128, 192, 256):
    for rec in (True, False):
        ts = []
        for _ in range(3):
            g.replay(S, amp_q16=6554, kind_mask=7, record=rec)
            ts.append(g.last_timing()["levels"])
        st = g.stats()
        print(f"S={S:4d} record={int(rec)} launches={st['replay_launches']} ms={min(ts):7.3f} "
              f"Gnode-scen/s={st['nodes']*S/min(ts)/1e6:8.1f}", flush=True)

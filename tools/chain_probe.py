"""Dev tool: replay time of C5-shaped graphs with fewer DP replicas (1 pipeline = 16 warps per
scenario chunk): separates the dependency chain from SM contention."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
c5 = w.config("C5")
for dp in (1, 4, 16, 64):
    t = c5.topo
    tm = w.Templates(w.Topology(t.tp, t.pp, dp, 1, t.vpp, t.rank_order), c5.ops, c5.tmpl_ptr, c5.static_mem)
    g = prism.Graph(tm, stream=torch.cuda.current_stream().cuda_stream, profile=True)
    for S, amp, rec in ((32, 6554, True), (32, 0, False), (64, 6554, True)):
        ts = []
        for _ in range(3):
            g.replay(S, amp_q16=amp, kind_mask=7, record=rec)
            ts.append(g.last_timing()["levels"])
        print(f"dp={dp:3d} S={S} amp={amp} record={int(rec)} ms={min(ts):7.3f}", flush=True)
    g.close()

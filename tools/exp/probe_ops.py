"""Dev experiment: per-op cost of the cell kernel on a chain with no cross-cell ops (tp=8, pp=1):
kernel time / template ops, for a lone warp (dp=1) and at occupancy (dp=DPS)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
for dp in [int(x) for x in os.environ.get("DPS", "1,1036").split(",")]:
    tm = w.uniform_pipeline(8, 1, dp, 64, layers_per_chunk=8, dp_ar_ns=-1)
    g = prism.Graph(tm, stream=torch.cuda.current_stream().cuda_stream, profile=True)
    ops = int(tm.tmpl_ptr[1] - tm.tmpl_ptr[0])
    for amp, rec in ((0, 0), (6554, 0), (0, 1), (6554, 1)):
        ts = []
        for _ in range(4):
            g.replay(32, amp_q16=amp, kind_mask=7, record=bool(rec), algo="cells")
            ts.append(g.last_timing()["levels"])
        ms = min(ts)
        print(f"dp={dp} ops={ops} amp={amp} rec={rec}: {ms:.3f} ms, {ms * 1e6 / ops:.1f} ns/op = {ms * 1e6 / ops * 1.965:.0f} cycles/op", flush=True)
    g.close()

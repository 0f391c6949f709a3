"""Dev experiment: one C5 pipeline (dp=DP) replayed under (amp, record) combinations; under ncu,
PROBE=amp,rec selects one combination."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
c5 = w.config("C5"); t = c5.topo
dp = int(os.environ.get("DP", "1"))
tm = w.Templates(w.Topology(t.tp, t.pp, dp, 1, t.vpp, t.rank_order), c5.ops, c5.tmpl_ptr, c5.static_mem)
g = prism.Graph(tm, stream=torch.cuda.current_stream().cuda_stream, profile=True)
combos = [(0, 0), (6554, 0), (0, 1), (6554, 1)]
if os.environ.get("PROBE"):
    a, r = os.environ["PROBE"].split(","); combos = [(int(a), int(r))]
for amp, rec in combos:
    ts = []
    for _ in range(4):
        g.replay(32, amp_q16=amp, kind_mask=7, record=bool(rec), algo="cells")
        ts.append(g.last_timing()["levels"])
    print(f"dp={dp} S=32 amp={amp} record={rec} ms={min(ts):7.3f}", flush=True)

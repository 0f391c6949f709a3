"""Dev experiment: full C5 (or CONFIG) replayed at S=64 under (amp, record) combinations, to split
the replay's time into hashing, fin stores and the dependency structure."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
tm = w.config(os.environ.get("CONFIG", "C5"))
S = int(os.environ.get("S", "64"))
g = prism.Graph(tm, stream=torch.cuda.current_stream().cuda_stream, profile=True)
for amp, rec in [(0, 0), (6554, 0), (0, 1), (6554, 1)]:
    ts = []
    for _ in range(5):
        g.replay(S, amp_q16=amp, kind_mask=7, record=bool(rec), algo="cells")
        ts.append(g.last_timing()["levels"])
    print(f"S={S} amp={amp} record={rec} ms={min(ts):7.3f} med={sorted(ts)[2]:7.3f}", flush=True)

"""Dev tool: device-side timeline of bench steps (CUDA events between phases) -> idle gaps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
tm = w.config("C5"); stream = torch.cuda.current_stream(); sh = stream.cuda_stream
it = torch.zeros(64, dtype=torch.int64, device="cuda"); pk = torch.zeros(tm.topo.world, dtype=torch.int64, device="cuda")
kw = dict(amp_q16=6554, kind_mask=7)
graphs = []
rows = []
for step in range(12):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(stream)
    g = prism.Graph(tm, stream=sh, asynchronous=True)
    ev[1].record(stream)
    while graphs:
        graphs.pop().close()
    g.replay_async(it.data_ptr(), 64, **kw)
    ev[2].record(stream)
    g.peak_memory_async(pk.data_ptr())
    ev[3].record(stream)
    graphs.append(g)
    rows.append(ev)
torch.cuda.synchronize()
for i, ev in enumerate(rows[2:], 2):
    nxt = rows[i + 1][0] if i + 1 < len(rows) else None
    b = ev[0].elapsed_time(ev[1]); r = ev[1].elapsed_time(ev[2]); p = ev[2].elapsed_time(ev[3])
    tot = ev[0].elapsed_time(nxt) if nxt else float("nan")
    print(f"step {i}: build(expand+H2D) {b:.3f} replay {r:.3f} peak {p:.3f} step total {tot:.3f} ms")

"""Dev experiment: consecutive replays of DIFFERENT graphs (same workload) on one stream vs
alternating between two streams (the tail of replay i overlapping the head of replay i+1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
tm = w.config(os.environ.get("CONFIG", "C5"))
S = 64
kw = dict(amp_q16=6554, kind_mask=7, seed=0x5EED)
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
graphs = [prism.Graph(tm, stream=s.cuda_stream) for s in streams]
out = torch.zeros(2, S, dtype=torch.int64, device="cuda")
ref = graphs[0].replay(S, record=True, **kw)
for mode in ("one stream", "two streams", "one stream", "two streams"):
    K = 20
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(streams[0])
    for i in range(K):
        gi = i % 2
        if mode == "one stream":
            if gi == 1:
                streams[1].wait_stream(streams[0])
            graphs[gi].replay_async(out[gi].data_ptr(), S, record=True, **kw)
            if gi == 1:
                streams[0].wait_stream(streams[1])
        else:
            graphs[gi].replay_async(out[gi].data_ptr(), S, record=True, **kw)
    streams[0].wait_stream(streams[1])
    e1.record(streams[0])
    torch.cuda.synchronize()
    ok = (out.cpu().numpy() == ref[None, :]).all()
    print(f"{mode:12s}: {e0.elapsed_time(e1) / K:.3f} ms per replay, results match {ok}", flush=True)
for g in graphs:
    g.sync()

"""Dev experiment: the bench step (build from host templates + replay + peak) of consecutive graphs
on one stream vs graphs alternating between two streams (step i+1's expansion can fill SMs while
step i's cooperative replay drains)."""
import gc, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
tm = w.config(os.environ.get("CONFIG", "C5"))
S = 64
kw = dict(amp_q16=6554, kind_mask=7, seed=0x5EED)
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
out = torch.zeros(2, S, dtype=torch.int64, device="cuda")
pk = torch.zeros(2, tm.topo.world, dtype=torch.int64, device="cuda")
ref = prism.Graph(tm, stream=streams[0].cuda_stream).replay(S, record=True, **kw)
gc.disable()
for mode in ("one stream", "two streams") * 2:
    K = 20
    live = []
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(streams[0])
    for i in range(K + 3):
        if i == 3:
            streams[1].wait_stream(streams[0]); streams[0].wait_stream(streams[1])
            e0.record(streams[0]); streams[1].wait_event(e0)
        si = i % 2 if mode == "two streams" else 0
        g = prism.Graph(tm, stream=streams[si].cuda_stream, asynchronous=True)
        g.replay_async(out[i % 2].data_ptr(), S, record=True, **kw)
        g.peak_memory_async(pk[i % 2].data_ptr())
        live.append(g)
        if len(live) > 2:
            live.pop(0).close()
    streams[0].wait_stream(streams[1])
    e1.record(streams[0])
    torch.cuda.synchronize()
    ok = (out.cpu().numpy() == ref[None, :]).all()
    print(f"{mode:12s}: {e0.elapsed_time(e1) / K:.3f} ms per step, results match {ok}", flush=True)
    for g in live:
        g.close()
gc.enable()

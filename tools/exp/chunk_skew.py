"""Dev experiment: C5's two 32-scenario chunks as two cooperative grids (two graphs, two streams,
scenarios 0-31 and 32-63), the second started after a delay: does offsetting the chunks' 1F1B
ramps beat starting them together? Reference: one S = 64 replay."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
tm = w.config(os.environ.get("CONFIG", "C5"))
kw = dict(amp_q16=6554, kind_mask=7, seed=0x5EED)
s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
g64 = prism.Graph(tm, stream=s0.cuda_stream)
ga = prism.Graph(tm, stream=s0.cuda_stream)
gb = prism.Graph(tm, stream=s1.cuda_stream)
out = torch.zeros(3, 64, dtype=torch.int64, device="cuda")
ref = g64.replay(64, record=True, **kw)
# cycles of torch.cuda._sleep per microsecond at the SM clock
cyc_per_us = 1965
def run(mode, skew_us):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s0); s1.wait_event(e0)
    if mode == "S64":
        g64.replay_async(out[2].data_ptr(), 64, record=True, **kw)
    else:
        ga.replay_async(out[0].data_ptr(), 32, record=True, first=0, **kw)
        with torch.cuda.stream(s1):
            if skew_us > 0:
                torch.cuda._sleep(int(skew_us * cyc_per_us))
        gb.replay_async(out[1].data_ptr(), 32, record=True, first=32, **kw)
    s0.wait_stream(s1); e1.record(s0)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)
for rep in range(2):
    print("S64 one grid", round(min(run("S64", 0) for _ in range(3)), 3), flush=True)
    for skew in (0, 100, 200, 400, 700):
        ms = min(run("two", skew) for _ in range(3))
        ok = np.array_equal(np.concatenate([out[0, :32].cpu().numpy(), out[1, :32].cpu().numpy()]), ref)
        print(f"two grids, skew {skew:4d} us: {ms:.3f} ms (results match {ok})", flush=True)
for g in (g64, ga, gb):
    g.sync()

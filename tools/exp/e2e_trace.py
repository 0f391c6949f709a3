"""Dev experiment: the bench's e2e loop (public API, host buffers) with host timestamps per call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
tm = w.config("C5"); sh = torch.cuda.current_stream().cuda_stream
kw = dict(amp_q16=6554, kind_mask=7, seed=0x5EED)
prev = prism.Graph(tm, stream=sh, asynchronous=True); prev.replay(64, **kw); prev.peak_memory()
for rep in range(6):
    t0 = time.perf_counter()
    g = prism.Graph(tm, stream=sh, asynchronous=True)
    t1 = time.perf_counter()
    prev.close()
    t2 = time.perf_counter()
    it = g.replay(64, record=True, **kw)
    t3 = time.perf_counter()
    pk = g.peak_memory()
    t4 = time.perf_counter()
    prev = g
    print(f"build {1e3*(t1-t0):.3f} close {1e3*(t2-t1):.3f} replay {1e3*(t3-t2):.3f} peak {1e3*(t4-t3):.3f} total {1e3*(t4-t0):.3f} ms", flush=True)

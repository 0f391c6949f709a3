"""Dev experiment: host time of prism.Graph(...) (plan + packing + queueing the upload and the
expansion, asynchronous build) for repeated builds of one config — the first plans, the rest hit
the plan cache."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
tm = w.config(os.environ.get("CONFIG", "C5")); sh = torch.cuda.current_stream().cuda_stream
ts = []
for i in range(12):
    t0 = time.perf_counter()
    g = prism.Graph(tm, stream=sh, asynchronous=True)
    ts.append((time.perf_counter() - t0) * 1e3)
    torch.cuda.synchronize(); g.close()
print("host build ms: first %.3f, then median %.3f (min %.3f)" % (ts[0], sorted(ts[1:])[len(ts[1:]) // 2], min(ts[1:])), flush=True)

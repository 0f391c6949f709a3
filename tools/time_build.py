"""Dev tool: where does prism_build_graph's time go? (host plan / wall / device expand)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
tm = w.config(sys.argv[1] if len(sys.argv) > 1 else "C5")
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    prism.plan(tm)
t0 = time.perf_counter()
for _ in range(10):
    prism.plan(tm)
print(f"host plan: {(time.perf_counter()-t0)/10*1e3:.2f} ms")
for i in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = prism.Graph(tm, stream=st, profile=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    e = g.last_timing()["expand"]
    g.replay(64, amp_q16=6554, kind_mask=7)
    t2 = time.perf_counter()
    g.close()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"build wall {(t1-t0)*1e3:.2f} ms (device expand {e:.2f} ms), first replay wall {(t2-t1)*1e3:.2f} ms, close {(t3-t2)*1e3:.2f} ms")

"""Dev tool: host cost of the bench step's API calls (C5), pipelined, plus the plan alone."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
tm = w.config("C5"); sh = torch.cuda.current_stream().cuda_stream
it = torch.zeros(64, dtype=torch.int64, device="cuda"); pk = torch.zeros(tm.topo.world, dtype=torch.int64, device="cuda")
for _ in range(5): prism.plan(tm)
t0 = time.perf_counter()
for _ in range(20): prism.plan(tm)
print("plan only %.3f ms" % ((time.perf_counter() - t0) / 20 * 1e3))
prev = None; rows = []
torch.cuda.synchronize()
T0 = time.perf_counter()
for rep in range(30):
    t0 = time.perf_counter()
    g = prism.Graph(tm, stream=sh, asynchronous=True)
    t1 = time.perf_counter()
    if prev: prev.close()
    t2 = time.perf_counter()
    g.replay_async(it.data_ptr(), 64, amp_q16=6554, kind_mask=7)
    t3 = time.perf_counter()
    g.peak_memory_async(pk.data_ptr())
    t4 = time.perf_counter()
    prev = g
    rows.append((t1 - t0, t2 - t1, t3 - t2, t4 - t3))
torch.cuda.synchronize()
T1 = time.perf_counter()
import numpy as np
r = np.array(rows[10:]) * 1e3
print("median build %.3f close %.3f replay %.3f peak %.3f ms; wall per step %.3f ms" % (*np.median(r, 0), 1e3 * (T1 - T0) / 30))

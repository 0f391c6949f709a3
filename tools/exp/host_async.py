"""Dev experiment: host time per bench step (asynchronous build + replay + peak submission) vs
the device time per step, to see whether the bench step is host-bound."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
tm = w.config("C5"); stream = torch.cuda.current_stream(); sh = stream.cuda_stream
it = torch.zeros(64, dtype=torch.int64, device="cuda"); pk = torch.zeros(tm.topo.world, dtype=torch.int64, device="cuda")
graphs = []
def step():
    t0 = time.perf_counter()
    g = prism.Graph(tm, stream=sh, asynchronous=True)
    t1 = time.perf_counter()
    while graphs: graphs.pop().close()
    t2 = time.perf_counter()
    g.replay_async(it.data_ptr(), 64, amp_q16=6554, kind_mask=7)
    t3 = time.perf_counter()
    g.peak_memory_async(pk.data_ptr())
    t4 = time.perf_counter()
    graphs.append(g)
    return (t1 - t0, t2 - t1, t3 - t2, t4 - t3)
for _ in range(3): step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
h = []
t0 = time.perf_counter(); e0.record(stream)
for _ in range(20): h.append(step())
th = time.perf_counter() - t0
e1.record(stream); torch.cuda.synchronize(); tt = time.perf_counter() - t0
import numpy as np
h = np.array(h) * 1e3
print("host per step: build %.3f close %.3f replay %.3f peak %.3f  total %.3f ms" % tuple(list(h.mean(0)) + [h.sum(1).mean()]))
print("host loop %.3f ms/step, device %.3f ms/step, wall %.3f ms/step" % (th * 50, e0.elapsed_time(e1) / 20, tt * 50))
t0 = time.perf_counter(); [prism.plan(tm) for _ in range(5)]; print("plan ms", (time.perf_counter() - t0) * 200)

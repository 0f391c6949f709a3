"""Dev tool: the bench.py step loop with a CUDA event at every step boundary (device timeline of
build / replay / peak and the gaps), with and without the build worker thread."""
import os, sys, time, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import concurrent.futures as cf
import torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
tm = w.config("C5"); stream = torch.cuda.current_stream(); sh = stream.cuda_stream
S = 64
iter_steps = torch.zeros(20, S, dtype=torch.int64, device="cuda")
pk = torch.zeros(tm.topo.world, dtype=torch.int64, device="cuda")
for worker in (False, True):
    pool = cf.ThreadPoolExecutor(1, initializer=lambda: torch.cuda.set_device(0)) if worker else None
    graphs = []
    new_graph = lambda: prism.Graph(tm, stream=sh, asynchronous=True, device=0)
    evs = []
    def step(i, nxt, prefetch):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(stream)
        g = nxt.result() if nxt is not None else new_graph()
        fut = pool.submit(new_graph) if (pool and prefetch) else None
        while graphs: graphs.pop().close()
        e[1].record(stream)
        g.replay_async(iter_steps[i].data_ptr(), S, amp_q16=6554, kind_mask=7)
        e[2].record(stream)
        g.peak_memory_async(pk.data_ptr())
        graphs.append(g)
        evs.append(e)
        return fut
    for i in range(4): step(0, None, False)
    torch.cuda.synchronize(); evs.clear(); gc.disable()
    t0 = time.perf_counter()
    fut = None
    for i in range(20): fut = step(i, fut, i + 1 < 20)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / 20 * 1e3
    gc.enable()
    tot = evs[0][0].elapsed_time(evs[-1][2])
    pre = [a[0].elapsed_time(a[1]) for a in evs]
    rep = [a[1].elapsed_time(a[2]) for a in evs]
    gap = [evs[i][2].elapsed_time(evs[i + 1][0]) for i in range(len(evs) - 1)]
    med = lambda v: sorted(v)[len(v) // 2]
    print(f"worker={worker}: wall/step {wall:.3f} ms; device first->last {tot / 19:.3f} ms/step; median build+close {med(pre):.3f} replay {med(rep):.3f} peak+gap {med(gap):.3f}", flush=True)
    print("  step intervals:", " ".join("%.2f" % evs[i][0].elapsed_time(evs[i + 1][0]) for i in range(len(evs) - 1)))
    print("  build+close:", " ".join("%.2f" % x for x in pre))
    for g in graphs: g.close()
    graphs.clear()

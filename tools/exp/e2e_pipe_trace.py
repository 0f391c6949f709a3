"""Dev experiment: the bench's PIPELINED e2e loop with host timestamps per phase (build, close,
queue replay + peak + copies, wait for the previous step)."""
import gc, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
tm = w.config(os.environ.get("CONFIG", "C5")); sh = torch.cuda.current_stream().cuda_stream
S = 64
kw = dict(amp_q16=6554, kind_mask=7, seed=0x5EED)
dev_it = torch.zeros(2, S, dtype=torch.int64, device="cuda")
dev_pk = torch.zeros(2, tm.topo.world, dtype=torch.int64, device="cuda")
pin_it = torch.zeros(2, S, dtype=torch.int64).pin_memory()
pin_pk = torch.zeros(2, tm.topo.world, dtype=torch.int64).pin_memory()
stream = torch.cuda.current_stream()
for trial in range(2):
    pending = None; rows = []
    gc.disable(); T0 = time.perf_counter()
    for i in range(21):
        t = [time.perf_counter()]
        cur = None
        if i < 20:
            j = i % 2
            g = prism.Graph(tm, stream=sh, asynchronous=True); t.append(time.perf_counter())
            g.replay_async(dev_it[j].data_ptr(), S, record=True, **kw); t.append(time.perf_counter())
            g.peak_memory_async(dev_pk[j].data_ptr())
            pin_it[j].copy_(dev_it[j], non_blocking=True); pin_pk[j].copy_(dev_pk[j], non_blocking=True)
            ev = torch.cuda.Event(); ev.record(stream); t.append(time.perf_counter())
            cur = (ev, g)
        if pending is not None:
            pending[0].synchronize(); t.append(time.perf_counter())
            pending[1].close(); t.append(time.perf_counter())
        pending = cur
        rows.append(np.diff(t) * 1e3)
    tot = (time.perf_counter() - T0) * 1e3 / 20
    gc.enable()
    r = [x for x in rows[2:-1] if len(x) == 5]
    m = np.median(np.array(r), axis=0)
    print(f"trial {trial}: {tot:.3f} ms/step; median host ms: build {m[0]:.3f} replay_async {m[1]:.3f} peak+copies+event {m[2]:.3f} wait_prev {m[3]:.3f} close_prev {m[4]:.3f}", flush=True)

"""Dev tool: host-side cost of one bench step's API calls (C5), to find gaps on the device timeline."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
tm = w.config("C5"); sh = torch.cuda.current_stream().cuda_stream
it = torch.zeros(64, dtype=torch.int64, device="cuda"); pk = torch.zeros(tm.topo.world, dtype=torch.int64, device="cuda")
prev = None
for rep in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = prism.Graph(tm, stream=sh)
    t1 = time.perf_counter()
    if prev: prev.close()
    t2 = time.perf_counter()
    g.replay_async(it.data_ptr(), 64, amp_q16=6554, kind_mask=7)
    t3 = time.perf_counter()
    g.peak_memory_async(pk.data_ptr())
    t4 = time.perf_counter()
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    prev = g
    print(f"build {1e3*(t1-t0):.3f} close {1e3*(t2-t1):.3f} replay-submit {1e3*(t3-t2):.3f} peak-submit {1e3*(t4-t3):.3f} wait {1e3*(t5-t4):.3f} total {1e3*(t5-t0):.3f} ms", flush=True)
os.environ["PLAN"] = "1"
t0 = time.perf_counter(); [prism.plan(tm) for _ in range(5)]; print("plan ms", (time.perf_counter()-t0)*200)

"""Dev tool: wall time of critical_path on C5 (first call incl. scratch allocation, then repeats),
and (under ncu) the per-kernel launch list of one call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
if os.environ.get("L2G"):  # cudaLimitMaxL2FetchGranularity experiment
    import ctypes
    rt = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
    rt = rt or ctypes.CDLL(torch.__path__[0] + "/lib/libcudart.so.12")
    print("setlimit", rt.cudaDeviceSetLimit(5, ctypes.c_size_t(int(os.environ["L2G"]))))
    v = ctypes.c_size_t(0); rt.cudaDeviceGetLimit(ctypes.byref(v), 5); print("L2 fetch granularity", v.value)
tm = w.config(os.environ.get("CFG", "C5")); sh = torch.cuda.current_stream().cuda_stream
g = prism.Graph(tm, stream=sh)
labs = {int(l): 1 for l in np.unique(tm.ops["label"]) if (int(l) >> 24) == w.OPCODES["ATTN_F"]}
f = np.full(tm.topo.world, 65536, np.int32); f[tm.topo.world // 2] = int(1.12 * 65536)
g.set_durations(label_dur=labs, rank_slow_q16=f)
g.replay(64, record=True, amp_q16=6554, kind_mask=7)
torch.cuda.synchronize()
ts = []
for i in range(int(os.environ.get("REPS", "6"))):
    t0 = time.perf_counter(); path, T = g.critical_path(i % 64); ts.append((time.perf_counter() - t0) * 1e3)
print("critical_path ms:", " ".join("%.3f" % t for t in ts), "nodes", len(path), "T", T)
if os.environ.get("KINETO", "1") == "1":
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for i in range(3):
            g.critical_path(i)
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=20))
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    for e in evs[-14:]:
        print("%-50s start %10.1f dur %8.1f us" % (e.name[:50], e.time_range.start, e.time_range.elapsed_us()))

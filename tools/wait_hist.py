"""Dev tool: where do cell-kernel warps wait? (needs a -DPRISM_CELL_STATS build)"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
tm = w.config(sys.argv[1] if len(sys.argv) > 1 else "C5")
g = prism.Graph(tm, stream=torch.cuda.current_stream().cuda_stream, profile=True)
L = prism.lib()
buf = (ctypes.c_ulonglong * (16 * 4096))()
REC = os.environ.get("REC", "1") == "1"
AMP = int(os.environ.get("AMP", "6554"))
g.replay(64, amp_q16=AMP, kind_mask=7, algo="cells", record=REC); L.prism_debug_wait_hist(buf)
g.replay(64, amp_q16=AMP, kind_mask=7, algo="cells", record=REC); L.prism_debug_wait_hist(buf)
lat = (ctypes.c_ulonglong * 4)()
L.prism_debug_lat(lat)
g.replay(64, amp_q16=AMP, kind_mask=7, algo="cells", record=REC); L.prism_debug_wait_hist(buf)
L.prism_debug_lat(lat)
print("kernel ms", g.last_timing()["levels"])
n = max(1, lat[2])
print(f"P2P rendezvous (chunk 0, {lat[2]} samples): handoff (consumer already waiting) latency mean {lat[0]/n/1e3:.2f} us max {lat[3]/1e3:.1f} us; partner lateness mean {lat[1]/n/1e3:.2f} us")
h = np.frombuffer(buf, dtype=np.uint64).reshape(16, 4096).astype(np.float64)
ncell = tm.topo.dp * 2  # warps per stage (2 chunks)
for s in (0, 1, 7, 14, 15):
    tmpl = tm.stage(s)
    row = h[s, :len(tmpl)] / ncell  # mean cycles per warp
    tot = row.sum()
    idx = np.argsort(-row)[:6]
    desc = [(int(i), int(tmpl[i]["kind"]), int(tmpl[i]["p2p_mask"]) if tmpl[i]["kind"] == 2 else int(tmpl[i]["role"]), f"{row[i]/1e3:.0f}k") for i in idx]
    # cumulative by phase: first quarter / middle / last quarter of the template
    n = len(tmpl); q = n // 4
    print(f"stage {s}: wait/warp {tot/1e6:.2f}M cyc; quarters {[round(row[a:b].sum()/1e6,2) for a,b in [(0,q),(q,2*q),(2*q,3*q),(3*q,n)]]}; top {desc}")
    sync_idx = np.nonzero(row)[0]
    print("   first 12 sync waits (k cyc):", [(int(i), round(row[i]/1e3)) for i in sync_idx[:12]])

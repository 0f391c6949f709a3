"""Dev tool (stats build): per-op wait cycles of a single C5 pipeline (dp=1, S=32, one warp per
stage) — where does the uncontended chain spend its time?"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
c5 = w.config("C5"); t = c5.topo
tm = w.Templates(w.Topology(t.tp, t.pp, 1, 1, t.vpp, t.rank_order), c5.ops, c5.tmpl_ptr, c5.static_mem)
g = prism.Graph(tm, stream=torch.cuda.current_stream().cuda_stream, profile=True)
L = prism.lib()
amp = int(os.environ.get("AMP", "0")); rec = os.environ.get("REC", "0") == "1"
buf = (ctypes.c_ulonglong * (16 * 4096))()
cst = (ctypes.c_ulonglong * (16384 * 8))()
for _ in range(2):
    g.replay(32, amp_q16=amp, kind_mask=7, record=rec); L.prism_debug_wait_hist(buf); L.prism_debug_cell_stats(cst, 16384 * 8)
g.replay(32, amp_q16=amp, kind_mask=7, record=rec)
L.prism_debug_wait_hist(buf); L.prism_debug_cell_stats(cst, 16384 * 8)
ms = g.last_timing()["levels"]
h = np.frombuffer(buf, dtype=np.uint64).reshape(16, 4096).astype(np.float64)
cs = np.frombuffer(cst, dtype=np.uint64).reshape(-1, 8)[:16].astype(np.float64)
print(f"kernel {ms:.3f} ms = {ms*1.965e6:.0f} cycles (1965 MHz)")
for s in range(16):
    T = tm.stage(s); n = len(T)
    row = h[s, :n]
    cross = np.nonzero(row)[0]
    tot = cs[s, 0]; wait = row.sum()
    print(f"stage {s:2d}: ops {n} cross ops {len(cross)} warp cycles {tot/1e6:.2f}M wait {wait/1e6:.2f}M "
          f"work {(tot-wait)/1e6:.2f}M ({(tot-wait)/max(1,n):.0f}/op); polls {int(cs[s,3])}; "
          f"min/median/max wait per cross op {row[cross].min()/1e3 if len(cross) else 0:.1f}k/"
          f"{np.median(row[cross])/1e3 if len(cross) else 0:.1f}k/{row[cross].max()/1e3 if len(cross) else 0:.1f}k")

"""Dev tool: per-warp time breakdown of the cell kernel (needs a -DPRISM_CELL_STATS build)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_15617_b200 as prism
import workloads as w

torch.cuda.set_device(0)
prism.use_torch_allocator()
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
tm = w.config(name)
g = prism.Graph(tm, stream=torch.cuda.current_stream().cuda_stream, profile=True)
L = prism.lib()
buf = (ctypes.c_ulonglong * (8192 * 8))()
for amp in (6554, 0):
    g.replay(64, amp_q16=amp, kind_mask=7, algo="cells")
    L.prism_debug_cell_stats(buf, 8192 * 8)
    g.replay(64, amp_q16=amp, kind_mask=7, algo="cells")
    ms = g.last_timing()["levels"]
    L.prism_debug_cell_stats(buf, 8192 * 8)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 8).astype(np.float64)
    nw = tm.topo.pp * tm.topo.dp * 2
    a = a[:nw]
    tot, cross, bar, polls, t0, t1, mx, ns = a[:, 0], a[:, 1], a[:, 2], a[:, 3], a[:, 4], a[:, 5], a[:, 6], a[:, 7]
    print(f"   small-group waits per warp {ns.mean():.0f}; max single small wait mean {mx.mean()/1e3:.1f}k cyc, max {mx.max()/1e3:.1f}k; large-group wait mean {bar.mean()/1e6:.2f}M cyc")
    span = (t1 - t0) / 1e3
    print(f"amp={amp} kernel {ms:.3f} ms; per-warp cycles: total mean {tot.mean()/1e6:.2f}M max {tot.max()/1e6:.2f}M; "
          f"cross-wait mean {cross.mean()/1e6:.2f}M ({cross.sum()/tot.sum()*100:.1f}%); tp-barrier mean {bar.mean()/1e6:.2f}M "
          f"({bar.sum()/tot.sum()*100:.1f}%); polls/warp {polls.mean():.0f}; start spread {(t0.max()-t0.min())/1e3:.1f} us; "
          f"warp span mean {span.mean():.1f} us max {span.max():.1f} us; end spread {(t1.max()-t1.min())/1e3:.1f} us")
    st = (np.arange(nw) % (tm.topo.pp * tm.topo.dp)) % tm.topo.pp
    for s in range(0, tm.topo.pp, 3):
        m = st == s
        print(f"   stage {s:2d}: total {tot[m].mean()/1e6:.2f}M cross {cross[m].mean()/1e6:.2f}M bar {bar[m].mean()/1e6:.2f}M end {(t1[m].mean()-t0.min())/1e3:.0f} us")

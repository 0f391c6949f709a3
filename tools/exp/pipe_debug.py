"""Dev check: small lone chains (tp=8, pp=1, dp=1) replayed with amp and record on, against the
CPU oracle (iteration times and the first mismatching op finish)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2605_15617_b200 as prism, workloads as w, oracle
torch.cuda.set_device(0); prism.use_torch_allocator()
for L in (1, 2, 8, 20):
    tm = w.uniform_pipeline(8, 1, 1, 4, layers_per_chunk=L, dp_ar_ns=-1)
    g = prism.Graph(tm, stream=torch.cuda.current_stream().cuda_stream)
    try:
        it = g.replay(32, amp_q16=6554, kind_mask=7, record=True, algo="cells")
        ref = oracle.replay(tm, 32, amp_q16=6554, kind_mask=7, times=True, peaks=False)
        ok = (it == ref["iter"]).all()
        msg = ""
        if not ok:
            for r in range(8):
                f = np.array([g.query_rank(r, k)["finish"] if False else 0 for k in range(1)])
        print("L", L, "ops", int(tm.tmpl_ptr[1]), "match", ok, "gpu", it[:3], "oracle", ref["iter"][:3], flush=True)
    except Exception as e:
        print("L", L, "error", e, flush=True)
        break
    g.close()

"""Dev tool: time the replay under controlled variations (isolates stores / hashing / syncs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_15617_b200 as prism
import workloads as w


def run(tm, label, S=64, amp=6554, record=True, algo="cells", reps=3):
    g = prism.Graph(tm, stream=torch.cuda.current_stream().cuda_stream, profile=True)
    ts = []
    for _ in range(reps):
        g.replay(S, amp_q16=amp, kind_mask=7, algo=algo, record=record)
        ts.append(g.last_timing()["levels"])
    st = g.stats()
    print(f"{label:50s} algo={g.last_algo():6s} nodes={st['nodes']:>9} ms={min(ts):8.3f} "
          f"ns/node-step={min(ts)*1e6/ (st['nodes']/ (tm.topo.tp*1.0)) * (tm.topo.pp*tm.topo.dp)/ (tm.topo.pp*tm.topo.dp):8.2f}",
          flush=True)
    g.close()


def main():
    torch.cuda.set_device(0)
    prism.use_torch_allocator()
    c5 = w.config("C5")
    run(c5, "C5 baseline")
    run(c5, "C5 record=0", record=False)
    run(c5, "C5 amp=0", amp=0)
    run(c5, "C5 amp=0 record=0", amp=0, record=False)
    run(c5, "C5 S=1 amp=0 record=0", S=1, amp=0, record=False)
    # strip cross-cell syncs: keep only compute + TP collectives, same node count per rank
    ops = c5.ops.copy()
    cross = (ops["kind"] == 2) | ((ops["kind"] == 1) & (ops["role"] != 1))
    ops["kind"][cross] = 0
    ops["role"][cross] = 0
    ops["p2p_mask"][cross] = 0
    tm = w.Templates(c5.topo, ops, c5.tmpl_ptr, c5.static_mem)
    run(tm, "C5 no cross-cell syncs")
    run(tm, "C5 no cross-cell syncs record=0 amp=0", record=False, amp=0)
    # compute only
    ops2 = ops.copy()
    ops2["kind"][:] = 0
    ops2["role"][:] = 0
    tm2 = w.Templates(c5.topo, ops2, c5.tmpl_ptr, c5.static_mem)
    run(tm2, "C5 compute only")
    run(tm2, "C5 compute only record=0 amp=0", record=False, amp=0)


if __name__ == "__main__":
    main()

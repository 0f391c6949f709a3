"""Dev tool: the number of cross-warp rendezvous on the longest dependency chain (every compute
span and TP collective 0 ns, every P2P / DP-class collective 1 ns: T = hop depth)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
sh = torch.cuda.current_stream().cuda_stream
for name in sys.argv[1:] or ["C5"]:
    tm = w.config(name)
    t = tm.topo
    parts = []
    for r in range(t.world):
        s = (r // t.tp) % t.pp if t.rank_order == 0 else r // (t.tp * t.dp)
        T = tm.stage(s)
        parts.append(((T["kind"] == 2) | ((T["kind"] == 1) & (T["role"] != 1))).astype(np.int64))
    d = np.concatenate(parts)
    g = prism.Graph(tm, stream=sh)
    g.set_durations(node_dur=d)
    print(name, "hop depth", g.replay(1, algo="ranks")[0], "cross ops per rank", d.sum() / t.world, flush=True)
    g.close()

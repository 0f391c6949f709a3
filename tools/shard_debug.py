"""Diagnose the in-process sharded replay: timings and statuses per shard."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2605_15617_b200 as P
import workloads as w
import oracle

P.use_torch_allocator()
tm = w.scaled(sys.argv[1] if len(sys.argv) > 1 else "C2")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2
S = 64
streams = [torch.cuda.Stream() for _ in range(n)]
gs = [P.Graph(tm, stream=streams[i].cuda_stream, n_shards=n, shard_index=i) for i in range(n)]
for g in gs: g.shard_prepare(S)
for g in gs: g.shard_connect_local(gs)
outs = [torch.full((S,), -1, dtype=torch.int64, device="cuda") for _ in gs]
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.time()
    for i, (g, o) in enumerate(zip(gs, outs)):
        g.replay_async(o.data_ptr(), S, amp_q16=6554, kind_mask=7)
        print("launched", i, time.time() - t0, flush=True)
    for i, s in enumerate(streams):
        s.synchronize()
        print("stream", i, "done", time.time() - t0, flush=True)
    for i, g in enumerate(gs):
        try:
            g.query_rank(P.shard_ranks(tm.topo, n, i)[0], 0)
            print("shard", i, "ok", outs[i][:3].tolist(), flush=True)
        except Exception as e:
            print("shard", i, "err", e, flush=True)
ref = oracle.replay(tm, S, amp_q16=6554, kind_mask=7, threads=8)
print("ref", ref["iter"][:3])

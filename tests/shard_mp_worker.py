"""Multi-process sharded replay on ONE GPU (2 processes, CUDA IPC exchange) — experiment of the
prism_shard_connect path; run by tests/test_gpu_shards.py::test_multiprocess_ipc under torchrun."""
import os, sys, time
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_15617_b200 as P
import workloads as w

rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = int(os.environ.get("SHARD_DEVICE", os.environ["LOCAL_RANK"]))
torch.cuda.set_device(dev)
dist.init_process_group("gloo")
P.use_torch_allocator()
tm = w.scaled(sys.argv[1] if len(sys.argv) > 1 else "C2")
S = 32
g = P.Graph(tm, stream=torch.cuda.current_stream().cuda_stream, n_shards=ws, shard_index=rank)
g.shard_connect_dist(S)
dist.barrier()
for rep in range(3):
    t0 = time.time()
    try:
        it = g.replay(S, amp_q16=6554, kind_mask=7)
        print(rank, "rep", rep, "ok", it.tolist(), round(time.time() - t0, 3), flush=True)
    except Exception as e:
        print(rank, "rep", rep, "err", e, round(time.time() - t0, 3), flush=True)
        g.shard_connect_dist(S)
    dist.barrier()
# per-rank outputs gathered to every process (prism_shard_gather): a rank owned by the OTHER shard
g.shard_gather(S - 1)
other = [r for r in range(tm.topo.world) if r not in set(g.owned_ranks())][0]
st, fi, _ = g.query_rank(other, S - 1)
path, T = g.critical_path(S - 1)
print(rank, "gathered", other, fi.tolist(), "T", T, "path", len(path), int(path.sum()), flush=True)
if rank == 0:
    import oracle
    ref = oracle.replay(tm, S, amp_q16=6554, kind_mask=7, threads=8, times=True)
    print("ref", ref["iter"].tolist())
    rpath, rT = oracle.critical_path(tm, S - 1, amp_q16=6554, kind_mask=7)
    rp = P.Graph(tm).export("rank_ptr")
    for r in range(tm.topo.world):
        print("reff", r, ref["finish"][S - 1, rp[r]:rp[r + 1]].tolist(), "T", rT, "path", len(rpath), int(rpath.sum()))
dist.barrier()
g.close()
dist.destroy_process_group()

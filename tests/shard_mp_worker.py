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
if rank == 0:
    import oracle
    print("ref", oracle.replay(tm, S, amp_q16=6554, kind_mask=7, threads=8)["iter"].tolist())
dist.barrier()
g.close()
dist.destroy_process_group()

"""Row e host logic on CPU: world_size-2 gloo process group (the N>1 path without a GPU).

Covers what every shard process does before its kernels run: the host-only plan (prism_plan,
identical on every shard), the DP-block partition of the ranks (disjoint, covering), and the
handle all-gather that feeds prism_shard_connect."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads as w


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2605_15617_b200 as P

        out = {}
        for name in ("C2", "C4"):
            tm = w.scaled(name)
            plan = P.plan(tm)
            own = P.shard_ranks(tm.topo, world, rank)
            got = [None] * world
            dist.all_gather_object(got, (plan, own))
            out[name] = got
        fake = bytes([rank]) * P.SHARD_HANDLE_BYTES
        out["handles"] = P.gather_handles(fake, world, rank)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_shard_plan_and_handles(world):
    import paper_2605_15617_b200 as P

    P.lib()  # the library must load (host-only calls below)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for name in ("C2", "C4"):
        tm = w.scaled(name)
        for r in range(world):
            plans = [g[0] for g in res[r][name]]
            assert all(p == plans[0] for p in plans)  # every shard plans the same graph
            owned = [set(g[1]) for g in res[r][name]]
            assert set().union(*owned) == set(range(tm.topo.world))
            assert sum(len(o) for o in owned) == tm.topo.world
    for r in range(world):
        assert res[r]["handles"] == [bytes([m]) * P.SHARD_HANDLE_BYTES for m in range(world)]


def test_dp_block_partition():
    import paper_2605_15617_b200 as P

    assert P.shard_dp_block(64, 8, 3) == (24, 32)
    with pytest.raises(ValueError):
        P.shard_dp_block(6, 4, 0)
    t = w.Topology(2, 3, 4, 2, 1, 1)  # Megatron order
    allr = sorted(r for i in range(4) for r in P.shard_ranks(t, 4, i))
    assert allr == list(range(24))

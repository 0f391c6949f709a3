"""Row e on the GPU: the rank-sharded replay (DP blocks, peer-memory exchange inside the cell
kernel) against the CPU oracle, bit-exact. All shards of a test live in one process on cuda:0,
each with its own stream, connected with prism_shard_connect_local and replayed together by
prism_replay_local_shards (one cooperative launch over every shard's cells, the cross-shard
exchange through the same peer-memory protocol as across GPUs); the multi-process path differs
in how the exchange buffers are mapped (CUDA IPC, prism_shard_connect) and in running one launch
per process."""
import os

import numpy as np
import pytest

import oracle
import workloads as w

pytestmark = pytest.mark.gpu
NPROC = os.cpu_count() or 1


@pytest.fixture(scope="module")
def prism():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_15617_b200 as P

    P.build_library()
    P.use_torch_allocator()
    return P


def _sharded(P, tm, n, S, axis="auto"):
    import torch

    streams = [torch.cuda.Stream() for _ in range(n)]
    gs = [P.Graph(tm, stream=streams[i].cuda_stream, n_shards=n, shard_index=i, shard_axis=axis) for i in range(n)]
    for g in gs:
        g.shard_prepare(S)
    for g in gs:
        g.shard_connect_local(gs)
    return gs, streams


def _replay_all(gs, S, **kw):
    import torch
    import paper_2605_15617_b200 as P

    out = torch.full((S,), -1, dtype=torch.int64, device="cuda")
    P.replay_local_shards(gs, out.data_ptr(), S, **kw)
    torch.cuda.synchronize()
    gs[0].sync()
    return [out.cpu().numpy()]


def _check(P, tm, n, S, reps=2, times=True, node_dur=None, axis="auto"):
    gs, _ = _sharded(P, tm, n, S, axis)
    if node_dur is not None:
        for g in gs:
            g.set_durations(node_dur=node_dur)
    ref = oracle.replay(tm, S, amp_q16=6554, kind_mask=7, times=times, threads=min(NPROC, S),
                        node_dur=node_dur)
    for rep in range(reps):  # repeated replays: exchange reset, parity flip, epoch flags
        outs = _replay_all(gs, S, amp_q16=6554, kind_mask=7)
        for i, o in enumerate(outs):
            assert np.array_equal(o, ref["iter"]), (rep, i, o[:4], ref["iter"][:4])
    for i, g in enumerate(gs):
        if not getattr(tm, "multistream", False):
            assert np.array_equal(g.peak_memory(), ref["peak"][0])
        assert g.last_algo() == "cells"
    if times:
        rng = np.random.default_rng(n)
        W = tm.topo.world
        rp = P.Graph(tm).export("rank_ptr")
        for i, g in enumerate(gs):
            own = g.owned_ranks()
            for r in rng.choice(own, min(8, len(own)), replace=False):
                for k in (0, S - 1):
                    st, fi, c = g.query_rank(int(r), k)
                    a, b = rp[r], rp[r + 1]
                    assert np.array_equal(fi, ref["finish"][k, a:b]) and np.array_equal(st, ref["start"][k, a:b])
            other = [r for r in range(W) if r not in set(own)]
            if other:
                with pytest.raises(P.PrismError):
                    g.query_rank(int(other[0]), 0)
        # gathered to every shard: any rank from any shard, and the critical path
        k = S - 1
        P.shard_gather_local(gs, k)
        for i, g in enumerate(gs):
            for r in rng.choice(W, min(6, W), replace=False):
                st, fi, _ = g.query_rank(int(r), k)
                a, b = rp[r], rp[r + 1]
                assert np.array_equal(fi, ref["finish"][k, a:b]) and np.array_equal(st, ref["start"][k, a:b])
        path, T = gs[-1].critical_path(k)
        rpath, rT = oracle.critical_path(tm, k, amp_q16=6554, kind_mask=7, node_dur=node_dur)
        assert T == rT == ref["iter"][k] and np.array_equal(path, rpath)
        if getattr(tm, "multistream", False):
            rt = oracle.replay(tm, 1, scen_first=k, amp_q16=6554, kind_mask=7, node_dur=node_dur)
            assert np.array_equal(gs[0].peak_memory_at(k), rt["peak"][0])
        if S > 1:
            with pytest.raises(P.PrismError):  # another scenario was not gathered
                gs[0].critical_path(0)
    for g in gs:
        g.close()


@pytest.mark.parametrize("name", ["C2", "C3", "C5"])
def test_sharded_scaled_dense(prism, name):
    _check(prism, w.scaled(name), 2, 64)


@pytest.mark.parametrize("n", [2, 4, 8])
def test_sharded_moe_ep_edp(prism, n):
    """C4-shaped MoE (dp 8, ep 4) forced onto DP blocks: EP all-to-alls and EDP groups span shards."""
    _check(prism, w.scaled("C4"), n, 33, axis="dp")


@pytest.mark.parametrize("n", [2, 4, 8])
def test_sharded_moe_pp_blocks(prism, n):
    """the MoE config sharded by PP-stage blocks (the planner's choice: EP
    all-to-alls stay inside a shard, only P2P messages at block edges cross)."""
    tm = w.scaled("C4")
    g = prism.Graph(tm, n_shards=n, shard_index=0)
    assert g.shard_info()["axis"] == "pp"
    g.close()
    _check(prism, tm, n, 33)


@pytest.mark.parametrize("axis", ["dp", "pp"])
@pytest.mark.parametrize("seed", range(400, 412))
def test_sharded_axes_random(prism, axis, seed):
    """Both shard axes forced on random templates (WORLD / EP / EDP collectives, batched P2P)."""
    tm = w.random_templates(seed, max_world=32, max_ops=40)
    if tm.topo.tp > 8 or (axis == "dp" and tm.topo.dp % 2) or (axis == "pp" and tm.topo.pp % 2):
        pytest.skip("needs an even block count on the axis and tp <= 8")
    _check(prism, tm, 2, [1, 5, 32, 40][seed % 4], axis=axis)


@pytest.mark.parametrize("n", [2, 4])
def test_sharded_dense_dp4(prism, n):
    tm = w.build_training_templates(w.TrainSetup(w.LLAMA3_70B, w.Topology(8, 4, 4), 8, [20] * 4), "dp4")
    _check(prism, tm, n, 64)


@pytest.mark.parametrize("seed", range(200, 230))
def test_sharded_random(prism, seed):
    tm = w.random_templates(seed, max_world=32, max_ops=40)
    if tm.topo.dp % 2 or tm.topo.tp > 8:
        pytest.skip("needs an even dp and tp <= 8")
    _check(prism, tm, 2, [1, 5, 32, 40][seed % 4], times=True)


def test_sharded_megatron_order(prism):
    tm = w.scaled("C2")
    tm = w.Templates(w.Topology(8, 8, 2, 1, 1, 1), tm.ops, tm.tmpl_ptr, tm.static_mem)
    _check(prism, tm, 2, 32)


def test_shard_errors(prism):
    tm = w.scaled("C2")
    with pytest.raises(prism.PrismError) as e:
        prism.Graph(tm, n_shards=3, shard_index=0)  # dp = 2
    assert e.value.name == "PRISM_E_INVALID_SPEC"
    g = prism.Graph(tm, n_shards=2, shard_index=0)
    with pytest.raises(prism.PrismError) as e:
        g.replay(4)
    assert e.value.name == "PRISM_E_INVALID_ARG"  # not connected
    g.close()
    gs, _ = _sharded(prism, tm, 2, 8)
    with pytest.raises(prism.PrismError) as e:  # same-device shards never replay in separate launches
        gs[0].replay(8)
    assert e.value.name == "PRISM_E_INVALID_ARG"
    import torch

    out = torch.zeros(8, dtype=torch.int64, device="cuda")
    with pytest.raises(prism.PrismError):  # scenario count differs from prepare's
        prism.replay_local_shards(gs, out.data_ptr(), 4)
    for g in gs:
        g.close()


def test_multiprocess_ipc(prism, tmp_path):
    """The multi-process path: 2 processes (torchrun, gloo for the handle all-gather) share cuda:0,
    map each other's exchange buffers with CUDA IPC (prism_shard_connect) and replay 3 times."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SHARD_DEVICE="0", PRISM_ALLOW_SAME_DEVICE_IPC="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29517",
                        os.path.join(root, "tests", "shard_mp_worker.py"), "C2"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l.split() for l in r.stdout.splitlines() if " rep " in l]
    ref = [l for l in r.stdout.splitlines() if l.startswith("ref")][0]
    want = ref[len("ref "):]
    assert len(lines) == 6
    for l in r.stdout.splitlines():
        if " rep " in l:
            assert " ok " in l and want in l, l
    reff = {int(l.split()[1]): l.split(" ", 2)[2] for l in r.stdout.splitlines() if l.startswith("reff")}
    gathered = [l for l in r.stdout.splitlines() if " gathered " in l]
    assert len(gathered) == 2
    for l in gathered:  # "<rank> gathered <other> <finishes> T <T> path <len> <sum>"
        other = int(l.split()[2])
        assert l.split(" ", 3)[3] == reff[other], (l[:200], reff[other][:200])


@pytest.mark.parametrize("seed", range(300, 316))
def test_sharded_multistream_and_durations(prism, seed):
    """Row e combined with rows f1/f2: multi-stream ranks (one rank per warp) and per-node
    measured durations, sharded over 2 DP blocks."""
    tm = w.random_templates(seed, max_world=32, max_ops=40, streams=2 + seed % 2)
    if tm.topo.dp % 2:
        pytest.skip("needs an even dp")
    tm.multistream = True
    d = np.random.default_rng(seed).integers(0, 900, tm.n_nodes) if seed % 2 else None
    _check(prism, tm, 2, [1, 5, 33][seed % 3], node_dur=d)


_C5_REF = {}


@pytest.mark.slow
@pytest.mark.parametrize("n", [2, 4, 8])
def test_sharded_full_c5(prism, n):
    """Full-size C5 (8192 ranks) sharded over 2 / 4 / 8 DP blocks of one device: all 64 iteration
    times and the owning shard's per-op times of sampled ranks equal the oracle's."""
    tm = w.config("C5")
    S = 64
    if "ref" not in _C5_REF:
        _C5_REF["ref"] = oracle.replay(tm, S, amp_q16=6554, kind_mask=7, peaks=False, threads=NPROC)
    ref = _C5_REF["ref"]
    gs, _ = _sharded(prism, tm, n, S)
    out = _replay_all(gs, S, amp_q16=6554, kind_mask=7)[0]
    assert np.array_equal(out, ref["iter"])
    for i, g in enumerate(gs):
        own = g.owned_ranks()
        for r in (own[0], own[len(own) // 2], own[-1]):
            _, fi, _ = g.query_rank(int(r), S - 1)
            assert fi[-1] == ref["rank_end"][S - 1, r]
    for g in gs:
        g.close()

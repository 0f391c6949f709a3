"""GPU: the host plan cache of prism_build_graph (abi.cu: builds of byte-identical templates reuse
the validated plan). A cached build must give exactly the replay and peaks of a fresh one, and any
change to the templates must miss the cache (the key is the input bytes themselves)."""
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


def _graph(P, tm, **kw):
    import torch

    return P.Graph(tm, stream=torch.cuda.current_stream().cuda_stream, **kw)


def _run(g, S=33):
    it = g.replay(S, amp_q16=6554, kind_mask=7)
    return it, g.peak_memory()


@pytest.mark.parametrize("name", ["C1", "C2", "C4"])
def test_cached_build_equals_fresh(prism, name):
    tm = w.config(name) if name == "C1" else w.scaled(name)
    ref = oracle.replay(tm, 33, amp_q16=6554, kind_mask=7, threads=NPROC)
    results = []
    for _ in range(3):  # the first build plans (or hits an earlier test's entry), the others hit
        g = _graph(prism, tm)
        results.append(_run(g))
        g.close()
    for it, pk in results:
        assert np.array_equal(it, ref["iter"])
        assert np.array_equal(pk, ref["peak"][0])


def test_changed_template_misses_cache(prism):
    tm = w.scaled("C2")
    g = _graph(prism, tm)
    it0, _ = _run(g)
    g.close()
    ops = tm.ops.copy()
    i = int(np.flatnonzero(ops["kind"] == 0)[3])  # a compute span of stage 0
    ops["dur_ns"][i] += 12345
    tm2 = w.Templates(tm.topo, ops, tm.tmpl_ptr, tm.static_mem)
    g2 = _graph(prism, tm2)
    it2, pk2 = _run(g2)
    g2.close()
    ref2 = oracle.replay(tm2, 33, amp_q16=6554, kind_mask=7, threads=NPROC)
    assert np.array_equal(it2, ref2["iter"])
    assert np.array_equal(pk2, ref2["peak"][0])
    assert not np.array_equal(it0, it2)


def test_interleaved_topologies(prism):
    """More distinct keys than cache entries, rebuilt in turn: every build is still exact."""
    tms = [w.scaled(n) for n in ("C2", "C3", "C4")] + [w.config("C1"),
                                                              w.random_templates(7, max_world=16, max_ops=30)]
    refs = [oracle.replay(tm, 33, amp_q16=6554, kind_mask=7, threads=NPROC)["iter"] for tm in tms]
    for rnd in range(2):
        for tm, ref in zip(tms, refs):
            g = _graph(prism, tm)
            it, _ = _run(g)
            g.close()
            assert np.array_equal(it, ref), (rnd, tm.topo)


def test_shard_options_are_part_of_the_key(prism):
    """The same templates built as shard 0 / shard 1 of 2 and unsharded: each build keeps its own
    shard layout (axis and block), on a miss and on a hit alike."""
    tm = w.scaled("C2")
    infos = {}
    for rnd in range(2):
        for opts in ({}, {"n_shards": 2, "shard_index": 0}, {"n_shards": 2, "shard_index": 1}):
            g = _graph(prism, tm, **opts)
            info = g.shard_info() if opts else None
            st = g.stats()
            g.close()
            key = tuple(sorted(opts.items()))
            if rnd == 0:
                infos[key] = (info, st)
            else:
                assert (info, st) == infos[key], key
    assert infos[(("n_shards", 2), ("shard_index", 0))][0] != infos[(("n_shards", 2), ("shard_index", 1))][0]

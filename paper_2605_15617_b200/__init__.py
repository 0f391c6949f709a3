"""paper_2605_15617_b200 — B200-native hot path of PrismLLM's hybrid emulation (arXiv 2605.15617).

A thin ctypes binding over the C ABI of ``libprism_b200.so`` (``include/prism.h``): argument
marshalling only, every step of the path runs in the CUDA kernels of ``csrc/``. PyTorch supplies
device memory (caching allocator hooks), the stream and, for multi-GPU runs, the process group.

There is no CPU fallback: if the library or a CUDA device is missing, every call raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Dict, Optional

import numpy as np

__all__ = ["lib", "Graph", "plan", "PrismError", "build_library", "LIB_PATH", "EXPORTED_SYMBOLS",
           "replay_local_shards"]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PRISM_LIB") or os.path.join(_HERE, "libprism_b200.so")  # PRISM_LIB: dev experiments

EXPORTED_SYMBOLS = [
    "prism_status_string", "prism_last_error", "prism_abi_version", "prism_set_allocator",
    "prism_build_graph", "prism_replay", "prism_replay_async", "prism_peak_memory",
    "prism_peak_memory_async", "prism_query_rank", "prism_graph_stats", "prism_destroy_graph",
    "prism_debug_export", "prism_plan", "prism_last_timing", "prism_last_algo",
    "prism_shard_prepare", "prism_shard_connect", "prism_shard_connect_local", "prism_shard_adopt",
    "prism_set_durations", "prism_critical_path", "prism_peak_memory_at", "prism_sync",
    "prism_debug_set", "prism_set_moe_load", "prism_replay_local_shards", "prism_shard_info",
    "prism_shard_gather", "prism_shard_gather_local",
]
SHARD_HANDLE_BYTES = 64

STATUS_NAMES = {
    0: "PRISM_OK", 1: "PRISM_E_INVALID_ARG", 2: "PRISM_E_INVALID_SPEC", 3: "PRISM_E_GA_TOO_SMALL",
    4: "PRISM_E_TEMPLATE_MISMATCH", 5: "PRISM_E_DEADLOCK", 6: "PRISM_E_NEGATIVE_MEMORY",
    7: "PRISM_E_UNKNOWN_RANK", 8: "PRISM_E_UNKNOWN_LABEL", 9: "PRISM_E_NOT_REPLAYED",
    10: "PRISM_E_OOM", 11: "PRISM_E_CUDA", 12: "PRISM_E_NCCL",
}


class PrismError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        self.name = STATUS_NAMES.get(status, str(status))
        super().__init__(f"{self.name}: {msg}")


class _Topology(ctypes.Structure):
    _fields_ = [("tp", ctypes.c_int32), ("pp", ctypes.c_int32), ("dp", ctypes.c_int32),
                ("ep", ctypes.c_int32), ("vpp", ctypes.c_int32), ("rank_order", ctypes.c_int32)]


class _Templates(ctypes.Structure):
    _fields_ = [("ops", ctypes.c_void_p), ("n_ops", ctypes.c_int64), ("tmpl_ptr", ctypes.c_void_p),
                ("static_mem", ctypes.c_void_p)]


class _BuildOpts(ctypes.Structure):
    _fields_ = [("stream", ctypes.c_void_p), ("device", ctypes.c_int32), ("n_shards", ctypes.c_int32),
                ("shard_index", ctypes.c_int32), ("flags", ctypes.c_int32)]


class _Scenarios(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("amp_q16", ctypes.c_int32), ("seed", ctypes.c_uint64),
                ("kind_mask", ctypes.c_uint32), ("record", ctypes.c_int32), ("algo", ctypes.c_int32),
                ("first", ctypes.c_int32), ("pad", ctypes.c_int32)]


class _MoeLoad(ctypes.Structure):
    _fields_ = [("op_event", ctypes.c_void_p), ("br_q16", ctypes.c_void_p), ("n_events", ctypes.c_int32),
                ("scale", ctypes.c_uint32)]


MOE_DUR, MOE_ALLOC, MOE_FREE = 1, 2, 4


class _Durations(ctypes.Structure):
    _fields_ = [("node_dur", ctypes.c_void_p), ("labels", ctypes.c_void_p), ("label_dur", ctypes.c_void_p),
                ("n_labels", ctypes.c_int32), ("pad", ctypes.c_int32), ("rank_slow_q16", ctypes.c_void_p),
                ("node_alloc", ctypes.c_void_p), ("node_free", ctypes.c_void_p)]


_ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
_FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)

_lib = None
_hooks = None


def build_library(force: bool = False, verbose: bool = False) -> str:
    from . import build as _b

    return _b.build(force=force, verbose=verbose)


def lib():
    """Load libprism_b200.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        L.prism_status_string.restype = ctypes.c_char_p
        L.prism_status_string.argtypes = [ctypes.c_int32]
        L.prism_last_error.restype = ctypes.c_char_p
        L.prism_abi_version.restype = ctypes.c_int32
        L.prism_set_allocator.argtypes = [_ALLOC_FN, _FREE_FN, P]
        L.prism_build_graph.argtypes = [P, P, P, ctypes.POINTER(P)]
        L.prism_replay.argtypes = [P, P, P]
        L.prism_replay_async.argtypes = [P, P, P]
        L.prism_peak_memory.argtypes = [P, P]
        L.prism_peak_memory_async.argtypes = [P, P]
        L.prism_query_rank.argtypes = [P, ctypes.c_int32, ctypes.c_int32, P, P, ctypes.c_int64, P, P]
        L.prism_graph_stats.argtypes = [P, P]
        L.prism_destroy_graph.argtypes = [P]
        L.prism_destroy_graph.restype = None
        L.prism_debug_export.argtypes = [P, ctypes.c_int32, P, ctypes.c_int64]
        L.prism_plan.argtypes = [P, P, P]
        L.prism_last_timing.argtypes = [P, P]
        L.prism_last_algo.argtypes = [P, P]
        L.prism_shard_prepare.argtypes = [P, ctypes.c_int32, P]
        L.prism_shard_connect.argtypes = [P, P]
        L.prism_shard_connect_local.argtypes = [P, P]
        L.prism_shard_adopt.argtypes = [P, P]
        L.prism_set_durations.argtypes = [P, P]
        L.prism_peak_memory_at.argtypes = [P, ctypes.c_int32, P]
        L.prism_critical_path.argtypes = [P, ctypes.c_int32, P, ctypes.c_int64, P, P]
        L.prism_sync.argtypes = [P]
        L.prism_set_moe_load.argtypes = [P, P]
        L.prism_replay_local_shards.argtypes = [P, ctypes.c_int32, P, P]
        L.prism_shard_info.argtypes = [P, P]
        L.prism_shard_gather.argtypes = [P, ctypes.c_int32]
        L.prism_shard_gather_local.argtypes = [P, ctypes.c_int32, ctypes.c_int32]
        L.prism_debug_set.argtypes = [P, ctypes.c_int32, ctypes.c_int64]
        for name in ("prism_set_allocator", "prism_build_graph", "prism_replay", "prism_replay_async",
                     "prism_peak_memory", "prism_peak_memory_async", "prism_query_rank",
                     "prism_graph_stats", "prism_debug_export", "prism_plan",
                     "prism_last_timing", "prism_last_algo", "prism_shard_prepare",
                     "prism_shard_connect", "prism_shard_connect_local", "prism_shard_adopt",
                     "prism_set_durations", "prism_critical_path", "prism_peak_memory_at",
                     "prism_sync", "prism_debug_set", "prism_set_moe_load", "prism_replay_local_shards",
                     "prism_shard_info", "prism_shard_gather", "prism_shard_gather_local"):
            getattr(L, name).restype = ctypes.c_int32
        _lib = L
    return _lib


def _check(status: int):
    if status != 0:
        raise PrismError(status, lib().prism_last_error().decode(errors="replace"))


def use_torch_allocator() -> None:
    """Route the library's device allocations through PyTorch's caching allocator. Idempotent: a
    graph keeps the hooks it was built with, so the ctypes thunks are installed once and live for
    the process (replacing them would leave older graphs calling freed thunks on destroy)."""
    global _hooks
    if _hooks is not None:
        return
    import torch

    def _alloc(nbytes, stream, ctx):
        try:
            return int(torch.cuda.caching_allocator_alloc(int(nbytes), stream=int(stream or 0)))
        except Exception:  # allocation failure -> NULL -> PRISM_E_OOM
            return None

    def _free(ptr, stream, ctx):
        torch.cuda.caching_allocator_delete(int(ptr))

    _hooks = (_ALLOC_FN(_alloc), _FREE_FN(_free))
    _check(lib().prism_set_allocator(_hooks[0], _hooks[1], None))


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


DEBUG_ARRAYS = {
    "rank_ptr": (0, np.int32), "node_rank": (1, np.int32), "node_dur": (2, np.int64),
    "node_kind": (3, np.uint8), "node_label": (4, np.uint32), "node_alloc": (5, np.int64),
    "node_free": (6, np.int64), "node_prev_sync": (7, np.int32), "node_gptr": (8, np.int32),
    "node_grp": (9, np.int32), "grp_ptr": (10, np.int32), "grp_mem": (11, np.int32),
    "grp_dur": (12, np.int64), "grp_uid": (13, np.uint64), "grp_level": (14, np.int32),
}


def _marshal(templates):
    t = templates.topo
    topo = _Topology(t.tp, t.pp, t.dp, t.ep, getattr(t, "vpp", 1), getattr(t, "rank_order", 0))
    ops = np.ascontiguousarray(templates.ops)
    if ops.dtype.itemsize != 48:
        raise ValueError("ops must use the 48-byte prism_op record layout")
    ptr = np.ascontiguousarray(templates.tmpl_ptr, dtype=np.int64)
    static = np.ascontiguousarray(templates.static_mem, dtype=np.int64)
    tm = _Templates(ops.ctypes.data if len(ops) else None, len(ops), ptr.ctypes.data, static.ctypes.data)
    return topo, tm, (ops, ptr, static)


def plan(templates) -> Dict[str, int]:
    """Host-only validation + quotient plan (prism_plan): sizes of the graph that would be built."""
    topo, tm, keep = _marshal(templates)
    out = np.zeros(8, np.int64)
    _check(lib().prism_plan(ctypes.byref(topo), ctypes.byref(tm), _ptr(out)))
    keys = ["world", "nodes", "groups", "memberships", "levels", "quotient_groups", "sync_nodes",
            "max_group"]
    return dict(zip(keys, (int(x) for x in out)))


class Graph:
    """An expanded execution graph resident on one GPU (prism_build_graph)."""

    SHARD_AXES = {"auto": 0, "dp": 4, "pp": 8}

    def __init__(self, templates, *, stream: Optional[int] = None, device: int = -1,
                 profile: bool = False, n_shards: int = 1, shard_index: int = 0, asynchronous: bool = False,
                 shard_axis: str = "auto"):
        L = lib()
        self.topo = templates.topo
        self.n_shards, self.shard_index = int(n_shards), int(shard_index)
        self._topo, self._tm, self._keep = _marshal(templates)
        flags = (1 if profile else 0) | (2 if asynchronous else 0) | self.SHARD_AXES[shard_axis]
        self._opts = _BuildOpts(stream or 0, device, self.n_shards, self.shard_index, flags)
        h = ctypes.c_void_p()
        self._h = None
        _check(L.prism_build_graph(ctypes.byref(self._topo), ctypes.byref(self._tm),
                                   ctypes.byref(self._opts), ctypes.byref(h)))
        self._h = h
        self._stats = None

    # ---------------------------------------------------------------- lifetime
    def close(self):
        if self._h is not None and _lib is not None:
            _lib.prism_destroy_graph(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---------------------------------------------------------------- calls
    def stats(self) -> Dict[str, int]:
        out = np.zeros(10, np.int64)
        _check(lib().prism_graph_stats(self._h, _ptr(out)))
        keys = ["world", "nodes", "groups", "memberships", "levels", "quotient_groups", "sync_nodes",
                "max_group", "structure_bytes", "replay_launches"]
        return dict(zip(keys, (int(x) for x in out)))

    def last_timing(self) -> Dict[str, float]:
        """Device ms of the last expand / level loop / tail / reduce / peak (profile=True graphs)."""
        out = np.zeros(5, np.float32)
        _check(lib().prism_last_timing(self._h, _ptr(out)))
        return dict(zip(["expand", "levels", "tail", "reduce", "peak"], (float(x) for x in out)))

    ALGOS = {"auto": 0, "levels": 1, "cells": 2, "ranks": 3}

    @classmethod
    def _scen(cls, n, seed, amp_q16, kind_mask, record, algo, first=0):
        return _Scenarios(int(n), int(amp_q16), int(seed) & (2**64 - 1), int(kind_mask), int(bool(record)),
                          cls.ALGOS[algo], int(first), 0)

    def replay(self, n: int = 1, *, seed: int = 0x5EED, amp_q16: int = 0, kind_mask: int = 0,
               record: bool = True, algo: str = "auto", first: int = 0) -> np.ndarray:
        """Iteration time (ns) of each of n scenarios first .. first+n-1 (host result, synchronizing)."""
        out = np.zeros(n, np.int64)
        sc = self._scen(n, seed, amp_q16, kind_mask, record, algo, first)
        _check(lib().prism_replay(self._h, ctypes.byref(sc), _ptr(out)))
        return out

    def replay_async(self, iter_dev_ptr: int, n: int = 1, *, seed: int = 0x5EED, amp_q16: int = 0,
                     kind_mask: int = 0, record: bool = True, algo: str = "auto", first: int = 0) -> None:
        """Asynchronous replay writing n int64 iteration times to a DEVICE pointer."""
        sc = self._scen(n, seed, amp_q16, kind_mask, record, algo, first)
        _check(lib().prism_replay_async(self._h, ctypes.byref(sc), ctypes.c_void_p(iter_dev_ptr)))

    def sync(self) -> None:
        """Wait for the graph's queued work; raises PrismError(PRISM_E_DEADLOCK) if a replay since the
        last synchronising call was aborted by the device watchdog (prism_sync)."""
        _check(lib().prism_sync(self._h))

    def debug_set(self, key: str, value: int) -> None:
        """Watchdog test hooks: key 'watchdog_ns' or 'stall_unit' (prism_debug_set)."""
        _check(lib().prism_debug_set(self._h, {"watchdog_ns": 0, "stall_unit": 1}[key], int(value)))

    def last_algo(self) -> str:
        v = ctypes.c_int32(0)
        _check(lib().prism_last_algo(self._h, ctypes.byref(v)))
        return {0: "none", 1: "levels", 2: "cells", 3: "ranks"}[v.value]

    def peak_memory(self) -> np.ndarray:
        out = np.zeros(self.topo.tp * self.topo.pp * self.topo.dp, np.int64)
        _check(lib().prism_peak_memory(self._h, _ptr(out)))
        return out

    def peak_memory_at(self, scenario: int = 0) -> np.ndarray:
        """Row f2: per-rank peak with events in time order, scenario of the last recorded replay."""
        out = np.zeros(self.topo.tp * self.topo.pp * self.topo.dp, np.int64)
        _check(lib().prism_peak_memory_at(self._h, int(scenario), _ptr(out)))
        return out

    def peak_memory_async(self, peak_dev_ptr: int) -> None:
        _check(lib().prism_peak_memory_async(self._h, ctypes.c_void_p(peak_dev_ptr)))

    def query_rank(self, rank: int, scenario: int = 0):
        """(start[n_ops], finish[n_ops], coords(tp, pp, dp, ep, edp)) of one rank."""
        n = ctypes.c_int64(0)
        coords = np.zeros(5, np.int32)
        st = lib().prism_query_rank(self._h, rank, scenario, None, None, 0, ctypes.byref(n), _ptr(coords))
        if st not in (0, 1):
            _check(st)
        start = np.zeros(max(1, n.value), np.int64)
        fin = np.zeros(max(1, n.value), np.int64)
        _check(lib().prism_query_rank(self._h, rank, scenario, _ptr(start), _ptr(fin), n.value, None, None))
        return start[: n.value], fin[: n.value], tuple(int(c) for c in coords)

    # ---------------------------------------------------------------- rows f1 / f3 / f4
    def set_durations(self, *, node_dur=None, label_dur=None, rank_slow_q16=None, node_alloc=None,
                      node_free=None) -> None:
        """Per-node durations (f1 calibration input), label overrides {label: ns} and per-rank
        compute slowdown in Q16 (f3 what-if / fault injection), per-node memory deltas (f4); no
        arguments = back to the templates. Applies to later replays (prism_set_durations).
        node_dur / node_alloc / node_free: numpy arrays or contiguous 1-D int64 CUDA tensors (one
        entry per node; copied on the device, no host upload)."""
        keep = []

        def arr(a, dt):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dtype=dt)
            keep.append(a)
            return a.ctypes.data

        def node_arr(a):  # per-node arrays: host (numpy) or a CUDA int64 tensor (copied on the device)
            if a is not None and type(a).__module__.startswith("torch") and getattr(a, "is_cuda", False):
                import torch

                if a.dtype != torch.int64 or a.dim() != 1 or not a.is_contiguous():
                    raise ValueError("per-node device arrays must be contiguous 1-D int64 CUDA tensors")
                if a.numel() != self.stats()["nodes"]:
                    raise ValueError("per-node arrays need one entry per node")
                keep.append(a)
                return a.data_ptr()
            return arr(a, np.int64)

        labs = sorted((label_dur or {}).items())
        la = np.array([int(k) for k, _ in labs], np.uint32)
        ld = np.array([int(v) for _, v in labs], np.int64)
        d = _Durations(node_arr(node_dur), arr(la, np.uint32) if len(la) else None,
                       arr(ld, np.int64) if len(ld) else None, len(labs), 0, arr(rank_slow_q16, np.int32),
                       node_arr(node_alloc), node_arr(node_free))
        _check(lib().prism_set_durations(self._h, ctypes.byref(d)))

    def set_moe_load(self, op_event=None, br_q16=None, scale: int = MOE_DUR | MOE_ALLOC | MOE_FREE) -> None:
        """Row f4 (prism_set_moe_load): op_event[n_ops] = gating event of each template op (-1 = not
        routed), br_q16[n_events, ep] = balance ratios in Q16; None clears the load."""
        if op_event is None:
            _check(lib().prism_set_moe_load(self._h, None))
            return
        ev = np.ascontiguousarray(op_event, dtype=np.int32)
        br = np.ascontiguousarray(br_q16, dtype=np.int32)
        if br.ndim != 2 or br.shape[1] != self.topo.ep:
            raise ValueError("br_q16 must have shape (n_events, ep)")
        m = _MoeLoad(ev.ctypes.data, br.ctypes.data, br.shape[0], int(scale))
        _check(lib().prism_set_moe_load(self._h, ctypes.byref(m)))

    def critical_path(self, scenario: int = 0):
        """(path [node ids, last first], T) of one scenario of the last recorded replay."""
        n = ctypes.c_int64(0)
        T = ctypes.c_int64(0)
        path = np.zeros(1 << 16, np.int32)  # one call in the common case; retried if the path is longer
        st = lib().prism_critical_path(self._h, int(scenario), _ptr(path), len(path), ctypes.byref(n),
                                       ctypes.byref(T))
        if st == 1 and n.value > len(path):
            path = np.zeros(n.value, np.int32)
            st = lib().prism_critical_path(self._h, int(scenario), _ptr(path), len(path), ctypes.byref(n),
                                           ctypes.byref(T))
        _check(st)
        return path[: n.value].copy(), int(T.value)

    # ---------------------------------------------------------------- row e: sharding
    def shard_info(self) -> Dict[str, object]:
        """n_shards, shard, axis ('dp' or 'pp' blocks) and block size of this graph."""
        out = np.zeros(4, np.int32)
        _check(lib().prism_shard_info(self._h, _ptr(out)))
        return {"n_shards": int(out[0]), "shard": int(out[1]), "axis": "pp" if out[2] == 1 else "dp",
                "block": int(out[3])}

    def owned_ranks(self):
        """The global ranks this shard replays (all of them unsharded)."""
        info = self.shard_info()
        return shard_ranks(self.topo, info["n_shards"], info["shard"], info["axis"])

    def shard_gather(self, scenario: int) -> None:
        """Collective over the shards (one per process): every rank's recorded times of `scenario`
        to every shard, so query_rank / critical_path / peak_memory_at answer for all ranks."""
        _check(lib().prism_shard_gather(self._h, int(scenario)))

    def shard_prepare(self, n_scenarios: int) -> bytes:
        """Allocate this shard's exchange buffer for replays of n_scenarios; returns its IPC handle."""
        h = ctypes.create_string_buffer(SHARD_HANDLE_BYTES)
        _check(lib().prism_shard_prepare(self._h, int(n_scenarios), h))
        return h.raw

    def shard_connect(self, handles) -> None:
        """Open the peers' exchange buffers (handles[m] = shard m's shard_prepare result)."""
        if len(handles) != self.n_shards:
            raise ValueError("need one handle per shard")
        buf = ctypes.create_string_buffer(b"".join(bytes(h) for h in handles), SHARD_HANDLE_BYTES * self.n_shards)
        _check(lib().prism_shard_connect(self._h, buf))

    def shard_connect_local(self, graphs) -> None:
        """Connect to the other shards of the same process (graphs[m] = shard m)."""
        arr = (ctypes.c_void_p * len(graphs))(*[g._h.value for g in graphs])
        _check(lib().prism_shard_connect_local(self._h, arr))

    def shard_adopt(self, other: "Graph") -> None:
        """Take over the connected exchange buffer of `other` (same plan and shard)."""
        _check(lib().prism_shard_adopt(self._h, other._h))

    def shard_connect_dist(self, n_scenarios: int, group=None) -> None:
        """SPMD helper: prepare, all-gather the handles over torch.distributed, connect."""
        import torch.distributed as dist

        mine = self.shard_prepare(n_scenarios)
        self.shard_connect(gather_handles(mine, self.n_shards, self.shard_index, group))

    def export(self, name: str, scen_pad: int = 0) -> np.ndarray:
        """Copy one device CSR array to the host (tests)."""
        st = self.stats()
        if name == "fin":
            which, dt, count = 15, np.int64, st["nodes"] * scen_pad
        else:
            which, dt = DEBUG_ARRAYS[name]
            W, N, G, M = st["world"], st["nodes"], st["groups"], st["memberships"]
            count = {"rank_ptr": W + 1, "node_gptr": N + 1, "grp_ptr": G + 1, "node_grp": M,
                     "grp_mem": M}.get(name)
            if count is None:
                count = G if name.startswith("grp_") else N
        out = np.zeros(max(1, count), dt)
        _check(lib().prism_debug_export(self._h, which, _ptr(out), out.nbytes))
        return out[:count]


def replay_local_shards(graphs, iter_dev_ptr: int, n: int = 1, *, seed: int = 0x5EED, amp_q16: int = 0,
                        kind_mask: int = 0, record: bool = True, first: int = 0) -> None:
    """Row e, shards sharing one device (prism_replay_local_shards): one cooperative launch replays
    every shard (graphs[i] = shard i, connected with shard_connect_local); n int64 iteration times
    are written to the DEVICE pointer on graphs[0]'s stream."""
    arr = (ctypes.c_void_p * len(graphs))(*[g._h.value for g in graphs])
    sc = Graph._scen(n, seed, amp_q16, kind_mask, record, "auto", first)
    _check(lib().prism_replay_local_shards(arr, len(graphs), ctypes.byref(sc), ctypes.c_void_p(iter_dev_ptr)))


def shard_gather_local(graphs, scenario: int) -> None:
    """prism_shard_gather for the shards of one device (graphs[i] = shard i), in one launch."""
    arr = (ctypes.c_void_p * len(graphs))(*[g._h.value for g in graphs])
    _check(lib().prism_shard_gather_local(arr, len(graphs), int(scenario)))


def gather_handles(mine: bytes, n_shards: int, shard_index: int, group=None):
    """All-gather every shard's exchange-buffer handle over torch.distributed, ordered by shard."""
    import torch.distributed as dist

    if dist.get_world_size(group) != n_shards:
        raise ValueError("the process group must hold exactly one process per shard")
    allh = [None] * n_shards
    dist.all_gather_object(allh, (shard_index, bytes(mine)), group=group)
    idx = [i for i, _ in allh]
    if sorted(idx) != list(range(n_shards)):
        raise ValueError(f"shard indices {idx} are not a permutation of 0..{n_shards - 1}")
    return [h for _, h in sorted(allh)]


def shard_dp_block(dp: int, n_shards: int, shard_index: int):
    """Row e host logic: the DP coordinates [d0, d1) replayed by one shard (DP-block sharding,
    include/prism.h "multi-GPU"); dp must be a multiple of n_shards."""
    if n_shards < 1 or dp % n_shards or not 0 <= shard_index < n_shards:
        raise ValueError("dp must be a multiple of n_shards and shard_index in [0, n_shards)")
    b = dp // n_shards
    return b * shard_index, b * (shard_index + 1)


def shard_ranks(topo, n_shards: int, shard_index: int, axis: str = "dp"):
    """The global ranks a shard owns: every (tp, pp) coordinate of its DP block, or every (tp, dp)
    coordinate of its PP-stage block (axis 'pp'); rank numbering of reading Z1."""
    if n_shards <= 1:
        return list(range(topo.tp * topo.pp * topo.dp))
    if axis == "pp":
        s0, s1 = shard_dp_block(topo.pp, n_shards, shard_index)
        d0, d1 = 0, topo.dp
    else:
        d0, d1 = shard_dp_block(topo.dp, n_shards, shard_index)
        s0, s1 = 0, topo.pp
    out = []
    for dpi in range(d0, d1):
        for s in range(s0, s1):
            for t in range(topo.tp):
                out.append(t + topo.tp * (s + topo.pp * dpi) if getattr(topo, "rank_order", 0) == 0
                           else t + topo.tp * (dpi + topo.dp * s))
    return sorted(out)

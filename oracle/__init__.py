"""CPU oracle for the PrismLLM hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package. The product path
(``paper_2605_15617_b200``) never imports it and fails loudly without its CUDA library.

``prism_oracle.cpp`` is a plain discrete-event replayer with its own template expansion
(PAPER.md P:982, P:1099, P:1298, P:1573, P:1578 — see the file header); ``brute.py`` is a
pure-Python path enumeration for tiny graphs used to pin the DES itself.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from typing import Dict, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "prism_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

STATUS = {0: "OK", 1: "INVALID_ARG", 2: "INVALID_SPEC", 4: "TEMPLATE_MISMATCH", 5: "DEADLOCK",
          6: "NEGATIVE_MEMORY"}


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


def build(force: bool = False) -> str:
    """Compile liboracle.so with g++ (building the checker is not using it)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-pthread", _SRC,
                               "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            lib.oracle_expand.argtypes = [P, P, ctypes.c_int64, P, P, P, P, P, P, P, P,
                                          ctypes.c_char_p, ctypes.c_int]
            lib.oracle_expand.restype = ctypes.c_int
            lib.oracle_replay.argtypes = [P, P, ctypes.c_int64, P, P, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.c_uint64, ctypes.c_int32, ctypes.c_uint32, P, P, P,
                                          P, P, ctypes.c_int32, ctypes.c_char_p, ctypes.c_int]
            lib.oracle_replay.restype = ctypes.c_int
            lib.oracle_replay_ov.argtypes = [P, P, ctypes.c_int64, P, P, P, P, P, ctypes.c_int32,
                                             ctypes.c_int32, ctypes.c_uint64, ctypes.c_int32,
                                             ctypes.c_uint32, P, P, P, P, P, ctypes.c_int32,
                                             ctypes.c_char_p, ctypes.c_int]
            lib.oracle_replay_ov.restype = ctypes.c_int
            lib.oracle_critical_path.argtypes = [P, P, ctypes.c_int64, P, P, P, ctypes.c_int32,
                                                 ctypes.c_uint64, ctypes.c_int32, ctypes.c_uint32, P,
                                                 ctypes.c_int64, P, P, ctypes.c_char_p, ctypes.c_int]
            lib.oracle_critical_path.restype = ctypes.c_int
            lib.oracle_moe_load.argtypes = [P, P, ctypes.c_int64, P, P, P, ctypes.c_int32, ctypes.c_uint32,
                                            P, P, P, P, P, P]
            lib.oracle_moe_load.restype = ctypes.c_int
            lib.oracle_splitmix64.argtypes = [ctypes.c_uint64]
            lib.oracle_splitmix64.restype = ctypes.c_uint64
            lib.oracle_perturb.argtypes = [ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32,
                                           ctypes.c_uint64, ctypes.c_int32]
            lib.oracle_perturb.restype = ctypes.c_int64
            _lib = lib
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _topo_buf(topo) -> np.ndarray:
    return np.array([topo.tp, topo.pp, topo.dp, topo.ep, topo.vpp, topo.rank_order], dtype=np.int32)


def _inputs(tm):
    ops = np.ascontiguousarray(tm.ops)
    ptr = np.ascontiguousarray(tm.tmpl_ptr, dtype=np.int64)
    st = np.ascontiguousarray(tm.static_mem, dtype=np.int64)
    return ops, ptr, st


def expand(tm) -> Dict[str, np.ndarray]:
    """The oracle's expanded sync groups: uid, dur, level, member node ids (sorted)."""
    lib = _load()
    topo = _topo_buf(tm.topo)
    ops, ptr, st = _inputs(tm)
    stats = np.zeros(8, dtype=np.int64)
    err = ctypes.create_string_buffer(512)
    s = lib.oracle_expand(_ptr(topo), _ptr(ops), len(ops), _ptr(ptr), _ptr(st), _ptr(stats),
                          None, None, None, None, None, err, 512)
    if s:
        raise OracleError(s, err.value.decode())
    G, M = int(stats[2]), int(stats[3])
    uid = np.zeros(G, np.uint64)
    dur = np.zeros(G, np.int64)
    gptr = np.zeros(G + 1, np.int64)
    mem = np.zeros(M, np.int32)
    lvl = np.zeros(G, np.int64)
    s = lib.oracle_expand(_ptr(topo), _ptr(ops), len(ops), _ptr(ptr), _ptr(st), _ptr(stats),
                          _ptr(uid), _ptr(dur), _ptr(gptr), _ptr(mem), _ptr(lvl), err, 512)
    if s:
        raise OracleError(s, err.value.decode())
    return {"stats": stats, "uid": uid, "dur": dur, "ptr": gptr, "mem": mem, "level": lvl,
            "world": int(stats[0]), "nodes": int(stats[1]), "groups": G, "memberships": M,
            "levels": int(stats[4]), "sync_nodes": int(stats[5]), "max_group": int(stats[6])}


def _opt64(a, n):
    if a is None:
        return None
    a = np.ascontiguousarray(a, dtype=np.int64)
    if a.shape != (n,):
        raise ValueError(f"per-node override must have shape ({n},)")
    return a


def replay(tm, n_scen: int = 1, *, seed: int = 0x5EED, amp_q16: int = 0, kind_mask: int = 0,
           scen_first: int = 0, times: bool = False, peaks: bool = True, threads: int = 1,
           node_dur=None, node_alloc=None, node_free=None):
    """Replay scenarios scen_first .. scen_first+n_scen-1. Returns a dict with
    iter [S], rank_end [S, W], peak [S, W] (if peaks), start/finish [S, N] (if times).
    node_dur / node_alloc / node_free: optional per-node overrides (rows f1/f3/f4), node order =
    rank-major program order; a sync group lasts the max of its members' durations (Z2)."""
    lib = _load()
    topo = _topo_buf(tm.topo)
    ops, ptr, st = _inputs(tm)
    W = tm.topo.world
    N = tm.n_nodes
    it = np.zeros(n_scen, np.int64)
    re = np.zeros((n_scen, W), np.int64)
    pk = np.zeros((n_scen, W), np.int64) if peaks else None
    s0 = np.zeros((n_scen, N), np.int64) if times else None
    f0 = np.zeros((n_scen, N), np.int64) if times else None
    err = ctypes.create_string_buffer(512)
    nd, na, nf = _opt64(node_dur, N), _opt64(node_alloc, N), _opt64(node_free, N)
    s = lib.oracle_replay_ov(_ptr(topo), _ptr(ops), len(ops), _ptr(ptr), _ptr(st), _ptr(nd), _ptr(na),
                             _ptr(nf), scen_first, n_scen, seed, amp_q16, kind_mask, _ptr(it), _ptr(re),
                             _ptr(pk), _ptr(s0), _ptr(f0), threads, err, 512)
    if s:
        raise OracleError(s, err.value.decode())
    out = {"iter": it, "rank_end": re}
    if peaks:
        out["peak"] = pk
    if times:
        out["start"] = s0
        out["finish"] = f0
    return out


def splitmix64(x: int) -> int:
    return int(_load().oracle_splitmix64(x & (2**64 - 1)))


def perturb(d: int, uid: int, k: int, seed: int, amp: int) -> int:
    return int(_load().oracle_perturb(d, uid & (2**64 - 1), k, seed & (2**64 - 1), amp))


def critical_path(tm, k: int = 0, *, seed: int = 0x5EED, amp_q16: int = 0, kind_mask: int = 0,
                  node_dur=None):
    """Row f3: (path [nodes, last first], T) of scenario k (walk and tie rules: prism_oracle.cpp
    oracle_critical_path)."""
    lib = _load()
    topo = _topo_buf(tm.topo)
    ops, ptr, st = _inputs(tm)
    N = tm.n_nodes
    nd = _opt64(node_dur, N)
    cap = N + 1
    path = np.zeros(cap, np.int32)
    n = ctypes.c_int64(0)
    T = ctypes.c_int64(0)
    err = ctypes.create_string_buffer(512)
    s = lib.oracle_critical_path(_ptr(topo), _ptr(ops), len(ops), _ptr(ptr), _ptr(st), _ptr(nd), k, seed,
                                 amp_q16, kind_mask, _ptr(path), cap, ctypes.byref(n), ctypes.byref(T), err, 512)
    if s:
        raise OracleError(s, err.value.decode())
    return path[: n.value].copy(), int(T.value)


def node_table(tm) -> Dict[str, np.ndarray]:
    """Per-node (rank-major program order) rank, template index, kind, label and template duration,
    expanded with plain loops from the templates (every rank of stage s runs template s)."""
    t = tm.topo
    rank, tidx, kind, label, dur = [], [], [], [], []
    for r in range(t.world):
        s = (r // t.tp) % t.pp if t.rank_order == 0 else r // (t.tp * t.dp)
        T = tm.stage(s)
        n = len(T)
        rank.append(np.full(n, r, np.int32))
        tidx.append(np.arange(n, dtype=np.int32))
        kind.append(T["kind"].astype(np.uint8))
        label.append(T["label"].astype(np.uint32))
        dur.append(T["dur_ns"].astype(np.int64))
    cat = (lambda xs, dt: np.concatenate(xs) if xs else np.zeros(0, dt))
    return {"rank": cat(rank, np.int32), "tidx": cat(tidx, np.int32), "kind": cat(kind, np.uint8),
            "label": cat(label, np.uint32), "dur": cat(dur, np.int64)}


class UnknownLabel(OracleError):
    def __init__(self, label):
        RuntimeError.__init__(self, f"UNKNOWN_LABEL: no node carries label {label:#x}")
        self.status, self.name = 8, "UNKNOWN_LABEL"


def whatif_durations(tm, *, node_dur=None, label_dur=None, rank_factor_q16=None) -> np.ndarray:
    """Row f3 (SPEC S:488-505 what_if / fault_inject): per-node durations after
    (1) the base (node_dur, else the template durations), (2) label overrides: every node whose
    label is a key of label_dur lasts label_dur[label] (UnknownLabel if no node carries it),
    (3) fault injection: every COMPUTE node of rank r lasts (d * rank_factor_q16[r]) >> 16."""
    nt = node_table(tm)
    d = (np.array(node_dur, dtype=np.int64) if node_dur is not None else nt["dur"].copy())
    for lab, v in (label_dur or {}).items():
        hit = nt["label"] == np.uint32(lab)
        if not hit.any():
            raise UnknownLabel(int(lab))
        d[hit] = int(v)
    if rank_factor_q16 is not None:
        f = np.asarray(rank_factor_q16, dtype=np.int64)
        comp = nt["kind"] == 0
        for i in np.nonzero(comp)[0]:  # plain loop: the definition, element by element
            d[i] = (int(d[i]) * int(f[nt["rank"][i]])) >> 16
    return d


def moe_load(tm, op_event, br_q16, scale: int = 7, *, node_dur=None, node_alloc=None, node_free=None):
    """Row f4 (App. F mock router; reading R7): per-node (duration, alloc, free) when
    every op routed by gating event v on a rank with EP coordinate e processes br_q16[v, e] / 65536
    times the uniform volume (floor; scale bits 1 duration, 2 alloc, 4 free). Base values: the given
    per-node arrays, else the templates. Feed the result to replay(node_dur=..., ...)."""
    lib = _load()
    topo = _topo_buf(tm.topo)
    ops, ptr, _ = _inputs(tm)
    ev = np.ascontiguousarray(op_event, dtype=np.int32)
    br = np.ascontiguousarray(br_q16, dtype=np.int32)
    if len(ev) != len(ops) or br.ndim != 2 or br.shape[1] != tm.topo.ep:
        raise ValueError("op_event must have one entry per template op, br_q16 shape (events, ep)")
    N = tm.n_nodes
    d, a, f = np.zeros(N, np.int64), np.zeros(N, np.int64), np.zeros(N, np.int64)
    nd, na, nf = _opt64(node_dur, N), _opt64(node_alloc, N), _opt64(node_free, N)
    s = lib.oracle_moe_load(_ptr(topo), _ptr(ops), len(ops), _ptr(ptr), _ptr(ev), _ptr(br), br.shape[0],
                            int(scale), _ptr(nd), _ptr(na), _ptr(nf), _ptr(d), _ptr(a), _ptr(f))
    if s:
        raise OracleError(s, "op_event / template mismatch")
    return d, a, f


def slice_local_finish(tm, node_dur, slices) -> np.ndarray:
    """Row f1, the UNcalibrated timing (reading R5): each slice's real ranks are timed
    in a run where every other rank is a virtual rank replaying the bare graph, i.e. with zero
    durations; a node's slice-local finish is taken from the run of its own rank's
    slice. Concatenating them is what inter-slice calibration corrects."""
    nt = node_table(tm)
    d = np.asarray(node_dur, dtype=np.int64)
    out = np.zeros(len(d), np.int64)
    for ranks in slices:
        sel = np.isin(nt["rank"], np.asarray(list(ranks), dtype=np.int32))
        r = replay(tm, 1, node_dur=np.where(sel, d, 0), times=True, peaks=False)
        out[sel] = r["finish"][0][sel]
    return out

"""Brute-force longest-path evaluation for TINY graphs — TEST INFRASTRUCTURE ONLY.

A second, independent statement of what the replay computes, used to pin the C++ DES
("length computed by exhaustive schedule enumeration"; "critical-path length
equals the makespan of the ASAP schedule").

The graph is rewritten as a plain vertex-weighted DAG:
  * one vertex per compute node, weight = its duration, with an edge from its stream predecessor
    (and, row f2, from the latest earlier op recording the event slot it waits on);
  * one vertex per sync group, weight = the group's duration (max of its members' op durations,
    reading Z2), with an edge from the stream predecessor of each member (all
    participants must reach the operation before any can proceed);
  * one zero-weight vertex per sync node, with an edge from each of its groups; its stream
    successor hangs off it.
finish(v) = the maximum over ALL source->v paths of the summed weights, found by explicit path
enumeration (exponential; only for graphs of a few dozen vertices). The iteration time is the
maximum finish.
"""
from __future__ import annotations

from typing import Dict, List, Tuple


def _coords(topo, r):
    tp = r % topo.tp
    if topo.rank_order == 1:
        dp = (r // topo.tp) % topo.dp
        pp = r // (topo.tp * topo.dp)
    else:
        pp = (r // topo.tp) % topo.pp
        dp = r // (topo.tp * topo.pp)
    return tp, pp, dp, dp % topo.ep, dp // topo.ep


def _rank(topo, tp, pp, dp):
    if topo.rank_order == 1:
        return tp + topo.tp * (dp + topo.dp * pp)
    return tp + topo.tp * (pp + topo.pp * dp)


def expand(tm, node_dur=None):
    """Returns (nodes, groups): nodes[n] = (rank, tidx, op); groups: key -> list of (node, dur).
    node_dur (optional, per node): durations replacing the template's (rows f1/f3/f4)."""
    topo = tm.topo
    W = topo.tp * topo.pp * topo.dp
    nodes: List[Tuple[int, int, object]] = []
    rank_nodes: List[List[int]] = []
    groups: Dict[tuple, List[Tuple[int, int]]] = {}
    dpreds: Dict[int, List[int]] = {}
    for r in range(W):
        tpi, s, dpi, epi, edpi = _coords(topo, r)
        tmpl = tm.stage(s)
        occ: Dict[object, int] = {}
        mine = []
        last_on: Dict[int, int] = {}
        last_rec: Dict[int, int] = {}
        for i, op in enumerate(tmpl):
            n = len(nodes)
            nodes.append((r, i, op))
            mine.append(n)
            # row f2: directional predecessors = previous op of the stream + event source
            ps = []
            if int(op["stream"]) in last_on:
                ps.append(last_on[int(op["stream"])])
            if int(op["ev_wait"]) and (int(op["ev_wait"]) - 1) in last_rec:
                ps.append(last_rec[int(op["ev_wait"]) - 1])
            dpreds[n] = ps
            last_on[int(op["stream"])] = n
            if int(op["ev_record"]):
                last_rec[int(op["ev_record"]) - 1] = n
            if op["kind"] == 1:
                role = int(op["role"])
                gid = {1: (s, dpi), 2: (tpi, s), 3: (tpi, s, edpi), 4: (tpi, s, epi), 5: ()}[role]
                k = occ.get(role, 0)
                occ[role] = k + 1
                groups.setdefault(("C", role, gid, k), []).append((n, _d(op, n, node_dur)))
            elif op["kind"] == 2:
                prev = _rank(topo, tpi, (s - 1) % topo.pp, dpi)
                nxt = _rank(topo, tpi, (s + 1) % topo.pp, dpi)
                for bit, (sender, d) in ((1, (r, 0)), (2, (prev, 0)), (4, (r, 1)), (8, (nxt, 1))):
                    if int(op["p2p_mask"]) & bit:
                        k = occ.get(("b", bit), 0)
                        occ[("b", bit)] = k + 1
                        groups.setdefault(("P", sender, d, k), []).append((n, _d(op, n, node_dur)))
        rank_nodes.append(mine)
    return nodes, rank_nodes, groups, dpreds


def _d(op, n, node_dur):
    return int(op["dur_ns"]) if node_dur is None else int(node_dur[n])


def _dag(tm, node_dur=None):
    """The plain vertex-weighted DAG of the module docstring: (n_nodes, weight, preds)."""
    nodes, rank_nodes, groups, dpreds = expand(tm, node_dur)
    # vertices: ("n", node) for every node; ("g", key) for groups
    weight: Dict[tuple, int] = {}
    preds: Dict[tuple, List[tuple]] = {}
    node_groups: Dict[int, List[tuple]] = {}
    for key, mem in groups.items():
        for n, _ in mem:
            node_groups.setdefault(n, []).append(key)
    for r, mine in enumerate(rank_nodes):
        for j, n in enumerate(mine):
            v = ("n", n)
            preds.setdefault(v, [])
            if n in node_groups:
                weight[v] = 0
                for key in node_groups[n]:
                    preds[v].append(("g", key))
            else:
                weight[v] = _d(nodes[n][2], n, node_dur)
                preds[v].extend(("n", p) for p in dpreds[n])
    for key, mem in groups.items():
        g = ("g", key)
        weight[g] = max(d for _, d in mem)
        preds[g] = []
        for n, _ in mem:
            preds[g].extend(("n", p) for p in dpreds[n])
    return len(nodes), weight, preds


def iteration_time(tm, node_dur=None) -> Tuple[int, List[int]]:
    """(T, finish per node) by exhaustive path enumeration."""
    n_nodes, weight, preds = _dag(tm, node_dur)
    succ: Dict[tuple, List[tuple]] = {v: [] for v in weight}
    for v, ps in preds.items():
        for p in ps:
            succ[p].append(v)
    best: Dict[tuple, int] = {v: -1 for v in weight}

    def walk(v, acc):  # enumerate every path explicitly
        acc += weight[v]
        if acc > best[v]:
            best[v] = acc
        for w in succ[v]:
            walk(w, acc)

    for v in weight:
        if not preds[v]:
            walk(v, 0)
    fin = [best[("n", n)] for n in range(n_nodes)]
    if any(f < 0 for f in fin):
        raise RuntimeError("deadlock: some node is unreachable from every source")
    return (max(fin) if fin else 0), fin


def fixed_point(tm, node_dur=None) -> Tuple[int, List[int]]:
    """(T, finish per node) by a Bellman-Ford-style fixed point on the same
    DAG: starting from f = -inf everywhere, sweep every vertex v in an arbitrary (here: reversed
    creation) order setting f(v) = weight(v) + max(0, max over preds f(p)) once all its preds are
    finite, until a sweep changes nothing (<= |V| sweeps on a DAG). Polynomial, so it runs on graphs
    far beyond path enumeration; no priority queue, no topological order."""
    n_nodes, weight, preds = _dag(tm, node_dur)
    order = list(reversed(list(weight)))
    NEG = None
    f: Dict[tuple, object] = {v: NEG for v in order}
    for _ in range(len(order) + 1):
        changed = False
        for v in order:
            ps = preds[v]
            if any(f[p] is NEG for p in ps):
                continue
            val = weight[v] + max([0] + [f[p] for p in ps])
            if f[v] is NEG or val != f[v]:
                f[v] = val
                changed = True
        if not changed:
            break
    fin = [f[("n", n)] for n in range(n_nodes)]
    if any(x is NEG for x in fin):
        raise RuntimeError("deadlock: some node never becomes ready")
    return (max(fin) if fin else 0), fin

"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic (no expansion, no matching, no replay, no
perturbation, no memory scan). It only writes per-pipeline-stage op templates in the binary
layout of ``include/prism.h``'s ``prism_op`` (48 bytes), plus a topology. Both sides consume
exactly these arrays: ``oracle/`` expands and replays them on the CPU, ``paper_2605_15617_b200``
on the GPU.

Where the shapes come from (DESIGN.md §4 states the full recipe):
  * template granularity: coarse spans between communication points (§5.1),
    "sliced per-rank templates" identical across DP replicas (§5.2);
  * pipeline schedules: Megatron-style 1F1B and interleaved 1F1B (Fig. 2 "dependencies of
    1F1B"; VPP column of the strategy table) emitted with the rules of SURVEY.md
    Appendix A;
  * configs C1-C5: BASELINE.json ``configs``; model shapes are the public model cards;
  * the integer cost model is generator-only: only integer ``dur_ns`` crosses
    into the templates.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

# ---------------------------------------------------------------------------------------------
# binary layout (mirrors include/prism.h; both sides read this layout, neither imports the other)
# ---------------------------------------------------------------------------------------------
OP_DTYPE = np.dtype(
    [
        ("kind", "u1"),
        ("coll", "u1"),
        ("role", "u1"),
        ("p2p_mask", "u1"),
        ("stream", "u1"),
        ("ev_record", "u1"),
        ("ev_wait", "u1"),
        ("pad0", "u1"),
        ("label", "<u4"),
        ("pad1", "<u4"),
        ("dur_ns", "<i8"),
        ("bytes", "<i8"),
        ("mem_alloc", "<i8"),
        ("mem_free", "<i8"),
    ]
)
assert OP_DTYPE.itemsize == 48

KIND_COMPUTE, KIND_COLLECTIVE, KIND_P2P = 0, 1, 2
COLL_AR, COLL_RS, COLL_AG, COLL_A2A, COLL_BCAST, COLL_BARRIER = range(6)
ROLE_TP, ROLE_DP, ROLE_EP, ROLE_EDP, ROLE_WORLD = 1, 2, 3, 4, 5
SEND_NEXT, RECV_PREV, SEND_PREV, RECV_NEXT = 1, 2, 4, 8
ORDER_TP_PP_DP, ORDER_MEGATRON = 0, 1

# op-type codes used in labels (label = code << 24 | layer << 12 | microbatch)
OPCODES = {
    "EMB_F": 1, "EMB_B": 2, "ATTN_F": 3, "ATTN_B": 4, "MLP_F": 5, "MLP_B": 6, "HEAD_F": 7,
    "HEAD_B": 8, "LAYER_F": 9, "LAYER_B": 10, "ATTN_ROUTER_F": 11, "ATTN_ROUTER_B": 12,
    "EXPERT_F": 13, "EXPERT_B": 14, "OPT": 15, "TP_AR": 16, "EP_A2A": 17, "DP_SYNC": 18,
    "DP_AG": 19, "EDP_SYNC": 20, "EDP_AG": 21, "P2P": 22, "SPAN": 23, "WORLD": 24,
}


def make_label(code: str, layer: int = 0, mb: int = 0) -> int:
    return (OPCODES[code] << 24) | ((layer & 0xFFF) << 12) | (mb & 0xFFF)


@dataclasses.dataclass(frozen=True)
class Topology:
    tp: int
    pp: int
    dp: int
    ep: int = 1
    vpp: int = 1
    rank_order: int = ORDER_TP_PP_DP

    @property
    def world(self) -> int:
        return self.tp * self.pp * self.dp


@dataclasses.dataclass
class Templates:
    """Per-stage templates: ops[tmpl_ptr[s]:tmpl_ptr[s+1]] is stage s's program."""

    topo: Topology
    ops: np.ndarray  # OP_DTYPE
    tmpl_ptr: np.ndarray  # int64 [pp+1]
    static_mem: np.ndarray  # int64 [pp]
    name: str = ""
    meta: Dict[str, object] = dataclasses.field(default_factory=dict)

    def stage(self, s: int) -> np.ndarray:
        return self.ops[self.tmpl_ptr[s] : self.tmpl_ptr[s + 1]]

    @property
    def n_nodes(self) -> int:
        """Node count of the expanded graph: every rank of stage s runs template s."""
        per_stage = np.diff(self.tmpl_ptr)
        return int(per_stage.sum()) * self.topo.tp * self.topo.dp


class _StageBuilder:
    def __init__(self) -> None:
        self.rows: List[tuple] = []

    def op(self, kind, dur, *, coll=0, role=0, mask=0, label=0, nbytes=0, alloc=0, free=0, stream=0,
           record=None, wait=None):
        """record / wait: event slot (0..7) recorded at the op's finish / waited for before its start
        (row f2: multi-stream ranks, CUDA-event semantics)."""
        self.rows.append((kind, coll, role, mask, stream, 0 if record is None else record + 1,
                          0 if wait is None else wait + 1, 0, label, 0, int(dur), int(nbytes), int(alloc),
                          int(free)))

    def compute(self, dur, label=0, alloc=0, free=0, **kw):
        self.op(KIND_COMPUTE, dur, label=label, alloc=alloc, free=free, **kw)

    def coll(self, role, coll, dur, label=0, nbytes=0, alloc=0, free=0, **kw):
        self.op(KIND_COLLECTIVE, dur, coll=coll, role=role, label=label, nbytes=nbytes,
                alloc=alloc, free=free, **kw)

    def p2p(self, mask, dur, label=0, nbytes=0, **kw):
        if mask:
            self.op(KIND_P2P, dur, mask=mask, label=label, nbytes=nbytes, **kw)

    def array(self) -> np.ndarray:
        return np.array(self.rows, dtype=OP_DTYPE)


def assemble(topo: Topology, stages: Sequence[np.ndarray], static_mem: Sequence[int],
             name: str = "", meta: Optional[dict] = None) -> Templates:
    assert len(stages) == topo.pp
    ptr = np.zeros(topo.pp + 1, dtype=np.int64)
    ptr[1:] = np.cumsum([len(s) for s in stages])
    ops = np.concatenate(stages) if len(stages) else np.zeros(0, OP_DTYPE)
    return Templates(topo, ops.astype(OP_DTYPE), ptr, np.asarray(static_mem, dtype=np.int64),
                     name, dict(meta or {}))


# ---------------------------------------------------------------------------------------------
# pipeline schedules (Megatron-style). Items:
#   ("F", mb, chunk)  ("B", mb, chunk)  ("P", mask)
# ---------------------------------------------------------------------------------------------
def schedule_1f1b(p: int, s: int, m: int) -> List[tuple]:
    out: List[tuple] = []
    w = min(p - s - 1, m)
    r = m - w
    fi = bi = 0
    for _ in range(w):
        if s > 0:
            out.append(("P", RECV_PREV))
        out.append(("F", fi, 0)); fi += 1
        if s < p - 1:
            out.append(("P", SEND_NEXT))
    if r > 0 and s > 0:
        out.append(("P", RECV_PREV))
    for i in range(r):
        out.append(("F", fi, 0)); fi += 1
        if s < p - 1:
            out.append(("P", SEND_NEXT | RECV_NEXT))
        out.append(("B", bi, 0)); bi += 1
        if s > 0:
            out.append(("P", SEND_PREV | (RECV_PREV if i < r - 1 else 0)))
    for _ in range(w):
        if s < p - 1:
            out.append(("P", RECV_NEXT))
        out.append(("B", bi, 0)); bi += 1
        if s > 0:
            out.append(("P", SEND_PREV))
    assert fi == m and bi == m
    return out


def schedule_interleaved(p: int, s: int, m: int, v: int) -> List[tuple]:
    if v < 2:
        return schedule_1f1b(p, s, m)
    if m % p != 0:
        raise ValueError("interleaved schedule needs m % pp == 0 (reading Z14)")
    if m < p:
        raise ValueError("GaTooSmall: interleaved schedule needs m >= pp (SPEC S:156)")
    total = m * v

    def chunk(k: int, fwd: bool) -> int:
        c = (k % (p * v)) // p  # Python % is floor modulo (Appendix A note)
        return c if fwd else v - 1 - c

    def mb_of(k: int) -> int:
        return (k // (p * v)) * p + (k % p)

    nw = min((p - s - 1) * 2 + (v - 1) * p, total)
    nr = total - nw
    out: List[tuple] = []
    if s != 0:
        out.append(("P", RECV_PREV))
    for k in range(nw):
        out.append(("F", mb_of(k), chunk(k, True)))
        recv_prev = not (s == 0 and chunk(k + 1, True) == 0) and k != total - 1
        send = not (s == p - 1 and chunk(k, True) == v - 1)
        mask = (SEND_NEXT if send else 0) | (RECV_PREV if recv_prev else 0)
        if k == nw - 1 and nr > 0:
            if not (s == p - 1 and chunk(0, False) == v - 1):
                mask |= RECV_NEXT
        out.append(("P", mask))
    for k in range(nr):
        fk = k + nw
        out.append(("F", mb_of(fk), chunk(fk, True)))
        out.append(("B", mb_of(k), chunk(k, False)))
        recv_prev = not (s == 0 and chunk(fk - (p - 1), True) == v - 1) and k != nr - 1
        recv_next = not (s == p - 1 and chunk(k - (p - 1), False) == 0)
        mask = 0
        if not (s == p - 1 and chunk(fk, True) == v - 1):
            mask |= SEND_NEXT
        if recv_prev:
            mask |= RECV_PREV
        if not (s == 0 and chunk(k, False) == 0):
            mask |= SEND_PREV
        if recv_next:
            mask |= RECV_NEXT
        out.append(("P", mask))
    if nr == 0 and s != p - 1:
        out.append(("P", RECV_NEXT))
    for k in range(nr, total):
        out.append(("B", mb_of(k), chunk(k, False)))
        mask = 0
        if not (s == 0 and chunk(k, False) == 0):
            mask |= SEND_PREV
        if not (s == p - 1 and chunk(k + 1, False) == v - 1) and k != total - 1:
            mask |= RECV_NEXT
        out.append(("P", mask))
    return [it for it in out if not (it[0] == "P" and it[1] == 0)]


# ---------------------------------------------------------------------------------------------
# integer cost model (generator-only)
# ---------------------------------------------------------------------------------------------
FLOPS_PER_NS = 445_050  # 989e12 FLOP/s x 0.45 MFU = 4.4505e14 FLOP/s (H100-class target, P:1546 unnamed)
NODE_GPUS = 8           # GPUs per node
ALPHA_INTRA, BETA_INTRA = 5_000, 400_000   # ns, MB/s
ALPHA_INTER, BETA_INTER = 15_000, 50_000


def cdiv(a: int, b: int) -> int:
    return -(-a // b)


def compute_ns(flops: int) -> int:
    return max(1, cdiv(int(flops), FLOPS_PER_NS))


def _tier(ranks: Sequence[int]) -> Tuple[int, int]:
    nodes = {r // NODE_GPUS for r in ranks}
    return (ALPHA_INTRA, BETA_INTRA) if len(nodes) <= 1 else (ALPHA_INTER, BETA_INTER)


def _step(alpha: int, beta: int, nbytes: int) -> int:
    return alpha + cdiv(nbytes * 1000, beta)


def coll_ns(coll: int, n: int, nbytes: int, ranks: Sequence[int]) -> int:
    """Ring cost: AR = 2(n-1) steps of ceil(B/n) bytes ((K-1) reduce + (K-1)
    broadcast rounds); RS/AG/A2A = (n-1) steps."""
    if n <= 1:
        return 0
    a, b = _tier(ranks)
    st = _step(a, b, cdiv(nbytes, n))
    return (2 * (n - 1) if coll == COLL_AR else (n - 1)) * st


def p2p_ns(nbytes: int, ranks: Sequence[int]) -> int:
    a, b = _tier(ranks)
    return _step(a, b, nbytes)


def coords_to_rank(topo: Topology, tp_i: int, pp_i: int, dp_i: int) -> int:
    if topo.rank_order == ORDER_MEGATRON:
        return tp_i + topo.tp * (dp_i + topo.dp * pp_i)
    return tp_i + topo.tp * (pp_i + topo.pp * dp_i)


def _role_ranks(topo: Topology, role: int, s: int) -> List[int]:
    """Members of the role's group that contains coordinates (tp 0, stage s, dp 0): the
    representative used to pick a bandwidth tier for the stage's template op."""
    if role == ROLE_TP:
        return [coords_to_rank(topo, t, s, 0) for t in range(topo.tp)]
    if role == ROLE_DP:
        return [coords_to_rank(topo, 0, s, d) for d in range(topo.dp)]
    if role == ROLE_EP:
        return [coords_to_rank(topo, 0, s, e) for e in range(topo.ep)]
    if role == ROLE_EDP:
        return [coords_to_rank(topo, 0, s, e * topo.ep) for e in range(topo.dp // topo.ep)]
    return list(range(topo.world))


# ---------------------------------------------------------------------------------------------
# model description -> per-stage templates
# ---------------------------------------------------------------------------------------------
@dataclasses.dataclass
class ModelShape:
    name: str
    layers: int
    hidden: int
    ffn: int
    heads: int
    kv_heads: int
    seq: int
    vocab: int
    swiglu: bool = True
    # MoE
    moe_first_dense: int = -1  # -1: dense model; else layers >= this index are MoE
    experts: int = 0
    topk: int = 0
    expert_ffn: int = 0
    shared_experts: int = 0


LLAMA3_70B = ModelShape("llama3-70b", 80, 8192, 28672, 64, 8, 8192, 128256)
GPT3_175B = ModelShape("gpt3-175b", 96, 12288, 49152, 96, 96, 2048, 50257, swiglu=False)
DSV3 = ModelShape("deepseek-v3-shaped", 61, 7168, 18432, 128, 128, 4096, 129280,
                  moe_first_dense=3, experts=256, topk=8, expert_ffn=2048, shared_experts=1)
LLAMA3_405B = ModelShape("llama3-405b-shaped", 126, 16384, 53248, 128, 8, 8192, 128256)


@dataclasses.dataclass
class TrainSetup:
    model: ModelShape
    topo: Topology
    microbatches: int
    layers_per_stage: Sequence[int]
    zero1: bool = False
    bucket_params: int = 40_000_000
    embed_and_head: bool = True


def _attn_params(m: ModelShape) -> int:
    kvdim = m.hidden * m.kv_heads // m.heads
    return 2 * m.hidden * m.hidden + 2 * m.hidden * kvdim


def _mlp_params(m: ModelShape, ffn: int) -> int:
    return (3 if m.swiglu else 2) * m.hidden * ffn


def _attn_flops(m: ModelShape) -> int:
    s, h = m.seq, m.hidden
    kvdim = h * m.kv_heads // m.heads
    return 2 * s * h * (h + 2 * kvdim) + 2 * s * h * h + 4 * s * s * h


def _mlp_flops(m: ModelShape, ffn: int, tokens: int) -> int:
    return 2 * tokens * (3 if m.swiglu else 2) * m.hidden * ffn


def build_training_templates(st: TrainSetup, name: str = "") -> Templates:
    """Per-stage templates for Megatron-style training (SURVEY.md §8.3 granularity table)."""
    m, topo = st.model, st.topo
    p, v, tp, dp = topo.pp, max(1, topo.vpp), topo.tp, topo.dp
    assert len(st.layers_per_stage) == p
    lps = list(st.layers_per_stage)
    # global layer index of (stage s, chunk c, local layer j)
    per_chunk = [[0] * v for _ in range(p)]
    for s in range(p):
        assert lps[s] % v == 0
        for c in range(v):
            per_chunk[s][c] = lps[s] // v
    order = [(c, s) for c in range(v) for s in range(p)]
    first_layer: Dict[Tuple[int, int], int] = {}
    acc = 0
    for c, s in order:
        first_layer[(s, c)] = acc
        acc += per_chunk[s][c]
    assert acc == m.layers, (acc, m.layers)

    s_tok, h = m.seq, m.hidden
    act_bytes = 2 * s_tok * h  # one bf16 activation
    stages, static = [], []
    for s in range(p):
        b = _StageBuilder()
        tp_ranks = _role_ranks(topo, ROLE_TP, s)
        ep_ranks = _role_ranks(topo, ROLE_EP, s)

        def tp_ar(label_code, layer, mb):
            if tp > 1:
                b.coll(ROLE_TP, COLL_AR, coll_ns(COLL_AR, tp, act_bytes, tp_ranks),
                       label=make_label("TP_AR", layer, mb), nbytes=act_bytes, alloc=act_bytes,
                       free=act_bytes)

        def ep_a2a(layer, mb):
            nb = act_bytes * m.topk
            if topo.ep > 1:
                b.coll(ROLE_EP, COLL_A2A, coll_ns(COLL_A2A, topo.ep, nb, ep_ranks),
                       label=make_label("EP_A2A", layer, mb), nbytes=nb, alloc=nb, free=nb)

        def layer_ops(layer: int, mb: int, fwd: bool):
            moe = m.moe_first_dense >= 0 and layer >= m.moe_first_dense
            mul = 1 if fwd else 2
            if moe:
                # MoE, TP=1: ATTN_ROUTER, A2A, EXPERT, A2A
                attn = compute_ns(mul * (_attn_flops(m) // tp + 2 * s_tok * h * m.experts))
                toks = s_tok * m.topk
                exp = compute_ns(mul * (_mlp_flops(m, m.expert_ffn, toks) +
                                        _mlp_flops(m, m.expert_ffn, s_tok) * m.shared_experts) // tp)
                a_attn = (act_bytes * 5) // tp
                a_exp = 2 * toks * (h + 2 * m.expert_ffn) // tp
                if fwd:
                    b.compute(attn, make_label("ATTN_ROUTER_F", layer, mb), alloc=a_attn)
                    ep_a2a(layer, mb)
                    b.compute(exp, make_label("EXPERT_F", layer, mb), alloc=a_exp)
                    ep_a2a(layer, mb)
                else:
                    ep_a2a(layer, mb)
                    b.compute(exp, make_label("EXPERT_B", layer, mb), free=a_exp)
                    ep_a2a(layer, mb)
                    b.compute(attn, make_label("ATTN_ROUTER_B", layer, mb), free=a_attn)
                return
            attn = compute_ns(mul * _attn_flops(m) // tp)
            mlp = compute_ns(mul * _mlp_flops(m, m.ffn, s_tok) // tp)
            a_attn = (act_bytes * 5) // tp + act_bytes
            a_mlp = (2 * s_tok * m.ffn * 3) // tp + act_bytes
            if tp == 1:
                if fwd:
                    b.compute(attn + mlp, make_label("LAYER_F", layer, mb), alloc=a_attn + a_mlp)
                else:
                    b.compute(attn + mlp, make_label("LAYER_B", layer, mb), free=a_attn + a_mlp)
                return
            if fwd:
                b.compute(attn, make_label("ATTN_F", layer, mb), alloc=a_attn)
                tp_ar("TP_AR", layer, mb)
                b.compute(mlp, make_label("MLP_F", layer, mb), alloc=a_mlp)
                tp_ar("TP_AR", layer, mb)
            else:
                b.compute(mlp, make_label("MLP_B", layer, mb), free=a_mlp)
                tp_ar("TP_AR", layer, mb)
                b.compute(attn, make_label("ATTN_B", layer, mb), free=a_attn)
                tp_ar("TP_AR", layer, mb)

        emb_ns = compute_ns(2 * s_tok * h)
        head_ns = compute_ns(2 * s_tok * h * m.vocab // tp)
        a_head = 2 * s_tok * m.vocab * 2 // tp

        def fwd(mb: int, c: int):
            if st.embed_and_head and s == 0 and c == 0:
                b.compute(emb_ns, make_label("EMB_F", 0, mb), alloc=act_bytes)
                tp_ar("TP_AR", 0, mb)
            f0 = first_layer[(s, c)]
            for j in range(per_chunk[s][c]):
                layer_ops(f0 + j, mb, True)
            if st.embed_and_head and s == p - 1 and c == v - 1:
                b.compute(head_ns, make_label("HEAD_F", m.layers, mb), alloc=a_head)
                tp_ar("TP_AR", m.layers, mb)

        def bwd(mb: int, c: int):
            if st.embed_and_head and s == p - 1 and c == v - 1:
                b.compute(2 * head_ns, make_label("HEAD_B", m.layers, mb), free=a_head)
                tp_ar("TP_AR", m.layers, mb)
            f0 = first_layer[(s, c)]
            for j in reversed(range(per_chunk[s][c])):
                layer_ops(f0 + j, mb, False)
            if st.embed_and_head and s == 0 and c == 0:
                b.compute(2 * emb_ns, make_label("EMB_B", 0, mb), free=act_bytes)
                tp_ar("TP_AR", 0, mb)

        prev_r = coords_to_rank(topo, 0, (s - 1) % p, 0)
        next_r = coords_to_rank(topo, 0, (s + 1) % p, 0)
        me = coords_to_rank(topo, 0, s, 0)
        p2p_cost = max(p2p_ns(act_bytes, [me, prev_r]), p2p_ns(act_bytes, [me, next_r]))
        sched = (schedule_interleaved(p, s, st.microbatches, v) if v > 1
                 else schedule_1f1b(p, s, st.microbatches))
        for item in sched:
            if item[0] == "F":
                fwd(item[1], item[2])
            elif item[0] == "B":
                bwd(item[1], item[2])
            else:
                b.p2p(item[1], p2p_cost, make_label("P2P"), nbytes=act_bytes)

        # parameters on this rank
        dense_layers = moe_layers = 0
        for c in range(v):
            for j in range(per_chunk[s][c]):
                L = first_layer[(s, c)] + j
                if m.moe_first_dense >= 0 and L >= m.moe_first_dense:
                    moe_layers += 1
                else:
                    dense_layers += 1
        dense_params = dense_layers * (_attn_params(m) + _mlp_params(m, m.ffn)) // tp
        dense_params += moe_layers * (_attn_params(m) + h * m.experts) // tp
        expert_params = moe_layers * (m.experts // max(1, topo.ep)) * _mlp_params(m, m.expert_ffn)
        if st.embed_and_head and s == 0:
            dense_params += m.vocab * h // tp
        if st.embed_and_head and s == p - 1:
            dense_params += m.vocab * h // tp

        dp_ranks = _role_ranks(topo, ROLE_DP, s)
        edp = dp // topo.ep
        edp_ranks = _role_ranks(topo, ROLE_EDP, s)

        def buckets(n_params: int) -> List[int]:
            nb = cdiv(n_params, st.bucket_params) if n_params > 0 else 0
            return [min(st.bucket_params, n_params - i * st.bucket_params) for i in range(nb)]

        sync_coll = COLL_RS if st.zero1 else COLL_AR
        for i, bp in enumerate(buckets(dense_params)):
            nb = 2 * bp
            if dp > 1:
                b.coll(ROLE_DP, sync_coll, coll_ns(sync_coll, dp, nb, dp_ranks),
                       label=make_label("DP_SYNC", i), nbytes=nb, alloc=nb, free=nb)
        for i, bp in enumerate(buckets(expert_params)):
            nb = 2 * bp
            if edp > 1:
                b.coll(ROLE_EDP, sync_coll, coll_ns(sync_coll, edp, nb, edp_ranks),
                       label=make_label("EDP_SYNC", i), nbytes=nb, alloc=nb, free=nb)
        opt_params = (dense_params // dp + expert_params // edp) if st.zero1 else (dense_params + expert_params)
        b.compute(max(1, cdiv(opt_params * 16, 3000)), make_label("OPT"))
        if st.zero1:
            for i, bp in enumerate(buckets(dense_params)):
                nb = 2 * bp
                if dp > 1:
                    b.coll(ROLE_DP, COLL_AG, coll_ns(COLL_AG, dp, nb, dp_ranks),
                           label=make_label("DP_AG", i), nbytes=nb, alloc=nb, free=nb)
            for i, bp in enumerate(buckets(expert_params)):
                nb = 2 * bp
                if edp > 1:
                    b.coll(ROLE_EDP, COLL_AG, coll_ns(COLL_AG, edp, nb, edp_ranks),
                           label=make_label("EDP_AG", i), nbytes=nb, alloc=nb, free=nb)
        n_par = dense_params + expert_params
        if st.zero1:
            static_b = 6 * n_par + (12 * dense_params) // dp + (12 * expert_params) // max(1, edp)
        else:
            static_b = 18 * n_par
        stages.append(b.array())
        static.append(static_b)
    return assemble(topo, stages, static, name or m.name,
                    {"microbatches": st.microbatches, "model": m.name})


# ---------------------------------------------------------------------------------------------
# uniform-cost pipelines (closed-form checks) and the BASELINE.json configs
# ---------------------------------------------------------------------------------------------
def uniform_pipeline(tp: int, pp: int, dp: int, m: int, *, vpp: int = 1, layers_per_chunk: int = 1,
                     f_ns: int = 1000, b_ns: int = 2000, tp_ar_ns: int = 100, p2p_c: int = 0,
                     dp_ar_ns: int = 300, opt_ns: int = 500, act_bytes: int = 1 << 20,
                     static_bytes: int = 1 << 30, dense_tp_layout: bool = True) -> Templates:
    """Every forward compute node f_ns, backward b_ns, TP AR tp_ar_ns, P2P message p2p_c, one DP AR
    dp_ar_ns then OPT opt_ns; each forward compute node allocates act_bytes freed by its
    backward; no transient buffers (C1 of BASELINE.json with 2 layers/stage)."""
    topo = Topology(tp, pp, dp, 1, vpp)
    stages, static = [], []
    for s in range(pp):
        b = _StageBuilder()

        def fwd(mb, c):
            for j in range(layers_per_chunk):
                L = (c * pp + s) * layers_per_chunk + j
                if tp > 1 and dense_tp_layout:
                    b.compute(f_ns, make_label("ATTN_F", L, mb), alloc=act_bytes)
                    b.coll(ROLE_TP, COLL_AR, tp_ar_ns, label=make_label("TP_AR", L, mb))
                    b.compute(f_ns, make_label("MLP_F", L, mb), alloc=act_bytes)
                    b.coll(ROLE_TP, COLL_AR, tp_ar_ns, label=make_label("TP_AR", L, mb))
                else:
                    b.compute(f_ns, make_label("LAYER_F", L, mb), alloc=act_bytes)

        def bwd(mb, c):
            for j in reversed(range(layers_per_chunk)):
                L = (c * pp + s) * layers_per_chunk + j
                if tp > 1 and dense_tp_layout:
                    b.compute(b_ns, make_label("MLP_B", L, mb), free=act_bytes)
                    b.coll(ROLE_TP, COLL_AR, tp_ar_ns, label=make_label("TP_AR", L, mb))
                    b.compute(b_ns, make_label("ATTN_B", L, mb), free=act_bytes)
                    b.coll(ROLE_TP, COLL_AR, tp_ar_ns, label=make_label("TP_AR", L, mb))
                else:
                    b.compute(b_ns, make_label("LAYER_B", L, mb), free=act_bytes)

        sched = schedule_interleaved(pp, s, m, vpp) if vpp > 1 else schedule_1f1b(pp, s, m)
        for it in sched:
            if it[0] == "F":
                fwd(it[1], it[2])
            elif it[0] == "B":
                bwd(it[1], it[2])
            else:
                b.p2p(it[1], p2p_c, make_label("P2P"))
        if dp > 1 and dp_ar_ns >= 0:
            b.coll(ROLE_DP, COLL_AR, dp_ar_ns, label=make_label("DP_SYNC"))
        if opt_ns >= 0:
            b.compute(opt_ns, make_label("OPT"))
        stages.append(b.array())
        static.append(static_bytes)
    return assemble(topo, stages, static, f"uniform_tp{tp}_pp{pp}_dp{dp}_m{m}_v{vpp}",
                    {"microbatches": m})


def config(name: str, **kw) -> Templates:
    """BASELINE.json configs (shapes in SURVEY.md §8.3 / DESIGN.md §4)."""
    name = name.upper()
    if name == "C1":
        return uniform_pipeline(2, 2, 2, 4, layers_per_chunk=2, p2p_c=kw.get("p2p_c", 0))
    if name == "C2":
        topo = Topology(8, 8, 16)
        return build_training_templates(TrainSetup(LLAMA3_70B, topo, 32, [10] * 8), "C2")
    if name == "C3":
        topo = Topology(8, 16, 32, 1, 2)
        return build_training_templates(TrainSetup(GPT3_175B, topo, 48, [6] * 16, zero1=True), "C3")
    if name == "C4":
        topo = Topology(1, 16, 128, 64)
        lps = [4] * 13 + [3] * 3
        return build_training_templates(TrainSetup(DSV3, topo, 32, lps, zero1=True), "C4")
    if name == "C5":
        topo = Topology(8, 16, 64)
        lps = [7] + [8] * 14 + [7]
        return build_training_templates(TrainSetup(LLAMA3_405B, topo, 32, lps), "C5")
    raise KeyError(name)


CONFIG_DESCRIPTIONS = {
    "C1": "8 ranks TP2 PP2 DP2, 4-layer GPT, m=4 1F1B, uniform op costs",
    "C2": "Llama-3-70B, 1024 ranks TP8 PP8 DP16, 1F1B m=32",
    "C3": "GPT-3-175B, 4096 ranks TP8 PP16 DP32, interleaved 1F1B v=2 m=48, ZeRO-1 RS/AG",
    "C4": "DeepSeek-V3-shaped MoE, 2048 ranks TP1 PP16 DP128 EP64, 1F1B m=32, ZeRO-1",
    "C5": "Llama-3-405B-shaped, 8192 ranks TP8 PP16 DP64, 1F1B m=32, 64 perturbed scenarios",
}


def scaled(name: str, shrink: int = 8) -> Templates:
    """A smaller graph with the same structure as a BASELINE config (fewer DP replicas and
    microbatches) for parity tests the oracle finishes in seconds."""
    name = name.upper()
    if name == "C2":
        return build_training_templates(TrainSetup(LLAMA3_70B, Topology(8, 8, 2), 8, [10] * 8), "C2s")
    if name == "C3":
        return build_training_templates(
            TrainSetup(GPT3_175B, Topology(8, 16, 2, 1, 2), 16, [6] * 16, zero1=True), "C3s")
    if name == "C4":
        return build_training_templates(
            TrainSetup(DSV3, Topology(1, 16, 8, 4), 8, [4] * 13 + [3] * 3, zero1=True), "C4s")
    if name == "C5":
        return build_training_templates(
            TrainSetup(LLAMA3_405B, Topology(8, 16, 2), 8, [7] + [8] * 14 + [7]), "C5s")
    raise KeyError(name)


# ---------------------------------------------------------------------------------------------
# random template fuzz (acyclic by construction)
# ---------------------------------------------------------------------------------------------
def random_templates(seed: int, max_world: int = 64, max_ops: int = 40,
                     max_dur: int = 1000, p_span0: float = 0.05, streams: int = 1) -> Templates:
    """Random topology and per-stage templates whose sync structure is acyclic by construction:
    stage-spanning sync events (P2P messages between ring neighbours, WORLD collectives) are drawn
    from ONE global sequence that every stage follows in the same order; intra-stage collectives
    (TP/DP/EP/EDP: all members run the same template) and compute spans are inserted at random
    positions. Consecutive messages of one stage with distinct mask bits may be batched into one
    P2P node. Durations include zeros; memory deltas keep every running total >= 0."""
    rng = np.random.default_rng(seed)
    while True:
        tp = int(rng.choice([1, 1, 2, 3, 4]))
        pp = int(rng.integers(1, 5))
        dp = int(rng.choice([1, 2, 3, 4]))
        if tp * pp * dp <= max_world:
            break
    divs = [e for e in range(1, dp + 1) if dp % e == 0]
    ep = int(rng.choice(divs))
    order = int(rng.integers(0, 2))
    topo = Topology(tp, pp, dp, ep, 1, order)

    def dur():
        return 0 if rng.random() < p_span0 else int(rng.integers(1, max_dur + 1))

    # global event list
    n_events = int(rng.integers(0, max_ops // 2 + 1))
    events: List[tuple] = []
    for _ in range(n_events):
        if pp > 1 and rng.random() < 0.8:
            s = int(rng.integers(0, pp))
            if rng.random() < 0.5:
                events.append(("msg", s, (s + 1) % pp, "next"))
            else:
                events.append(("msg", s, (s - 1) % pp, "prev"))
        else:
            events.append(("world", int(rng.integers(0, 6))))
    per_stage: List[List[tuple]] = [[] for _ in range(pp)]
    for ev in events:
        if ev[0] == "msg":
            _, src, dst, d = ev
            if d == "next":
                per_stage[src].append(("p2p", SEND_NEXT))
                per_stage[dst].append(("p2p", RECV_PREV))
            else:
                per_stage[src].append(("p2p", SEND_PREV))
                per_stage[dst].append(("p2p", RECV_NEXT))
        else:
            for s in range(pp):
                per_stage[s].append(("world", ev[1]))
    stages, static = [], []
    for s in range(pp):
        b = _StageBuilder()
        live: List[int] = []
        seq = per_stage[s]
        i = 0
        roles = [ROLE_TP, ROLE_DP, ROLE_EP, ROLE_EDP]
        while i < len(seq) or rng.random() < 0.5:
            # local ops before the next global event
            for _ in range(int(rng.integers(0, 3))):
                r = rng.random()
                if r < 0.6:
                    alloc = int(rng.integers(0, 1000)) if rng.random() < 0.5 else 0
                    free = 0
                    if live and rng.random() < 0.5:
                        free = live.pop(int(rng.integers(0, len(live))))
                    if alloc:
                        live.append(alloc)
                    b.compute(dur(), label=int(rng.integers(0, 8)), alloc=alloc, free=free)
                else:
                    role = int(rng.choice(roles))
                    t = int(rng.integers(0, 6))
                    b.coll(role, t, dur(), label=100 + role, nbytes=int(rng.integers(0, 1 << 20)),
                           alloc=int(rng.integers(0, 50)) * 0, free=0)
            if i >= len(seq):
                if len(b.rows) > max_ops:
                    break
                continue
            ev = seq[i]
            i += 1
            if ev[0] == "world":
                b.coll(ROLE_WORLD, ev[1], dur(), label=200)
            else:
                mask = ev[1]
                # batch following messages with distinct bits
                while i < len(seq) and seq[i][0] == "p2p" and not (seq[i][1] & mask) and rng.random() < 0.5:
                    mask |= seq[i][1]
                    i += 1
                b.p2p(mask, dur(), label=300)
            if len(b.rows) > 4 * max_ops:
                # keep going: events must all be emitted
                pass
        for a in live:
            if rng.random() < 0.7:
                b.compute(dur(), label=7, free=a)
        arr = b.array()
        if streams > 1:  # row f2: random streams and CUDA-event record / wait pairs
            srng = np.random.default_rng(seed * 7919 + s)
            arr["stream"] = srng.integers(0, streams, len(arr))
            rec = srng.random(len(arr)) < 0.3
            arr["ev_record"] = np.where(rec, srng.integers(1, 5, len(arr)), 0)
            wt = srng.random(len(arr)) < 0.3
            arr["ev_wait"] = np.where(wt, srng.integers(1, 5, len(arr)), 0)
            # program-order memory deltas are not time-consistent across streams
            arr["mem_alloc"] = 0
            arr["mem_free"] = 0
        stages.append(arr)
        static.append(int(rng.integers(0, 1 << 20)))
    return assemble(topo, stages, static, f"random{seed}" + (f"_s{streams}" if streams > 1 else ""),
                    {"seed": seed})


def overlap_grad_reduce(tm: Templates, comm_stream: int = 1) -> Templates:
    """Row f2 input (P:699 overlapped gradient communication; Megatron overlap_grad_reduce): the DP
    / EDP gradient buckets that follow a stage's last backward move onto a side stream. Bucket j is
    issued right after the backward compute span of the last microbatch that completes it (the
    last microbatch's backward spans are split evenly over the buckets, in order), waits for that
    span (event slot j mod 4), and the optimizer step waits for the last bucket (slot 7). Every
    other op keeps stream 0 and its place."""
    t = tm.topo
    stages = []
    for s in range(t.pp):
        T = tm.stage(s).copy()
        code = (T["label"].astype(np.int64) >> 24)
        is_bucket = (T["kind"] == KIND_COLLECTIVE) & np.isin(T["role"], [ROLE_DP, ROLE_EDP]) & \
            np.isin(code, [OPCODES["DP_SYNC"], OPCODES["EDP_SYNC"]])
        bidx = np.nonzero(is_bucket)[0]
        opt = np.nonzero(code == OPCODES["OPT"])[0]
        if len(bidx) == 0 or len(opt) == 0:
            stages.append(T)
            continue
        first_b = int(bidx[0])
        # the last microbatch's backward compute spans (after the last P2P before the buckets)
        p2p_before = np.nonzero(T["kind"][:first_b] == KIND_P2P)[0]
        seg0 = int(p2p_before[-1]) + 1 if len(p2p_before) else 0
        bwd = [i for i in range(seg0, first_b) if T["kind"][i] == KIND_COMPUTE]
        if not bwd:
            stages.append(T)
            continue
        nb = len(bidx)
        anchor = {}  # backward span index -> buckets issued after it
        for j in range(nb):
            a = bwd[min(len(bwd) - 1, ((j + 1) * len(bwd)) // nb - 1)]
            anchor.setdefault(a, []).append(j)
        rows = []
        for i in range(len(T)):
            if is_bucket[i]:
                continue
            r = T[i].copy()
            if i == int(opt[0]):
                r["ev_wait"] = 8  # slot 7: the last bucket
            if i in anchor:
                r["ev_record"] = (anchor[i][0] % 4) + 1
            rows.append(r)
            for j in anchor.get(i, []):
                b = T[int(bidx[j])].copy()
                b["stream"] = comm_stream
                b["ev_wait"] = (anchor[i][0] % 4) + 1
                b["ev_record"] = 8 if j == nb - 1 else 0
                rows.append(b)
        stages.append(np.array(rows, dtype=OP_DTYPE))
    return assemble(t, stages, list(tm.static_mem), (tm.name or "") + "_overlap", dict(tm.meta or {}))

"""MoE mock-router inputs (row f4; Appendix F "MoE Mock Router", and the
imbalance statistics of Fig. 3's caption): a balance-ratio (br) schedule per gating event
and EP rank with the given pooled statistics, its Q16 encoding, and which template op belongs to
which gating event. An INPUT generator (seeded, host-only): it holds none of the method's
arithmetic — how br scales a rank's work and buffers is implemented independently by the CUDA path
(prism_set_moe_load) and the oracle (oracle.moe_load), which both consume these arrays.

Readings (R6-R8): br of (event, rank) = tokens the rank's experts process / the
uniform share (Appendix F); one gating event per (MoE layer, microbatch); an EP rank's expert
compute, its all-to-all payload (hence its member duration; the group lasts the max, Z2) and its
expert activations scale with br; statistics are pooled over events x ranks (SPEC S:603 notes that
Fig. 3's br_avg = 1.48 > 1 rules out per-event normalisation); the generative procedure (the
paper gives the statistics, not the procedure) is a monotone quantile function pinned at min /
median / max whose interior knots are fitted to (avg, std, skew), sampled at stratified
quantiles and permuted by the seed."""
from __future__ import annotations

import dataclasses
import math

import numpy as np


@dataclasses.dataclass(frozen=True)
class BrProfile:
    br_min: float
    br_max: float
    br_avg: float
    br_std: float
    br_med: float
    br_skew: float


FIG3_PROFILE = BrProfile(0.71, 2.16, 1.48, 0.37, 1.38, 0.90)
UNIFORM = BrProfile(1.0, 1.0, 1.0, 0.0, 1.0, 0.0)


class InfeasibleProfile(ValueError):
    pass


def stats(x) -> BrProfile:
    """Pooled min / max / mean / population std / median / Fisher skewness."""
    x = np.asarray(x, dtype=np.float64).ravel()
    mu, sd = float(x.mean()), float(x.std())
    sk = float(((x - mu) ** 3).mean() / sd ** 3) if sd > 0 else 0.0
    return BrProfile(float(x.min()), float(x.max()), mu, sd, float(np.median(x)), sk)


def within(p: BrProfile, q: BrProfile) -> bool:
    """SPEC S:552 tolerances: avg/std/med +-5 % relative, min/max +-0.05, skew +-0.15."""
    rel = lambda a, b: abs(a - b) <= 0.05 * abs(b) + 1e-12
    return (rel(p.br_avg, q.br_avg) and rel(p.br_std, q.br_std) and rel(p.br_med, q.br_med)
            and abs(p.br_min - q.br_min) <= 0.05 and abs(p.br_max - q.br_max) <= 0.05
            and abs(p.br_skew - q.br_skew) <= 0.15)


_U_LO = np.array([0.05, 0.2, 0.35])              # interior knots below the median
_U_HI = np.array([0.6, 0.7, 0.8, 0.88, 0.94, 0.98])  # ... and above (the right tail carries the skew)


def _quantile_samples(p: BrProfile, n: int, free: np.ndarray) -> np.ndarray:
    """n stratified samples of a monotone piecewise-linear quantile function with Q(0) = min,
    Q(1/2) = med, Q(1) = max and interior knots _U_LO / _U_HI (softplus increments keep it
    monotone)."""
    k1 = len(_U_LO)
    sp = np.logaddexp(0.0, free) + 1e-9
    lo = np.cumsum(sp[: k1 + 1])[:-1] / np.sum(sp[: k1 + 1])
    hi = np.cumsum(sp[k1 + 1:])[:-1] / np.sum(sp[k1 + 1:])
    u_k = np.concatenate([[0.0], _U_LO, [0.5], _U_HI, [1.0]])
    q_k = np.concatenate([[p.br_min], p.br_min + lo * (p.br_med - p.br_min), [p.br_med],
                          p.br_med + hi * (p.br_max - p.br_med), [p.br_max]])
    u = (np.arange(n) + 0.5) / n
    x = np.interp(u, u_k, q_k)
    x[0], x[-1] = p.br_min, p.br_max  # the profile states the extremes: pin them
    return x


def derive_schedule(p: BrProfile, events: int, ranks: int, seed: int = 0) -> np.ndarray:
    """A [events, ranks] br schedule whose pooled stats match p within the SPEC tolerances: the
    stratified samples of a quantile function pinned at (min, med, max) whose interior knots are
    fitted to (avg, std, skew) (reading R8), randomly permuted by the seed."""
    if events * ranks < 8:
        raise InfeasibleProfile("need at least 8 samples")
    if not (p.br_min <= p.br_med <= p.br_max and p.br_min <= p.br_avg <= p.br_max and p.br_std >= 0):
        raise InfeasibleProfile("order statistics out of order")
    if p.br_std > 0.5 * (p.br_max - p.br_min) + 1e-12:
        raise InfeasibleProfile("std too large for [min, max]")
    n = events * ranks
    if p.br_max == p.br_min:
        return np.full((events, ranks), p.br_avg)
    from scipy.optimize import minimize

    def loss(fr):
        st = stats(_quantile_samples(p, n, fr))
        return (((st.br_avg - p.br_avg) / max(p.br_avg, 1e-9)) ** 2 + ((st.br_std - p.br_std) / max(p.br_std, 1e-9)) ** 2
                + (0.25 * (st.br_skew - p.br_skew)) ** 2)

    best = None
    for start in range(8):
        x0 = np.random.default_rng(start).normal(0, 1, len(_U_LO) + len(_U_HI) + 2)
        r = minimize(loss, x0, method="Nelder-Mead", options={"maxiter": 4000, "xatol": 1e-8, "fatol": 1e-12})
        if best is None or r.fun < best.fun:
            best = r
        x = _quantile_samples(p, n, best.x)
        if within(stats(x), p):
            return np.random.default_rng(seed).permutation(x).reshape(events, ranks)
    raise InfeasibleProfile("no schedule within tolerance: " + repr(stats(_quantile_samples(p, n, best.x))))


def br_to_counts(row, total_tokens: int, normalize: bool = True) -> np.ndarray:
    """count_r = round(br_r * total / ranks), largest-remainder corrected so the counts
    sum to total when normalize is set."""
    row = np.asarray(row, dtype=np.float64)
    R = len(row)
    if not normalize:
        return np.rint(row * total_tokens / R).astype(np.int64)
    w_ = row / row.sum() * total_tokens
    base = np.floor(w_).astype(np.int64)
    rem = total_tokens - int(base.sum())
    order = np.argsort(-(w_ - base), kind="stable")
    base[order[:rem]] += 1
    return base


def br_q16(sched) -> np.ndarray:
    """Input encoding of a float br schedule [events, ep] as the ABI's Q16 integers (nearest)."""
    return np.rint(np.asarray(sched, dtype=np.float64) * 65536).astype(np.int32)


def op_events(tm, n_events: int) -> np.ndarray:
    """Which gating event routes each template op (structure of the input, from the generator's
    own labels): the ops of MoE layer L in microbatch mb (EXPERT_F / EXPERT_B and their EP all-to-
    alls) belong to gating event (L, mb) (reading R7: one routing decision per MoE layer and
    microbatch, forward and backward); the distinct (L, mb) keys in sorted order are numbered and
    folded onto n_events schedule rows (index mod n_events); -1 = not routed."""
    from . import OPCODES  # label codes of the generator

    lab = tm.ops["label"].astype(np.int64)
    routed = np.isin(lab >> 24, [OPCODES["EXPERT_F"], OPCODES["EXPERT_B"], OPCODES["EP_A2A"]])
    keys = sorted({(int((x >> 12) & 0xFFF), int(x & 0xFFF)) for x in lab[routed]})
    index = {k: i for i, k in enumerate(keys)}
    ev = np.full(len(lab), -1, np.int32)
    for i in np.nonzero(routed)[0]:
        ev[i] = index[(int((lab[i] >> 12) & 0xFFF), int(lab[i] & 0xFFF))] % n_events
    return ev

"""oracle/maturity.py -- TEST INFRASTRUCTURE ONLY.  Non-stall maturity exit on IVF, step by step.

PAPER.md §3.3 "Non-Stall Retrieval" and App. B.2: the search
monitors the quality of newly discovered candidates,

    RQ_t = (d_t - d_best) / (d_worst - d_best)

smooths it with an exponential moving average (window 500 candidates) and halts
when the smoothed signal exceeds tau (0.9) AND the LLM engine is ready for
its next step; otherwise the search stops naturally.  The paper's ANN is HNSW;
SURVEY.md §8(f)1 carries the mechanism to the IVF list order.  The readings (DESIGN.md
§2, R14-R19) followed here, in order:

  R14  a step t is one probed list, in probe-rank order (best centroid first);
  R15  d = -s (inner-product similarity s, higher is better), so
           RQ_t = (s_best - s_t) / (s_best - s_worst);
       s_t = the best score among the rows of list t (the "new candidate"; SPEC.md S:96
       reads one record per step from the best newly discovered candidate);
  R16  s_best / s_worst are the first / last entries of the result list R (the running
       top-k, c1 order: score desc, id asc) AFTER list t has been inserted; if
       s_best == s_worst, RQ_t = 1.0; RQ is not clamped;
       an empty list discovers no candidate: RQ_t = 1.0 (SPEC.md DESIGN DECISIONS);
  R17  EMA_1 = RQ_1, EMA_t = a*RQ_t + (1-a)*EMA_{t-1}, a = 2/(W+1);
  R18  the exit test "EMA_t >= tau and engine ready" is evaluated after every g-th list
       (checkpoints t = g, 2g, ...); the first checkpoint passing it ends the search
       (SPEC.md maturity_point); otherwise the search ends after nprobe_max
       lists (natural stop);
  R19  the result is R as it stood after the last scanned list (SPEC.md results_at_step,
       S:132-138), padded with (-1, -inf).

Scores are fp64 dot products of the stored bf16 values (numpy matmul as a library step);
RQ and EMA are evaluated in fp64.
"""
from __future__ import annotations

import math

import numpy as np

from . import bf16_to_f64


def rq(s_t: float, s_best: float, s_worst: float) -> float:
    """R15/R16: relative quality of the new candidate (similarity form of P:172-174)."""
    if s_best == s_worst:
        return 1.0
    return (s_best - s_t) / (s_best - s_worst)


def ema_update(prev: float | None, x: float, window: int) -> float:
    """R17: EMA seeded with the first observation, alpha = 2/(window+1)."""
    if prev is None:
        return x
    a = 2.0 / (window + 1)
    return a * x + (1.0 - a) * prev


def maturity_point(emas, tau: float, g: int = 1):
    """R18: the first checkpoint t (1-based, t % g == 0) with EMA_t >= tau, else None."""
    for t, e in enumerate(emas, start=1):
        if t % g == 0 and e >= tau:
            return t
    return None


def _topk_union(ids: np.ndarray, sc: np.ndarray, k: int):
    """Definition c1: rank by (score desc, id asc), keep the first k."""
    order = np.lexsort((ids, -sc))[:k]
    return ids[order], sc[order]


def search_query(X_bits: np.ndarray, lists, probe_order, q_bits: np.ndarray, k: int,
                 tau: float, window: int, g: int = 1, ready=True):
    """One query.  probe_order: list ids best first (nprobe_max of them).
    ready(t) -> bool (or a constant): is the engine ready at checkpoint t.
    Returns dict(ids, scores, t_exit, rq [T], ema [T], s_t [T], s_best [T], s_worst [T])."""
    q = bf16_to_f64(q_bits)
    R_ids = np.empty(0, dtype=np.int64)
    R_sc = np.empty(0, dtype=np.float64)
    ema = None
    rqs, emas, sts, sbs, sws = [], [], [], [], []
    t_exit = len(probe_order)
    for t, l in enumerate(probe_order, start=1):
        rows = np.asarray(lists[l], dtype=np.int64)
        if rows.size:
            s = bf16_to_f64(X_bits[rows]) @ q
            s_t = float(s.max())
            R_ids, R_sc = _topk_union(np.concatenate([R_ids, rows]),
                                      np.concatenate([R_sc, s]), k)
            r = rq(s_t, float(R_sc[0]), float(R_sc[-1]))
        else:
            s_t = -math.inf
            r = 1.0
        sbs.append(float(R_sc[0]) if R_sc.size else -math.inf)
        sws.append(float(R_sc[-1]) if R_sc.size else -math.inf)
        ema = ema_update(ema, r, window)
        rqs.append(r)
        emas.append(ema)
        sts.append(s_t)
        is_ready = ready(t) if callable(ready) else bool(ready)
        if t % g == 0 and ema >= tau and is_ready:
            t_exit = t
            break
    ids = np.full(k, -1, dtype=np.int64)
    sc = np.full(k, -np.inf)
    ids[:R_ids.size] = R_ids
    sc[:R_sc.size] = R_sc
    return {"ids": ids, "scores": sc, "t_exit": t_exit, "rq": np.array(rqs),
            "ema": np.array(emas), "s_t": np.array(sts), "s_best": np.array(sbs),
            "s_worst": np.array(sws)}


def search(X_bits, lists, P, Q_bits, k, tau, window, g=1, ready=True):
    """All queries; P [nq, nprobe_max] probe orders.  Returns per-query dicts."""
    return [search_query(X_bits, lists, P[i], Q_bits[i], k, tau, window, g, ready)
            for i in range(Q_bits.shape[0])]

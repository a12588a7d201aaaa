"""oracle/scheduler.py -- TEST INFRASTRUCTURE ONLY.  SearchAgent-X priority scheduling.

PAPER.md §3.2 "Priority Scheduling", written out literally:

  Eq. 1  T_{M,k} = min(M) + (k/G) * (max(M) - min(M)),  0 <= k < G,  M in {R, W, C}
  Eq. 2  k_i = max{ j in [0, G-1] | R_i > T_{R,j} or W_i > T_{W,j} or C_i > T_{C,j} },
         0 when no threshold is exceeded ("assigned to the base level 0")
  order: levels from highest to lowest; inside a level W^cur_i descending

R_i = retrievals completed, C_i = context length of the current sequence, W_i = waiting
time since the initial arrival, W^cur_i = time since the current sequence became ready.
Readings (R20-R21): min/max are taken over the sequences being ordered (the
current waiting set); remaining ties go to the lower request id.
"""
from __future__ import annotations

from fractions import Fraction


def thresholds(values, G):
    """Eq. 1 in exact rational arithmetic (inputs are converted exactly from floats)."""
    vals = [Fraction(v) for v in values]
    lo, hi = min(vals), max(vals)
    return [lo + Fraction(k, G) * (hi - lo) for k in range(G)]


def levels(R, W, C, G):
    """Eq. 2 for every sequence, by enumerating every (j, metric) pair."""
    TR, TW, TC = thresholds(R, G), thresholds(W, G), thresholds(C, G)
    out = []
    for r, w, c in zip(R, W, C):
        r, w, c = Fraction(r), Fraction(w), Fraction(c)
        k = 0
        for j in range(G):
            if r > TR[j] or w > TW[j] or c > TC[j]:
                k = j
        out.append(k)
    return out


def order(ids, R, W, C, Wcur, G):
    """Execution order: level desc, W^cur desc, id asc.  Returns (order as input positions,
    levels)."""
    lv = levels(R, W, C, G)
    pos = sorted(range(len(ids)), key=lambda i: (-lv[i], -Fraction(Wcur[i]), ids[i]))
    return pos, lv

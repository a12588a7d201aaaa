"""oracle/exact.py -- TEST INFRASTRUCTURE ONLY.  Second, independent oracle.

Exact top-k by rational arithmetic: every bf16 value is a dyadic rational,
so with fractions.Fraction the inner products are the exact real numbers and
the ranking (score desc, id asc; PAPER.md P:52 ENN, SPEC.md S:69 tie rule)
is the mathematically exact one.  Pure Python loops -- tiny inputs only
(n, d <= ~64).  Shares no code with oracle.c (pin P9: the two agree).
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np


def _bits_to_fraction(b: int) -> Fraction:
    b = int(b) & 0xFFFF
    sign = -1 if (b >> 15) else 1
    e = (b >> 7) & 0xFF
    m = b & 0x7F
    if e == 0xFF:
        raise ValueError("non-finite bf16 input (precondition R7)")
    if e == 0:                      # subnormal: m * 2^(1-127-7)
        return sign * Fraction(m, 1 << 133)
    v = Fraction(128 + m) * (Fraction(2) ** (e - 127 - 7))
    return sign * v


def exact_topk(X_bits: np.ndarray, Q_bits: np.ndarray, k: int):
    """Returns (ids [nq,k] int64, scores [nq,k] Fraction-or-None)."""
    Xf = [[_bits_to_fraction(v) for v in row] for row in np.asarray(X_bits)]
    Qf = [[_bits_to_fraction(v) for v in row] for row in np.asarray(Q_bits)]
    n = len(Xf)
    ids = np.full((len(Qf), k), -1, dtype=np.int64)
    scores = [[None] * k for _ in Qf]
    for qi, q in enumerate(Qf):
        s = [(sum((a * b for a, b in zip(q, x)), Fraction(0)), i) for i, x in enumerate(Xf)]
        s.sort(key=lambda t: (-t[0], t[1]))
        for j in range(min(k, n)):
            ids[qi, j] = s[j][1]
            scores[qi][j] = s[j][0]
    return ids, scores

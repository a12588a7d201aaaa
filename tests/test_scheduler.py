"""Priority scheduling (§3.2 Eq. 1-2): oracle pins and the native
sa_priority_order against the oracle.  CPU only (host code).

Pins (SPEC.md scheduler examples S:357-395, evaluated by hand):
  S1  Eq. 1: min=0, max=10, G=5 -> thresholds (0, 2, 4, 6, 8); min=max=7 -> all 7; G=1 -> min
  S2  Eq. 2: R spans [0, 5], G=6, R_i=3 with other metrics at their minima -> level 3
      (3 > T_{R,3} = 2.5, 3 is not > T_{R,4} = 10/3); all metrics at minima -> level 0;
      a metric at its maximum (non-degenerate range) -> level G-1
  S3  within a level W^cur descending; G=1 puts everything in level 0 (order = W^cur desc)
  S4  Fig. 3b's scenario: A (r=6, ready later) vs B (r=1, ready earlier): FCFS would serve B
      first; priority serves A first
"""
from fractions import Fraction

import numpy as np
import pytest

from oracle import scheduler as osch


def test_s1_thresholds():
    assert osch.thresholds([0, 10, 3], 5) == [0, 2, 4, 6, 8]
    assert osch.thresholds([7, 7], 4) == [7, 7, 7, 7]
    assert osch.thresholds([3, 9], 1) == [3]
    assert osch.thresholds([0, 5], 6)[3] == Fraction(5, 2)


def test_s2_levels():
    assert osch.levels([0, 5, 3], [0, 0, 0], [0, 0, 0], 6) == [0, 5, 3]
    assert osch.levels([2, 2], [1, 1], [4, 4], 6) == [0, 0]         # degenerate ranges
    # G=4: T_W = (0, 2.5, 5, 7.5), T_C = (100, 150, 200, 250); R degenerate
    lv = osch.levels([0, 0, 0], [10, 0, 5], [100, 300, 200], 4)
    assert lv == [3, 3, 1]          # W max; C max; W=5 and C=200 exceed only the k=1 thresholds


def test_s3_order_within_level_and_g1():
    pos, lv = osch.order([10, 11, 12], [1, 1, 1], [0, 0, 0], [0, 0, 0], [5, 9, 7], 6)
    assert pos == [1, 2, 0] and lv == [0, 0, 0]
    pos, _ = osch.order([0, 1, 2], [0, 5, 3], [1, 2, 3], [9, 9, 9], [1, 3, 2], 1)
    assert pos == [1, 2, 0]                                           # G=1: W^cur desc only


def test_s4_fig3b_priority_beats_fcfs():
    # A: r=6, became ready 1 s ago; B: r=1, ready 5 s ago (FCFS would take B first)
    pos, lv = osch.order([0, 1], [6, 1], [10, 10], [500, 500], [1, 5], 6)
    assert pos == [0, 1] and lv == [5, 0]


def brute_level(i, R, W, C, G):
    """Eq. 2 straight from the definition with float thresholds computed as rationals."""
    best = 0
    for j in range(G):
        for M in (R, W, C):
            T = Fraction(min(M)) + Fraction(j, G) * (Fraction(max(M)) - Fraction(min(M)))
            if Fraction(M[i]) > T:
                best = max(best, j)
    return best


def test_native_matches_oracle_random(sa):
    g = np.random.default_rng(7)
    for trial in range(1000):
        n = int(g.integers(1, 21))
        G = int(g.integers(1, 9))
        R = g.integers(0, 8, n)
        W = g.integers(0, 10_000_000, n) if trial % 3 else g.integers(0, 4, n)
        C = g.integers(100, 20_000, n)
        Wc = g.integers(0, 5_000_000, n) if trial % 2 else g.integers(0, 3, n)
        ids = g.permutation(1000)[:n]
        order, lv = sa.sa_priority_order(R, W, C, Wc, ids, G)
        pos, olv = osch.order(ids.tolist(), R.tolist(), W.tolist(), C.tolist(), Wc.tolist(), G)
        assert lv.tolist() == olv
        assert order.tolist() == pos
        if trial < 100:
            assert olv == [brute_level(i, R.tolist(), W.tolist(), C.tolist(), G) for i in range(n)]


def test_native_exact_at_level_boundaries(sa):
    # metric values exactly on thresholds: strict '>' keeps them one level down
    R = np.array([0, 6, 3, 2, 4])       # G=6 over [0, 6]: T = 0,1,2,3,4,5
    z = np.zeros(5, dtype=np.int64)
    order, lv = sa.sa_priority_order(R, z, z, z, np.arange(5), 6)
    assert lv.tolist() == [0, 5, 2, 1, 3]
    assert order.tolist() == [1, 4, 2, 3, 0]


def test_native_rejects_bad_input(sa):
    z = np.zeros(3, dtype=np.int64)
    with pytest.raises(sa.SAError):
        sa.sa_priority_order(z, z, z, z, z, 0)
    with pytest.raises(sa.SAError):
        sa.sa_priority_order(np.array([-1, 0, 0]), z, z, z, z, 6)
    order, lv = sa.sa_priority_order(np.zeros(0), np.zeros(0), np.zeros(0), np.zeros(0),
                                     np.zeros(0), 6)
    assert order.size == 0

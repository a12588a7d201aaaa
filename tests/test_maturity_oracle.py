"""Pins for the maturity-exit oracle (oracle/maturity.py) -- CPU only.

M1  hand-evaluated trace on a 5-list IVF (tests/golden/maturity_trace.txt)
M2  SPEC.md's rq / ema_update / maturity_point examples, converted to the
    similarity form of reading R15 (d = -s)
M3  never ready -> natural stop: result == exact top-k over the union of all probed lists
    (oracle.c, an independent routine)
M4  results-at-exit: the result equals the exact top-k over the union of the first t_exit
    lists (oracle.c); RQ >= 0; RQ == 0 exactly when the list holds the new best
M5  tau = 0 with the engine ready exits at the first checkpoint (EMA >= 0 always)
"""
import math
import os

import numpy as np
import pytest

import oracle
from oracle import ivf, maturity

HERE = os.path.dirname(os.path.abspath(__file__))


def bits(x):
    return oracle.bf16_round(np.asarray(x, dtype=np.float32))


def load_golden():
    rows, empties, steps, exits = [], [], [], []
    k = window = None
    for line in open(os.path.join(HERE, "golden", "maturity_trace.txt")):
        line = line.split("#")[0].split()
        if not line:
            continue
        tag, vals = line[0], line[1:]
        if tag == "row":
            rows.append((int(vals[0]), int(vals[1]), float(vals[2])))
        elif tag == "empty":
            empties.append(int(vals[0]))
        elif tag == "k":
            k = int(vals[0])
        elif tag == "window":
            window = int(vals[0])
        elif tag == "step":
            steps.append((int(vals[0]), int(vals[1]), float(vals[2]), float(vals[3]),
                          float(vals[4])))
        elif tag == "exit":
            exits.append((float(vals[0]), int(vals[1]), bool(int(vals[2])), int(vals[3]),
                          [int(v) for v in vals[4:]]))
    return rows, empties, k, window, steps, exits


def golden_geometry():
    """The vectors the golden file describes (shared with the GPU test)."""
    rows, empties, k, window, steps, exits = load_golden()
    nlist, d = 5, 8
    eps = [1 / 8, 1 / 16, 1 / 32, 1 / 64, 1 / 128]
    X = np.zeros((len(rows), d))
    lists = [[] for _ in range(nlist)]
    for gid, l, s in rows:
        X[gid, 0] = s - eps[l] / 2
        X[gid, l + 1] = 0.5
        lists[l].append(gid)
    C = np.zeros((nlist, d))
    for j in range(nlist):
        C[j, j + 1] = 1.0
    q = np.zeros(d)
    q[0] = 1.0
    for j in range(nlist):
        q[j + 1] = eps[j]
    return bits(X), [np.array(v, dtype=np.int64) for v in lists], C, bits(q[None, :]), k, window


def test_m1_golden_trace():
    X, lists, C, Q, k, window = golden_geometry()
    _, _, _, _, steps, exits = load_golden()
    # the geometry itself: probe order 0..4 and the designed scores are exact
    P, _ = ivf.probe(Q, bits(C), 5)
    assert list(P[0]) == [0, 1, 2, 3, 4]
    r = maturity.search_query(X, lists, P[0], Q[0], k, tau=math.inf, window=window)
    assert r["t_exit"] == 5
    for (t, l, s_t, rq, ema) in steps:
        assert P[0][t - 1] == l
        assert r["s_t"][t - 1] == s_t
        assert r["rq"][t - 1] == rq
        assert r["ema"][t - 1] == ema
    for tau, g, ready, t_exit, ids in exits:
        r = maturity.search_query(X, lists, P[0], Q[0], k, tau=tau, window=window, g=g,
                                  ready=ready)
        assert r["t_exit"] == t_exit, (tau, g, ready)
        assert list(r["ids"]) == ids


def test_m2_spec_examples():
    # rq, distances d -> similarities s = -d
    assert maturity.rq(-0.2, -0.2, -0.8) == 0.0
    assert maturity.rq(-0.8, -0.2, -0.8) == 1.0
    assert maturity.rq(-0.5, -0.2, -0.8) == pytest.approx(0.5, abs=1e-15)
    assert maturity.rq(-0.3, -0.3, -0.3) == 1.0          # degenerate list: saturated
    assert maturity.rq(-2.0, -0.2, -0.8) == pytest.approx(3.0, abs=1e-14)  # not clamped
    # ema_update
    assert maturity.ema_update(None, 0.4, 500) == 0.4
    assert maturity.ema_update(0.7, 0.7, 37) == 0.7
    assert maturity.ema_update(0.0, 1.0, 1) == 1.0
    assert maturity.ema_update(1.0, 0.0, 3) == 0.5
    # maturity_point
    assert maturity.maturity_point([0.2, 0.5, 0.91, 0.95], 0.9) == 3
    assert maturity.maturity_point([0.2, 0.5], 0.0) == 1
    assert maturity.maturity_point([0.2, 0.5, 0.3], 0.9) is None
    assert maturity.maturity_point([0.95, 0.5, 0.91, 0.95], 0.9, g=2) == 4


def mixture_ivf(n=3000, d=32, nlist=24, nq=12, seed=3):
    g = np.random.default_rng(seed)
    cent = g.standard_normal((8, d))
    X = cent[g.integers(0, 8, n)] + 0.6 * g.standard_normal((n, d))
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    Q = cent[g.integers(0, 8, nq)] + 0.6 * g.standard_normal((nq, d))
    Q /= np.linalg.norm(Q, axis=1, keepdims=True)
    Xb, Qb = bits(X), bits(Q)
    C, Cb, assign, lists = ivf.build(Xb, nlist, iters=4)
    return Xb, Qb, Cb, lists


@pytest.mark.parametrize("k", [1, 5, 10])
def test_m3_m4_prefix_results_are_exact(k):
    Xb, Qb, Cb, lists = mixture_ivf()
    P, _ = ivf.probe(Qb, Cb, 12)
    for tau, g in [(math.inf, 1), (0.5, 1), (1.0, 3), (2.0, 2)]:
        res = maturity.search(Xb, lists, P, Qb, k, tau=tau, window=4, g=g)
        for qi, r in enumerate(res):
            t = r["t_exit"]
            assert 1 <= t <= 12
            if tau == math.inf:
                assert t == 12
            else:
                assert t == 12 or (t % g == 0 and r["ema"][t - 1] >= tau)
            rows = np.sort(np.concatenate([lists[j] for j in P[qi][:t]]))
            ids, sc = oracle.flat_topk(Xb[rows], Qb[qi:qi + 1], k)
            want = np.where(ids[0] >= 0, rows[np.maximum(ids[0], 0)], -1)
            assert np.array_equal(r["ids"], want)
            assert np.allclose(r["scores"][want >= 0], sc[0][want >= 0], rtol=0, atol=1e-12)
            assert np.all(r["rq"] >= 0)
            # RQ == 0 exactly when list t brought the new best
            # (s_best after list t = the running max of s_1..s_t)
            for tt in range(len(r["rq"])):
                if len(lists[P[qi][tt]]) == 0 or k == 1:   # no candidate / s_best == s_worst
                    assert r["rq"][tt] == 1.0
                else:
                    new_best = r["s_t"][tt] == np.max(r["s_t"][:tt + 1])
                    assert (r["rq"][tt] == 0.0) == new_best


def test_m5_tau_zero_exits_at_first_checkpoint():
    Xb, Qb, Cb, lists = mixture_ivf()
    P, _ = ivf.probe(Qb, Cb, 9)
    for g in (1, 2, 4):
        for r in maturity.search(Xb, lists, P, Qb, 5, tau=0.0, window=8, g=g):
            assert r["t_exit"] == g


def test_ready_callback_delays_exit():
    """Engine readiness gates the exit: ready only from checkpoint 6 on."""
    Xb, Qb, Cb, lists = mixture_ivf()
    P, _ = ivf.probe(Qb, Cb, 12)
    for r in maturity.search(Xb, lists, P, Qb, 5, tau=0.0, window=8, g=2,
                             ready=lambda t: t >= 6):
        assert r["t_exit"] == 6

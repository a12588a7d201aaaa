"""Pins for the exact-search oracle (P1-P6, P9) -- CPU only.

Each test pins oracle/oracle.c to something other than itself: a worked
example from the spec, closed forms, exact ties, a library routine (torch's
RNE cast), or an independent exact-rational oracle (oracle/exact.py).
"""
import os

import numpy as np
import pytest
import torch

import oracle
from oracle.exact import exact_topk

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def bits(x):
    return oracle.bf16_round(np.asarray(x, dtype=np.float32))


# ---- bf16 rounding (reading R3) pinned to torch's RNE cast -------------------

def test_bf16_round_matches_torch_cast():
    g = np.random.default_rng(0)
    x = np.concatenate([
        g.standard_normal(100_000).astype(np.float32),
        (g.standard_normal(10_000) * 1e-39).astype(np.float32),     # subnormals
        (g.standard_normal(10_000) * 1e30).astype(np.float32),
        np.array([0.0, -0.0, 1.0, -1.0, 3.4e38, -3.4e38, 1e-45, 0.9,
                  np.inf, -np.inf], dtype=np.float32),
    ])
    # exact ties: bit patterns with the low 16 bits == 0x8000
    ties = (g.integers(0, 1 << 15, 5000).astype(np.uint32) << 16 | 0x8000).astype(np.uint32)
    ties = ties[((ties >> 23) & 0xFF) != 0xFF].view(np.float32)
    x = np.concatenate([x, ties])
    want = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    got = oracle.bf16_round(x)
    assert np.array_equal(got, want)


def test_bf16_round_known_values():
    # 0.9 -> 0x3F66 (0.8984375); 1 + 2^-8 is a tie -> even (1.0); 1 + 3*2^-8 -> up
    assert oracle.bf16_round(np.float32([0.9]))[0] == 0x3F66
    assert oracle.bf16_round(np.float32([1 + 2 ** -8]))[0] == 0x3F80
    assert oracle.bf16_round(np.float32([1 + 3 * 2 ** -8]))[0] == 0x3F82


# ---- P1: worked example from SPEC.md S:73 converted to IP ----------------------

def _load_golden(name):
    rows, q, k, exp = [], None, None, []
    for line in open(os.path.join(GOLDEN, name)):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        tag, *vals = line.split()
        if tag == "row":
            rows.append([float(v) for v in vals])
        elif tag == "query":
            q = [float(v) for v in vals]
        elif tag == "k":
            k = int(vals[0])
        elif tag == "expect":
            exp.append((int(vals[0]), float(vals[1])))
    return np.array(rows, np.float32), np.array([q], np.float32), k, exp


def test_p1_spec_example():
    X, Q, k, exp = _load_golden("p1_spec_example.txt")
    ids, sc = oracle.flat_topk(bits(X), bits(Q), k)
    assert ids[0].tolist() == [e[0] for e in exp]
    assert sc[0].tolist() == [e[1] for e in exp]        # exact values


# ---- P2: query = corpus row -> that row first, score = its squared norm --------

def test_p2_self_query():
    g = np.random.default_rng(1)
    X = g.standard_normal((500, 64)).astype(np.float32)
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    Xb = bits(X)
    ids, sc = oracle.flat_topk(Xb, Xb[[7, 300]], 3)
    assert ids[:, 0].tolist() == [7, 300]
    # closed form: |x|^2 of the stored bf16 row, by exact rational arithmetic
    _, ex = exact_topk(Xb[7:8], Xb[7:8], 1)
    assert sc[0, 0] == float(ex[0][0])


# ---- P3: k = n is a sorted permutation; k = n + 3 pads (-1, -inf) -------------

def test_p3_k_equals_n_and_padding():
    g = np.random.default_rng(2)
    X = bits(g.standard_normal((37, 16)))
    Q = bits(g.standard_normal((4, 16)))
    ids, sc = oracle.flat_topk(X, Q, 37)
    for qi in range(4):
        assert sorted(ids[qi].tolist()) == list(range(37))
        assert np.all(np.diff(sc[qi]) <= 0)
    ids3, sc3 = oracle.flat_topk(X, Q, 40)
    assert np.array_equal(ids3[:, :37], ids)
    assert np.all(ids3[:, 37:] == -1) and np.all(np.isneginf(sc3[:, 37:]))


# ---- P4: orthonormal corpus -> exact ties at 0 broken by lowest id ------------

def test_p4_orthonormal_ties():
    d = 32
    X = bits(np.eye(d))
    for j in (0, 5, 31):
        ids, sc = oracle.flat_topk(X, X[j:j + 1], 6)
        rest = [i for i in range(d) if i != j][:5]
        assert ids[0].tolist() == [j] + rest
        assert sc[0].tolist() == [1.0] + [0.0] * 5


# ---- P5: duplicate rows -> both returned, lower id first ------------------------

def test_p5_duplicates():
    g = np.random.default_rng(3)
    X = g.standard_normal((200, 24)).astype(np.float32)
    X[150] = X[20]
    X[199] = X[20]
    q = X[20:21] + 0.01 * g.standard_normal((1, 24)).astype(np.float32)
    ids, sc = oracle.flat_topk(bits(X), bits(q), 3)
    assert ids[0].tolist() == [20, 150, 199]
    assert sc[0, 0] == sc[0, 1] == sc[0, 2]


# ---- P6: all scores negative -> least-negative win (init is -inf, not 0) --------

def test_p6_all_negative():
    g = np.random.default_rng(4)
    q = g.standard_normal(16).astype(np.float32)
    scale = np.array([3.0, 0.5, 2.0, 0.25, 1.0, 4.0], np.float32)   # exact in bf16
    X = -scale[:, None] * bits_to_f32(bits(q))[None, :]
    ids, sc = oracle.flat_topk(bits(X), bits(q[None]), 3)
    assert ids[0].tolist() == [3, 1, 4]          # ascending scale = least negative
    assert np.all(sc[0] < 0)


def bits_to_f32(b):
    return (b.astype(np.uint32) << 16).view(np.float32)


# ---- P9: C oracle == exact rational oracle on random tiny instances -----------

@pytest.mark.parametrize("seed", range(4))
def test_p9_against_exact_rational(seed):
    g = np.random.default_rng(100 + seed)
    for _ in range(250):
        n = int(g.integers(1, 48))
        d = int(g.integers(1, 17))
        k = int(g.integers(1, n + 4))
        nq = int(g.integers(1, 4))
        kind = g.integers(0, 3)
        if kind == 0:
            X = g.standard_normal((n, d))
        elif kind == 1:     # small integers: many exact ties
            X = g.integers(-2, 3, (n, d)).astype(np.float64)
        else:               # duplicated rows
            base = g.standard_normal((max(1, n // 3), d))
            X = base[g.integers(0, base.shape[0], n)]
        Q = g.integers(-2, 3, (nq, d)).astype(np.float64) if kind == 1 else g.standard_normal((nq, d))
        Xb, Qb = bits(X), bits(Q)
        ids, sc = oracle.flat_topk(Xb, Qb, k)
        eids, esc = exact_topk(Xb, Qb, k)
        assert np.array_equal(ids, eids), (n, d, k)
        for qi in range(nq):
            for j in range(k):
                if esc[qi][j] is None:
                    assert np.isneginf(sc[qi, j])
                else:
                    assert sc[qi, j] == float(esc[qi][j])


# ---- streaming: chunked updates == one call (used at full size) --------------

def test_streaming_chunks_equal_single_call():
    g = np.random.default_rng(5)
    X = bits(g.standard_normal((1000, 32)))
    Q = bits(g.standard_normal((7, 32)))
    ids, sc = oracle.flat_topk(X, Q, 12)
    t = oracle.TopK(Q, 12)
    for lo in range(0, 1000, 137):
        t.update(X[lo:lo + 137], lo)
    assert np.array_equal(t.ids, ids) and np.array_equal(t.scores, sc)


def test_pair_scores_match_topk_scores():
    g = np.random.default_rng(6)
    X = bits(g.standard_normal((300, 48)))
    Q = bits(g.standard_normal((5, 48)))
    ids, sc = oracle.flat_topk(X, Q, 4)
    qi = np.repeat(np.arange(5), 4)
    ps = oracle.pair_scores(X, Q, qi, ids.reshape(-1))
    assert np.array_equal(ps.reshape(5, 4), sc)

"""Pins for the fp8 oracle (oracle/fp8.py, readings R30-R33) -- CPU only.

F1  e4m3 rounding == torch's float8_e4m3fn cast (a library routine) on 100k+ values spanning
    subnormals, ties and the top binade (|v| <= 448), values and byte codes
F2  hand-evaluated values: ties to even (1.0625 -> 1, 1.1875 -> 1.25, 2^-10 -> 0,
    3*2^-10 -> 2^-8), saturation (460 / 464 / 470 / 1e6 -> 448), signed zero (-1e-5 -> 0x80)
F3  scale exponent by hand (448 -> 0, 449 -> -1, 0.875 -> 9, 0.876 -> 8, 1 -> 8) and
    scale invariance: scaling the corpus by 2^j shifts e by -j and leaves the codes unchanged
F4  n_cand >= n: the fp8 + re-rank search is the exact search (oracle.c), ids and scores
F5  the re-rank: the result is the exact top-k over the candidate rows, and contains the
    exact top-k whenever those lie among the candidates
"""
import numpy as np
import torch

import oracle
from oracle import fp8
from datagen import make_mixture, draw_rows, to_bf16_bits


def test_f1_rounding_matches_torch():
    g = np.random.default_rng(0)
    x = np.concatenate([g.standard_normal(100_000) * np.exp(g.uniform(-14, 7, 100_000)),
                        np.arange(-4000, 4000) * 2.0 ** -12,      # grid points and midpoints
                        np.arange(-3600, 3600) * 0.125])
    x = x[np.abs(x) <= 448]
    t = torch.from_numpy(x).to(torch.float8_e4m3fn)
    r = fp8.e4m3_round(x)
    assert np.array_equal(r, t.to(torch.float64).numpy())
    assert np.array_equal(fp8.e4m3_bits(r), t.view(torch.uint8).numpy())


def test_f2_hand_values():
    v = np.array([1.0625, 1.1875, 2.0 ** -10, 3 * 2.0 ** -10, 460, 464, 470, 1e6, -1e6,
                  -2.0 ** -9, -1e-5, 15.5, 0.0])
    r = fp8.e4m3_round(v)
    assert r.tolist() == [1.0, 1.25, 0.0, 2.0 ** -8, 448, 448, 448, 448, -448,
                          -2.0 ** -9, 0.0, 16.0, 0.0]
    assert [int(b) for b in fp8.e4m3_bits(r)] == [0x38, 0x3A, 0x00, 0x02, 0x7E, 0x7E, 0x7E,
                                                 0x7E, 0xFE, 0x81, 0x80, 0x58, 0x00]


def test_f3_scale_exponent():
    assert [fp8.scale_exponent(m) for m in (448, 449, 0.875, 0.876, 1.0, 0.0)] == [0, -1, 9, 8,
                                                                                  8, 0]
    mx = make_mixture(d=64, C=4, r=8)
    Xb = to_bf16_bits(draw_rows(mx, 300, row_seed=3))
    X8, e = fp8.quantize_corpus(Xb)
    for j in (-3, 2):
        Xs = oracle.bf16_round((oracle.bf16_to_f64(Xb) * 2.0 ** j).astype(np.float32))
        X8s, es = fp8.quantize_corpus(Xs)
        assert es == e - j and np.array_equal(fp8.e4m3_bits(X8s), fp8.e4m3_bits(X8))
    # queries: each row on its own scale
    Q8, eq = fp8.quantize_queries(Xb[:5])
    for i in range(5):
        assert eq[i] == fp8.scale_exponent(np.abs(oracle.bf16_to_f64(Xb[i])).max())


def test_f4_all_candidates_is_exact():
    mx = make_mixture(d=128, C=16, r=16)
    Xb = to_bf16_bits(draw_rows(mx, 500, row_seed=5))
    Qb = to_bf16_bits(draw_rows(mx, 20, row_seed=6))
    ids, sc, rows = fp8.search(Xb, Qb, 10, 500)
    ei, es = oracle.flat_topk(Xb, Qb, 10)
    assert np.array_equal(ids, ei) and np.array_equal(sc, es)


def test_f5_rerank_is_exact_over_candidates():
    mx = make_mixture(d=128, C=16, r=16)
    Xb = to_bf16_bits(draw_rows(mx, 3000, row_seed=7))
    Qb = to_bf16_bits(draw_rows(mx, 30, row_seed=8))
    ids, sc, rows = fp8.search(Xb, Qb, 10, 32)
    ei, es = oracle.flat_topk(Xb, Qb, 10)
    hit = 0
    for q in range(30):
        r = rows[q]
        ci, cs = oracle.flat_topk(Xb[r], Qb[q:q + 1], 10)
        assert np.array_equal(ids[q], r[ci[0]]) and np.array_equal(sc[q], cs[0])
        if set(ei[q]) <= set(r):
            hit += 1
            assert np.array_equal(ids[q], ei[q])
    assert hit >= 28      # e4m3 candidates keep the true top-10 for almost every query

"""oracle/fp8.py -- TEST INFRASTRUCTURE ONLY.  e4m3 flat scan + bf16 re-rank, step by step.

Not in the paper (SURVEY.md §8(f)4 "fp8-e4m3 corpus for the flat scan ... with bf16 re-rank");
a compressed variant of the exact mode (ENN).  Readings:

  R30  corpus: X8 = e4m3(x * 2^e) with e the largest integer such that max|x| * 2^e <= 448,
       max over the whole corpus; e4m3 = round to nearest, ties to even, on the OCP E4M3
       ("fn") grid -- 3 mantissa bits, exponent bias 7, subnormal quantum 2^-9, largest
       finite 448 -- saturating to +-448 (no inf; 480 would be the NaN code);
  R31  queries: the same per query row, with the row's own maximum;
  R32  candidates: the n_cand best rows by <q8, x8> (score desc, row asc);
  R33  re-rank: the candidates re-scored on the bf16 values, the k best (score desc, id asc),
       padded (-1, -inf).
  R35  IVF: with nprobe > 0 the candidates of R32 are taken among the rows of the query's
       nprobe best lists (probed on the bf16 query, R11) -- `candidates` over that row subset.

Values are fp64; every e4m3 value times a power of two is exactly a bf16 value (3 <= 7 mantissa
bits, exponents in range), so the fp8 scores of R32 are the C oracle's exact fp64 scan over
those bf16 values (oracle.flat_topk, a library step).
"""
from __future__ import annotations

import numpy as np

from . import bf16_to_f64, flat_topk, pair_scores

E4M3_MAX = 448.0


def e4m3_round(v) -> np.ndarray:
    """R30's rounding on fp64 values -> fp64 values on the e4m3 grid (sign kept, incl. -0)."""
    v = np.asarray(v, dtype=np.float64)
    a = np.abs(v)
    out = np.zeros_like(a)
    nz = a > 0
    # binade exponent E = floor(log2 a) (a = f * 2^X, f in [0.5, 1): E = X - 1, exact),
    # at least -6 (below it the subnormal quantum 2^-9), at most 8 (the top binade)
    _, X = np.frexp(a)
    E = np.clip(np.where(nz, X.astype(np.int64) - 1, -6), -6, 8)
    quantum = np.ldexp(1.0, E - 3)
    out = np.round(a / quantum) * quantum     # np.round: ties to even; a/quantum is exact
    out = np.minimum(out, E4M3_MAX)
    return np.copysign(out, v)


def e4m3_bits(v) -> np.ndarray:
    """Encode values already on the e4m3 grid (e4m3_round output) to their byte codes."""
    v = np.asarray(v, dtype=np.float64)
    a = np.abs(v)
    code = np.zeros(a.shape, dtype=np.int64)
    sub = a < 2.0 ** -6
    code[sub] = np.round(a[sub] / 2.0 ** -9).astype(np.int64)   # exponent field 0
    nrm = ~sub
    if nrm.any():
        E = np.frexp(a[nrm])[1].astype(np.int64) - 1
        mant = a[nrm] / np.ldexp(1.0, E) * 8 - 8
        code[nrm] = ((E + 7) << 3) | np.round(mant).astype(np.int64)
    code |= np.signbit(v).astype(np.int64) << 7
    return code.astype(np.uint8)


def scale_exponent(m: float) -> int:
    """The largest integer e with m * 2^e <= 448 (0 when m == 0)."""
    if m == 0:
        return 0
    e = 0
    while m * 2.0 ** (e + 1) <= E4M3_MAX:
        e += 1
    while m * 2.0 ** e > E4M3_MAX:
        e -= 1
    return e


def quantize_corpus(X_bits: np.ndarray):
    """R30 -> (e4m3 values fp64 [n, d], e)."""
    X = bf16_to_f64(X_bits)
    e = scale_exponent(float(np.abs(X).max()) if X.size else 0.0)
    return e4m3_round(X * 2.0 ** e), e


def quantize_queries(Q_bits: np.ndarray):
    """R31 -> (e4m3 values fp64 [nq, d], e per row)."""
    Q = bf16_to_f64(Q_bits)
    es = np.array([scale_exponent(float(np.abs(q).max())) for q in Q], dtype=np.int64)
    return e4m3_round(Q * np.ldexp(1.0, es)[:, None]), es


def _as_bf16_bits(v: np.ndarray) -> np.ndarray:
    """fp64 values that are exactly bf16 (e4m3 grid values) -> bf16 bit patterns."""
    f = np.ascontiguousarray(v, dtype=np.float32)
    bits = f.view(np.uint32)
    assert np.all(bits & 0xFFFF == 0), "value not exactly representable in bf16"
    return (bits >> 16).astype(np.uint16)


def candidates(X_bits: np.ndarray, Q_bits: np.ndarray, n_cand: int):
    """R32 -> (rows int64 [nq, n_cand], fp8 scores fp64 [nq, n_cand] in the scaled units),
    padded (-1, -inf)."""
    X8, _ = quantize_corpus(X_bits)
    Q8, _ = quantize_queries(Q_bits)
    return flat_topk(_as_bf16_bits(X8), _as_bf16_bits(Q8), n_cand)


def search(X_bits: np.ndarray, Q_bits: np.ndarray, k: int, n_cand: int, ids=None):
    """R30-R33 -> (ids int64 [nq, k], scores fp64 [nq, k], candidate rows [nq, n_cand]).
    ids: optional global id of each row (default: the row index)."""
    rows, _ = candidates(X_bits, Q_bits, n_cand)
    gid = np.arange(X_bits.shape[0], dtype=np.int64) if ids is None else np.asarray(ids)
    nq = Q_bits.shape[0]
    out_i = np.full((nq, k), -1, dtype=np.int64)
    out_s = np.full((nq, k), -np.inf)
    for q in range(nq):
        r = rows[q][rows[q] >= 0]
        s = pair_scores(X_bits, Q_bits, np.full(r.size, q), r)
        g = gid[r]
        order = np.lexsort((g, -s))[:k]
        out_i[q, :order.size] = g[order]
        out_s[q, :order.size] = s[order]
    return out_i, out_s, rows

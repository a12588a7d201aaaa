"""oracle/ivf.py -- TEST INFRASTRUCTURE ONLY.  IVF build + search, step by step.

The paper has no IVF (its ANN is HNSW, App. B.3); BASELINE.json
names IVF with an nprobe knob as the approximate mode.  This oracle follows
the algorithm fixed by DESIGN.md readings R8-R11 in order,
in float64, with numpy matmul / argmax / sort as library steps:

  1. sample  rows floor(t * n_total / n_train), n_train = min(n_total, 256*nlist)   (R9)
  2. init    c_j = sample[j * s + o], s = n_train // nlist, o = splitmix64(seed) % s (R9)
  3. repeat `iters` times (no early stop)                                          (R8)
       c_bf16 = RNE_bf16(float32(c))
       a(x)   = argmax_j <x, c_bf16_j>   (first maximum = lowest j)
       c_j    = normalise(sum of members) ; empty lists -> R10
  4. assign every row with the final c_bf16; list = rows in ascending id
  5. probe   top-nprobe lists by <q, c_bf16> (score desc, id asc)                   (R11)
  6. scan    exact top-k over the union of the probed lists (oracle.c definition)

The library computes the same decisions with fp32 tensor-core products;
tests compare on inputs whose decisions have margins far above both
precisions, and otherwise check properties.
"""
from __future__ import annotations

import numpy as np

from . import bf16_round, bf16_to_f64, flat_topk

MASK64 = (1 << 64) - 1


def splitmix64(z: int) -> int:
    """SplitMix64 output for state z (Steele et al.; reference vector: z=0 ->
    0xE220A8397B1DCDAF)."""
    z = (z + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def sample_rows(n_total: int, nlist: int, train_per_list: int = 256) -> np.ndarray:
    n_train = min(n_total, train_per_list * nlist)
    t = np.arange(n_train, dtype=np.int64)
    return (t * n_total) // n_train


def centroids_bf16(C: np.ndarray) -> np.ndarray:
    """fp64 centroids -> stored fp32 -> RNE bf16 bits."""
    return bf16_round(C.astype(np.float32))


def kmeans(X_bits: np.ndarray, nlist: int, iters: int = 20, train_per_list: int = 256,
           seed: int = 0x5A2505, trace: list | None = None):
    """Returns (C float64 [nlist, d], last assignment of the sample, sample row ids)."""
    n = X_bits.shape[0]
    rows = sample_rows(n, nlist, train_per_list)
    S = bf16_to_f64(X_bits[rows])
    n_train = S.shape[0]
    stride = n_train // nlist
    o = splitmix64(seed) % stride
    C = S[np.arange(nlist) * stride + o].copy()
    a = None
    for _ in range(iters):
        C, a, margin = lloyd_step(S, C)
        if trace is not None:
            trace.append(float(np.min(margin)) if nlist > 1 else np.inf)
    return C, a, rows


def lloyd_step(S: np.ndarray, C: np.ndarray):
    """One iteration of step 3 (R8, R10) from centroids C (fp64 [nlist, d]) over the sample S
    (fp64 [n_train, d]).  Returns (new C, assignment, margin) -- margin = best minus second-best
    score of each sample row (+inf when nlist = 1), the size of the decision a(x)."""
    nlist, n_train = C.shape[0], S.shape[0]
    Cb = bf16_to_f64(centroids_bf16(C))
    sc = S @ Cb.T
    a = np.argmax(sc, axis=1)
    best = sc[np.arange(n_train), a]
    if nlist > 1:
        srt = np.sort(sc, axis=1)
        margin = srt[:, -1] - srt[:, -2]
    else:
        margin = np.full(n_train, np.inf)
    newC = np.zeros_like(C)
    empty = []
    for j in range(nlist):
        m = a == j
        if not m.any():
            empty.append(j)
            continue
        s = S[m].sum(axis=0)
        newC[j] = s / np.linalg.norm(s)
    if empty:
        # R10: empty lists (ascending) take the lowest-scored sample rows, (score, row) ascending
        order = np.lexsort((np.arange(n_train), best))
        for r, j in zip(order, empty):
            newC[j] = S[r]
    return newC, a, margin


def build(X_bits: np.ndarray, nlist: int, iters: int = 20, train_per_list: int = 256,
          seed: int = 0x5A2505, trace: list | None = None):
    C, _, _ = kmeans(X_bits, nlist, iters, train_per_list, seed, trace)
    Cb_bits = centroids_bf16(C)
    sc = bf16_to_f64(X_bits) @ bf16_to_f64(Cb_bits).T
    assign = np.argmax(sc, axis=1)
    lists = [np.nonzero(assign == j)[0] for j in range(nlist)]
    return C, Cb_bits, assign, lists


def probe(Q_bits: np.ndarray, Cb_bits: np.ndarray, nprobe: int):
    ids, scores = flat_topk(Cb_bits, Q_bits, nprobe)
    return ids, scores


def search(X_bits: np.ndarray, lists, Cb_bits: np.ndarray, Q_bits: np.ndarray, k: int,
           nprobe: int):
    P, _ = probe(Q_bits, Cb_bits, nprobe)
    nq = Q_bits.shape[0]
    out_ids = np.full((nq, k), -1, dtype=np.int64)
    out_sc = np.full((nq, k), -np.inf)
    for qi in range(nq):
        rows = np.sort(np.concatenate([lists[j] for j in P[qi]]))
        if rows.size == 0:
            continue
        ids, sc = flat_topk(X_bits[rows], Q_bits[qi:qi + 1], k)
        valid = ids[0] >= 0
        out_ids[qi, :valid.sum()] = rows[ids[0][valid]]
        out_sc[qi, :valid.sum()] = sc[0][valid]
    return out_ids, out_sc, P

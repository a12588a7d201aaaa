"""oracle/graph.py -- TEST INFRASTRUCTURE ONLY.  Proximity-graph ANN (build + beam search),
step by step.

The paper's retriever is a graph index (HNSW, §2, App. B.3) whose
"search range" (efSearch) trades recall for effort (§2.2.1).  SURVEY.md §8(f)3 asks
for a GPU graph index with that knob.  The build follows the rank-based recipe of GPU graph
indexes (an approximate kNN graph, detour-count pruning, reverse edges); the search is
best-first beam search over a candidate list of size L (the search range).  Readings
(R22-R27), in order:

  R22  knn(i): the K best rows by inner product (score desc, id asc) among the candidates
       of row i, excluding i itself (candidates: every row, or a given set such as the
       union of i's probed IVF lists);
  R23  detour(i, j) for the neighbour c_j at 0-based rank j of knn(i):
           #{ k < j : c_j occurs in knn(c_k) at a 0-based rank r < j };
  R24  fwd(i): knn(i) reordered by (detour asc, rank asc), first R entries;
  R25  rev(c): every (p, i) with fwd(i)[p] == c, ordered by (p asc, i asc);
  R26  nbr(c): the first R/2 entries of fwd(c); then rev(c) ids not yet present, in order,
       up to R; then the remaining fwd(c) entries not yet present, up to R;
  R27  search(q, L, w, E, T): the list holds at most L (score, id) entries in c1 order with
       an "expanded" mark; the visited set starts as the entry ids; entries are scored and
       the list is the top-L of them.  Repeat at most T times: take the first w unexpanded
       list entries (stop if there are none), mark them expanded, collect their neighbours
       not yet visited (mark visited), score them and keep the top-L of list + new ones.
       Result: the first k list entries, padded (-1, -inf).
  R34  search_fp8: R27 with every score taken on the e4m3 values of oracle/fp8.py (R30
       corpus, R31 query), then the final list's L entries re-scored on the bf16 values; the
       k best (score desc, id asc), padded.

Scores are fp64 dot products of the stored bf16 values (numpy matmul as a library step).
Graph-building steps R23-R26 are integer logic on the kNN lists.
"""
from __future__ import annotations

import numpy as np

from . import bf16_to_f64


def knn(X_bits: np.ndarray, K: int, candidates=None) -> np.ndarray:
    """R22.  Returns int64 [n, K] (padded -1 when fewer than K candidates)."""
    X = bf16_to_f64(X_bits)
    n = X.shape[0]
    out = np.full((n, K), -1, dtype=np.int64)
    for i in range(n):
        cand = np.arange(n) if candidates is None else np.asarray(candidates[i], dtype=np.int64)
        cand = cand[cand != i]
        s = X[cand] @ X[i]
        order = np.lexsort((cand, -s))[:K]
        out[i, :order.size] = cand[order]
    return out


def prune(knn_lists: np.ndarray, R: int) -> np.ndarray:
    """R23 + R24.  knn_lists int64 [n, K] (-1 padded) -> fwd int64 [n, R] (-1 padded)."""
    n, K = knn_lists.shape
    rank_of = [dict() for _ in range(n)]
    for i in range(n):
        for r, c in enumerate(knn_lists[i]):
            if c >= 0:
                rank_of[i][int(c)] = r
    fwd = np.full((n, R), -1, dtype=np.int64)
    for i in range(n):
        lst = [int(c) for c in knn_lists[i] if c >= 0]
        det = []
        for j, cj in enumerate(lst):
            cnt = 0
            for k in range(j):
                r = rank_of[lst[k]].get(cj)
                if r is not None and r < j:
                    cnt += 1
            det.append((cnt, j, cj))
        det.sort()
        keep = [c for _, _, c in det[:R]]
        fwd[i, :len(keep)] = keep
    return fwd


def reverse_merge(fwd: np.ndarray) -> np.ndarray:
    """R25 + R26.  fwd int64 [n, R] -> final neighbour lists int64 [n, R] (-1 padded)."""
    n, R = fwd.shape
    rev = [[] for _ in range(n)]
    for i in range(n):
        for p, c in enumerate(fwd[i]):
            if c >= 0:
                rev[int(c)].append((p, i))
    out = np.full((n, R), -1, dtype=np.int64)
    for c in range(n):
        f = [int(x) for x in fwd[c] if x >= 0]
        lst = f[:R // 2]
        seen = set(lst)
        for _, i in sorted(rev[c]):
            if len(lst) >= R:
                break
            if i not in seen:
                lst.append(i)
                seen.add(i)
        for x in f[R // 2:]:
            if len(lst) >= R:
                break
            if x not in seen:
                lst.append(x)
                seen.add(x)
        out[c, :len(lst)] = lst
    return out


def build(X_bits: np.ndarray, K: int, R: int, candidates=None):
    kn = knn(X_bits, K, candidates)
    return reverse_merge(prune(kn, R)), kn


def search(X_bits: np.ndarray, nbr: np.ndarray, q_bits: np.ndarray, k: int, L: int, w: int,
           entries, T: int, tau=None, window: int = 1, g: int = 1, ready=True, values=None,
           qv=None):
    """R27 for one query.  Returns dict(ids, scores, expanded, iterations, certified[, rq, ema]).

    certified (diagnostic for parity tests, not part of R27): True when every order decision
    the trajectory took -- the top-L truncations, the choice of the w entries to expand, and
    the order / k-th boundary of the result -- separates two scores by more than the sum of
    their fp32 accumulation error bounds, eb = (d - 1) * 2^-24 * sum_j |q_j x_j| (bf16
    products are exact in fp32; the bound holds for any summation order).  A search that
    scores in fp32 then provably takes the same path and returns the same list; when False
    the two may legitimately differ at a near-tie.  `near_tie` holds the smallest such gap.

    With tau set, the non-stall maturity exit of PAPER.md §3.3 (App. B.2) runs on
    the beam search itself -- the paper's own setting (HNSW).  Readings R28-R29: a step is
    one iteration (w expansions); after its new rows are merged, s_t = the best score among
    the rows scored in the step (none -> RQ = 1), RQ_t = (s_best - s_t)/(s_best - s_worst)
    over the list's first / last entries (1 if equal), EMA as R17 (alpha = 2/(window+1),
    seeded with RQ_1); after every g-th step the search stops if EMA >= tau and the engine is
    ready (ready(t) or a constant); the result is the list at that point (R19).
    values / qv: fp64 rows / query to score with instead of the bf16 ones (R34)."""
    X = bf16_to_f64(X_bits) if values is None else values
    q = bf16_to_f64(q_bits) if qv is None else qv
    u_d = (X.shape[1] - 1) * 2.0 ** -24
    cert = {"ok": True, "gap": np.inf}

    def bound(rows):
        return u_d * (np.abs(X[rows]) @ np.abs(q))

    def separate(a, b):   # a, b: list entries [score, id, expanded, error bound]
        if a[1] == b[1]:
            return
        gap = abs(a[0] - b[0])
        if gap <= a[3] + b[3]:
            cert["ok"] = False
            cert["gap"] = min(cert["gap"], gap)

    visited = set()
    ent = []
    for e in entries:
        if e >= 0 and e not in visited:
            visited.add(int(e))
            ent.append(int(e))
    ids = np.array(ent, dtype=np.int64)
    sc = X[ids] @ q if ids.size else np.empty(0)
    eb = bound(ids) if ids.size else np.empty(0)
    order = np.lexsort((ids, -sc))
    if order.size > L:
        separate([sc[order[L - 1]], ids[order[L - 1]], 0, eb[order[L - 1]]],
                 [sc[order[L]], ids[order[L]], 0, eb[order[L]]])
    lst = [[float(sc[o]), int(ids[o]), False, float(eb[o])] for o in order[:L]]
    it = 0
    expanded = 0
    ema = None
    rqs, emas = [], []
    while it < T:
        unexp = [e for e in lst if not e[2]]
        pick = unexp[:w]
        if not pick:
            break
        if len(unexp) > w:
            separate(unexp[w - 1], unexp[w])
        it += 1
        new = []
        for e in pick:
            e[2] = True
            expanded += 1
            for c in nbr[e[1]]:
                c = int(c)
                if c >= 0 and c not in visited:
                    visited.add(c)
                    new.append(c)
        s_t = None
        if new:
            nid = np.array(new, dtype=np.int64)
            ns = X[nid] @ q
            s_t = float(ns.max())
            allv = lst + [[float(s), int(i), False, float(b)]
                          for s, i, b in zip(ns, nid, bound(nid))]
            allv.sort(key=lambda e: (-e[0], e[1]))
            if len(allv) > L:
                separate(allv[L - 1], allv[L])
            lst = allv[:L]
        if tau is not None:
            sb, sw = lst[0][0], lst[-1][0]
            r = 1.0 if (s_t is None or sb == sw) else (sb - s_t) / (sb - sw)
            a = 2.0 / (window + 1)
            ema = r if ema is None else a * r + (1.0 - a) * ema
            rqs.append(r)
            emas.append(ema)
            is_ready = ready(it) if callable(ready) else bool(ready)
            if it % g == 0 and ema >= tau and is_ready:
                break
    for j in range(min(k + 1, len(lst)) - 1):
        separate(lst[j], lst[j + 1])      # result order and its k-th boundary
    out_ids = np.full(k, -1, dtype=np.int64)
    out_sc = np.full(k, -np.inf)
    for j, e in enumerate(lst[:k]):
        out_ids[j] = e[1]
        out_sc[j] = e[0]
    out = {"ids": out_ids, "scores": out_sc, "expanded": expanded, "iterations": it,
           "list_ids": np.array([e[1] for e in lst], dtype=np.int64),
           "certified": cert["ok"], "near_tie": cert["gap"]}
    if tau is not None:
        out["rq"] = np.array(rqs)
        out["ema"] = np.array(emas)
    return out


def search_fp8(X_bits: np.ndarray, nbr: np.ndarray, q_bits: np.ndarray, k: int, L: int, w: int,
               entries, T: int, X8=None):
    """R34 for one query.  X8: oracle.fp8.quantize_corpus(X_bits)[0] (computed if None)."""
    from . import fp8
    if X8 is None:
        X8 = fp8.quantize_corpus(X_bits)[0]
    q8 = fp8.quantize_queries(np.asarray(q_bits)[None, :])[0][0]
    r = search(X_bits, nbr, q_bits, L, L, w, entries, T, values=X8, qv=q8)
    cand = r["list_ids"]
    Xc, qf = bf16_to_f64(X_bits[cand]), bf16_to_f64(q_bits)
    s = Xc @ qf if cand.size else np.empty(0)
    order = np.lexsort((cand, -s))
    # certification of the re-rank's order / k-th boundary (see search)
    eb = (X_bits.shape[1] - 1) * 2.0 ** -24 * (np.abs(Xc) @ np.abs(qf)) if cand.size else s
    cert, gap = r["certified"], r["near_tie"]
    for j in range(min(k + 1, order.size) - 1):
        a, b = order[j], order[j + 1]
        if abs(s[a] - s[b]) <= eb[a] + eb[b]:
            cert, gap = False, min(gap, abs(s[a] - s[b]))
    order = order[:k]
    out_ids = np.full(k, -1, dtype=np.int64)
    out_sc = np.full(k, -np.inf)
    out_ids[:order.size] = cand[order]
    out_sc[:order.size] = s[order]
    return {"ids": out_ids, "scores": out_sc, "expanded": r["expanded"],
            "iterations": r["iterations"], "list_ids": cand, "certified": cert,
            "near_tie": gap}

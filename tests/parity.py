"""Band-rule parity checker (DESIGN.md §2 "parity rule").

Compares a library result (ids int64 [nq,k], fp32 scores [nq,k]) against the
fp64 oracle.  tol(s) = rtol * max(|s|, 1e-3) with rtol = 1e-3 (BASELINE.json
north_star: "except where oracle scores at the k-th boundary differ by less
than 1e-3 relative").  With s_k the oracle's k-th score:

  must-include   every oracle id with s > s_k + tol(s_k) is returned
  must-exclude   every returned id has oracle score >= s_k - tol(s_k)
  order          returned list is strictly ordered by (gpu score desc, id asc)
                 and oracle scores are non-increasing up to tol
  scores         |gpu - oracle| <= tol(oracle) for every returned id
  padding        slots beyond the available candidates are (-1, -inf)

When no oracle score lies inside the band this is exact set and order
equality.  `rtol=1e-5` gives the sharper diagnostic band.
"""
from __future__ import annotations

import numpy as np


def tol_of(s, rtol):
    return rtol * np.maximum(np.abs(s), 1e-3)


def check(gpu_ids, gpu_scores, or_ids, or_scores, score_of, k, rtol=1e-3, n_avail=None):
    """score_of(qi, ids) -> oracle fp64 scores of those ids for query qi.

    or_ids/or_scores: oracle top-kk (kk >= k) per query, sorted, padded.
    n_avail: number of candidates per query (defaults: count of valid oracle ids, capped).
    Returns a dict report; report["ok"] is the verdict.
    """
    gpu_ids = np.asarray(gpu_ids)
    gpu_scores = np.asarray(gpu_scores, dtype=np.float64)
    nq = gpu_ids.shape[0]
    fails = []
    band_sizes = []
    max_rel = 0.0
    for qi in range(nq):
        oi, os_ = or_ids[qi], or_scores[qi]
        valid = oi >= 0
        navail = int(valid.sum()) if n_avail is None else int(min(n_avail, k))
        navail = min(navail, k)
        gi, gs = gpu_ids[qi], gpu_scores[qi]
        # padding
        if not np.all(gi[navail:] == -1) or not np.all(np.isneginf(gs[navail:])):
            fails.append((qi, "padding", gi[navail:].tolist()))
            continue
        gi, gs = gi[:navail], gs[:navail]
        if navail == 0:
            band_sizes.append(0)
            continue
        if np.any(gi < 0):
            fails.append((qi, "missing", gi.tolist()))
            continue
        if len(set(gi.tolist())) != navail:
            fails.append((qi, "duplicate ids", gi.tolist()))
            continue
        sk = os_[navail - 1]
        t = tol_of(sk, rtol)
        band_sizes.append(int(np.sum(np.abs(os_[valid] - sk) <= t)))
        # must-include
        must = set(oi[valid][os_[valid] > sk + t].tolist())
        miss = must - set(gi.tolist())
        if miss:
            fails.append((qi, "must-include", sorted(miss)))
        # oracle scores of returned ids
        s_or = np.asarray(score_of(qi, gi), dtype=np.float64)
        bad = gi[s_or < sk - t]
        if bad.size:
            fails.append((qi, "must-exclude", bad.tolist()))
        # scores
        rel = np.abs(gs - s_or) / np.maximum(np.abs(s_or), 1e-3)
        max_rel = max(max_rel, float(rel.max()))
        if np.any(np.abs(gs - s_or) > tol_of(s_or, rtol)):
            fails.append((qi, "score", float(rel.max())))
        # order: strict (score desc, id asc) on the gpu's own fp32 scores
        for j in range(navail - 1):
            if gs[j] < gs[j + 1] or (gs[j] == gs[j + 1] and gi[j] >= gi[j + 1]):
                fails.append((qi, "order", j))
                break
        # order vs oracle outside near-tie groups
        for j in range(navail - 1):
            if s_or[j] < s_or[j + 1] - tol_of(s_or[j + 1], rtol):
                fails.append((qi, "oracle-order", j))
                break
    return {
        "ok": not fails,
        "fails": fails[:20],
        "n_fail_queries": len({f[0] for f in fails}),
        "band_median": float(np.median(band_sizes)) if band_sizes else 0.0,
        "band_max": int(max(band_sizes)) if band_sizes else 0,
        "max_rel_score_err": max_rel,
    }


def check_against_rows(gpu_ids, gpu_scores, X_bits, Q_bits, k, kk_extra=16, rtol=1e-3):
    """Full check on a corpus small enough to hold on the host."""
    import oracle
    n = X_bits.shape[0]
    or_ids, or_scores = oracle.flat_topk(X_bits, Q_bits, min(k + kk_extra, max(n, 1)) if n else k)

    def score_of(qi, ids):
        return oracle.pair_scores(X_bits, Q_bits, np.full(len(ids), qi), ids)

    return check(gpu_ids, gpu_scores, or_ids, or_scores, score_of, k, rtol=rtol,
                 n_avail=min(n, k))

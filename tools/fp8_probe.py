"""tools/fp8_probe.py -- the fp8 flat scan + bf16 re-rank on the C3 corpus (or --n rows):
q/s and recall@10 against the exact bf16 mode per n_cand, for ncu captures.  One JSON line.

  python tools/fp8_probe.py [--n 21015324] [--nq 512] [--cands 16,32] [--reps 5]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2505_12065_b200 as sa  # noqa: E402
from datagen import CONFIGS, CORPUS_SEED, QUERY_SEED, make_mixture, draw_rows_into  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=CONFIGS["c3"]["n"])
    ap.add_argument("--nq", type=int, default=512)
    ap.add_argument("--cands", default="16")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--no-exact", action="store_true", help="skip the exact reference run")
    args = ap.parse_args()
    cfg = dict(CONFIGS["c3"])
    n, d, nq = args.n, cfg["d"], args.nq
    mix = make_mixture(d, cfg["C"], cfg["r"], cfg["s_sub"], cfg["s_n"], CORPUS_SEED, "cuda")
    X = torch.empty(n, d, dtype=torch.bfloat16, device="cuda")
    draw_rows_into(mix, X, CORPUS_SEED, 0)
    idx = sa.Index.build(X, 0)
    del X
    idx.build_fp8()
    Q = torch.empty(nq, d, dtype=torch.bfloat16, device="cuda")
    draw_rows_into(mix, Q, QUERY_SEED, 0)
    gt = None if args.no_exact else idx.search(Q, 10, 0)[0]
    out = {"n": n, "nq": nq, "rows": []}
    for c in (int(x) for x in args.cands.split(",")):
        for _ in range(2):
            idx.search_fp8(Q, 10, c)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            ids, _ = idx.search_fp8(Q, 10, c)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        r = {"n_cand": c, "ms": ms, "qps": nq / (ms / 1e3)}
        if gt is not None:
            g, t = ids.cpu().numpy(), gt.cpu().numpy()
            r["recall"] = float(np.mean([len(set(g[i]) & set(t[i])) / 10 for i in range(nq)]))
        out["rows"].append(r)
    print(json.dumps(out))
    idx.free()


if __name__ == "__main__":
    main()

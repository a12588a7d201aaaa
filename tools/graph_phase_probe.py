"""tools/graph_phase_probe.py -- where a beam-search CTA spends its time (tuning library only:
SA_LIBRARY=tuning, SA_GRAPH_DBG): per query the globaltimer start/end and thread 0's clock64
cycles in merge / pick / expand / score (each up to its closing barrier), on the C3 graph at the
bench setting.  Prints a summary: start/end spread (the tail), phase shares, iterations.

  SA_LIBRARY=tuning python tools/graph_phase_probe.py [--n 21015324] [--L 100] [--nq 512]
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
    ap.add_argument("--L", default="100")
    ap.add_argument("--nq", type=int, default=512)
    ap.add_argument("--pf", default="0")
    args = ap.parse_args()
    assert sa.TUNING, "needs SA_LIBRARY=tuning"
    cfg = dict(CONFIGS["c3"])
    n, d = args.n, cfg["d"]
    mix = make_mixture(d, cfg["C"], cfg["r"], cfg["s_sub"], cfg["s_n"], CORPUS_SEED, "cuda")
    X = torch.empty(n, d, dtype=torch.bfloat16, device="cuda")
    draw_rows_into(mix, X, CORPUS_SEED, 0)
    idx = sa.Index.build(X, 16384)
    del X
    torch.cuda.empty_cache()
    idx.build_graph(knn_k=64, degree=48, nprobe_build=8)
    Q = torch.empty(args.nq, d, dtype=torch.bfloat16, device="cuda")
    draw_rows_into(mix, Q, QUERY_SEED, 0)
    dbg = torch.zeros(args.nq, 8, dtype=torch.int64, device="cuda")
    os.environ["SA_GRAPH_PF"] = args.pf
    for L in [int(x) for x in args.L.split(",")]:
        for _ in range(3):
            idx.search_graph(Q, 10, L, search_width=4, n_entries=16)
        torch.cuda.synchronize()
        os.environ["SA_GRAPH_DBG"] = str(dbg.data_ptr())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        idx.search_graph(Q, 10, L, search_width=4, n_entries=16)
        e1.record()
        torch.cuda.synchronize()
        del os.environ["SA_GRAPH_DBG"]
        D = dbg.cpu().numpy().astype(np.float64)
        t0 = D[:, 0].min()
        st, en = (D[:, 0] - t0) / 1e3, (D[:, 1] - t0) / 1e3   # us
        cyc = D[:, 2:6]
        tot = cyc.sum(1)
        dur = en - st
        out = {"L": L, "call_ms": e0.elapsed_time(e1), "kernel_span_us": float(en.max()),
               "start_us_p50_max": [float(np.median(st)), float(st.max())],
               "end_us_min_p10_p50_p90_max": [float(np.percentile(en, p)) for p in (0, 10, 50, 90, 100)],
               "cta_dur_us_mean_max": [float(dur.mean()), float(dur.max())],
               "phase_share_merge_pick_expand_score": [float(x) for x in (cyc.sum(0) / tot.sum())],
               "ghz_est": float(tot.sum() / (dur.sum() * 1e3)),
               "iters_mean_max": [float(D[:, 6].mean()), float(D[:, 6].max())],
               "us_per_iter": float(dur.mean() / D[:, 6].mean())}
        print(json.dumps(out), flush=True)
    idx.free()


if __name__ == "__main__":
    main()

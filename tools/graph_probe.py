"""tools/graph_probe.py -- graph index build time, recall@10 and q/s per search range on the
C3 corpus (or --n rows).  One JSON line.

  python tools/graph_probe.py [--n 21015324] [--knn 64] [--degree 32] [--nprobe-build 8]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2505_12065_b200 as sa  # noqa: E402
from datagen import CONFIGS, CORPUS_SEED, QUERY_SEED, make_mixture, draw_rows_into  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=CONFIGS["c3"]["n"])
    ap.add_argument("--nlist", type=int, default=16384)
    ap.add_argument("--knn", type=int, default=64)
    ap.add_argument("--degree", type=int, default=32)
    ap.add_argument("--nprobe-build", type=int, default=8)
    ap.add_argument("--nq", type=int, default=512)
    ap.add_argument("--ranges", default="16,32,48,64,96,128,192,256")
    ap.add_argument("--widths", default="1,2,4")
    ap.add_argument("--entries", default="8")
    ap.add_argument("--latency", action="store_true", help="also time agent-step batches")
    ap.add_argument("--fp8", default="0", help="comma list of 0/1: bf16 and/or fp8 navigation")
    ap.add_argument("--pf", default="", help="comma list of SA_GRAPH_PF values (tuning library)")
    args = ap.parse_args()
    cfg = dict(CONFIGS["c3"])
    n, d = args.n, cfg["d"]
    mix = make_mixture(d, cfg["C"], cfg["r"], cfg["s_sub"], cfg["s_n"], CORPUS_SEED, "cuda")
    X = torch.empty(n, d, dtype=torch.bfloat16, device="cuda")
    draw_rows_into(mix, X, CORPUS_SEED, 0)
    t0 = time.perf_counter()
    idx = sa.Index.build(X, args.nlist)
    torch.cuda.synchronize()
    ivf_s = time.perf_counter() - t0
    del X
    torch.cuda.empty_cache()
    t0 = time.perf_counter()
    idx.build_graph(knn_k=args.knn, degree=args.degree, nprobe_build=args.nprobe_build)
    torch.cuda.synchronize()
    graph_s = time.perf_counter() - t0
    fp8s = [int(x) for x in args.fp8.split(",")]
    if any(fp8s):
        idx.build_fp8()
    Q = torch.empty(4 * args.nq, d, dtype=torch.bfloat16, device="cuda")
    draw_rows_into(mix, Q, QUERY_SEED, 0)
    qs = [Q[i * args.nq:(i + 1) * args.nq] for i in range(4)]
    gt = [idx.search(q, 10, 0)[0].cpu().numpy() for q in qs]
    out = {"n": n, "nlist": args.nlist, "knn": args.knn, "degree": args.degree,
           "nprobe_build": args.nprobe_build, "ivf_build_s": ivf_s, "graph_build_s": graph_s,
           "nq": args.nq, "rows": []}
    stream = torch.cuda.current_stream()
    for pf, f8, E, w, L in [(pf, f8, E, w, L) for pf in (args.pf.split(",") if args.pf else [None])
                        for f8 in fp8s
                        for E in [int(x) for x in args.entries.split(",")]
                        for w in [int(x) for x in args.widths.split(",")]
                        for L in [int(x) for x in args.ranges.split(",")]]:
        if pf is not None:
            os.environ["SA_GRAPH_PF"] = pf
        if True:
            rec, exp, scd = [], [], []
            for q, t in zip(qs, gt):
                gi, _, ex, sc_rows = idx.search_graph(q, 10, L, search_width=w, n_entries=E,
                                                      expanded=True, fp8=bool(f8))
                gi = gi.cpu().numpy()
                rec.append(np.mean([len(set(gi[i]) & set(t[i])) / 10 for i in range(len(t))]))
                exp.append(ex.float().mean().item())
                scd.append(sc_rows.float().cpu().numpy())
            scd = np.concatenate(scd)
            torch.cuda.synchronize()
            reps = []
            for rep in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for i in range(8):
                    idx.search_graph(qs[i % 4], 10, L, search_width=w, n_entries=E, fp8=bool(f8))
                e1.record(stream)
                torch.cuda.synchronize()
                reps.append(e0.elapsed_time(e1) / 8)
            ms = float(np.median(reps))
            sa.profile_enable(True)
            for i in range(8):
                idx.search_graph(qs[i % 4], 10, L, search_width=w, n_entries=E, fp8=bool(f8))
            torch.cuda.synchronize()
            kern = {kd: round(sa.profile_read(kd)[0] / 8, 4) for kd in sa.KERNEL_KINDS}
            sa.profile_enable(False)
            out["rows"].append({"pf": pf, "fp8": f8, "L": L, "w": w, "E": E, "recall": float(np.mean(rec)),
                                "expanded": float(np.mean(exp)), "ms_per_batch": ms,
                                "scored_mean": float(scd.mean()),
                                "scored_p90_p99_max": [float(np.percentile(scd, 90)),
                                                       float(np.percentile(scd, 99)),
                                                       float(scd.max())],
                                "qps": args.nq / (ms / 1e3), "kernel_ms": kern})
            print(json.dumps(out["rows"][-1]), file=sys.stderr, flush=True)
    if args.latency:
        # agent-step batches: device time per call (stage + probe + search), median of 50
        out["latency"] = []
        Lr = int(args.ranges.split(",")[0])
        for b in (1, 8, 64, 148, 149):
            q = qs[0][:b].contiguous()
            ts = []
            for i in range(55):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                idx.search_graph(q, 5, Lr, search_width=int(args.widths.split(",")[0]),
                                 n_entries=16)
                e1.record(stream)
                torch.cuda.synchronize()
                if i >= 5:
                    ts.append(e0.elapsed_time(e1))
            out["latency"].append({"batch": b, "L": Lr, "p50_ms": float(np.median(ts))})
            print(json.dumps(out["latency"][-1]), file=sys.stderr, flush=True)
    print(json.dumps(out))
    idx.free()


if __name__ == "__main__":
    main()

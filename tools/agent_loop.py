"""tools/agent_loop.py -- PAPER.md Algorithm 1 (App. A.1) driving the B200
retriever, with a timing-only stand-in for the LLM engine.

The engine is NOT modelled beyond its clock: every engine step takes `--step-ms` of wall time
and advances each admitted sequence by one decode step; a request is a seeded list of
segments (decode steps, then a retrieval; the last segment answers).  What is real: the
retrieval -- queries go through sa_retriever_submit (asynchronous H2D + IVF / maturity-exit
search + D2H on the GPU), completions are polled every loop pass (Alg. 1 step 3), the
waiting queue is ordered by sa_priority_order (Eq. 1-2, G=6) before every step (line 23),
and in mode `mature` the engine-ready flag is raised while the engine has waiting sequences
(lines 10-11).  Reported per mode: retrieval latency (submit -> completion, observed
by polling during the engine step), the stall
per retrieval (result available -> the sequence's next admission, in engine steps), and
end-to-end request latency.

  python tools/agent_loop.py [--requests 64] [--step-ms 20] [--nprobe 48] [--modes exact,fixed,mature]
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
    ap.add_argument("--requests", type=int, default=64)
    ap.add_argument("--batch", type=int, default=32, help="max sequences per engine step")
    ap.add_argument("--step-ms", type=float, default=20.0)
    ap.add_argument("--nprobe", type=int, default=48)
    ap.add_argument("--k", type=int, default=5)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--modes", default="fixed,mature",
                    help="comma list of: exact, fixed, mature (maturity exit + engine flag), "
                         "graph (fixed search range), graph_mature (the paper's own setting: "
                         "maturity exit on the graph beam search + engine flag)")
    ap.add_argument("--search-range", type=int, default=104)
    ap.add_argument("--graph-tau", type=float, default=0.9, help="the paper's tau (P:387)")
    args = ap.parse_args()
    cfg = dict(CONFIGS["c3"])
    n = args.n or cfg["n"]
    d = cfg["d"]
    mix = make_mixture(d, cfg["C"], cfg["r"], cfg["s_sub"], cfg["s_n"], CORPUS_SEED, "cuda")
    X = torch.empty(n, d, dtype=torch.bfloat16, device="cuda")
    draw_rows_into(mix, X, CORPUS_SEED, 0)
    idx = sa.Index.build(X, 16384 if n > 1_000_000 else 1024)
    del X
    torch.cuda.empty_cache()
    if any(m.startswith("graph") for m in args.modes.split(",")):
        idx.build_graph(knn_k=64, degree=48, nprobe_build=8)
    g = np.random.default_rng(2505)
    # request traces: 1-5 retrievals (P:236-238 report ~2.3-3.3 per request), 20-60 steps each
    traces = []
    for i in range(args.requests):
        nret = int(g.integers(1, 6))
        traces.append([int(s) for s in g.integers(20, 61, nret + 1)])
    nq_total = sum(len(t) - 1 for t in traces)
    Q = torch.empty(nq_total, d, dtype=torch.bfloat16, device="cuda")
    draw_rows_into(mix, Q, QUERY_SEED, 0)
    Qh = Q.float().cpu().numpy()

    out = {"n": n, "requests": args.requests, "step_ms": args.step_ms, "nprobe": args.nprobe,
           "modes": {}}
    for mode in args.modes.split(","):
        r = sa.Retriever(idx, streams=4, slots=64, max_nq=1, max_k=args.k)
        qnext = 0
        t0 = time.perf_counter()
        # per request: segment index, remaining steps, state, counters
        st = [{"seg": 0, "left": tr[0], "state": "waiting", "R": 0, "ctx": 512,
               "t_arr": 0.0, "t_ready": 0.0, "q": None} for tr in traces]
        active = {}                      # task -> request
        ret_lat, stall_steps, e2e = [], [], {}
        steps = 0
        while len(e2e) < len(traces):
            now = time.perf_counter() - t0
            waiting = [i for i, s in enumerate(st) if s["state"] == "waiting"]
            if mode in ("mature", "graph_mature"):   # Alg. 1 lines 10-11: engine has waiting
                r.set_engine_ready(bool(waiting) and bool(active))
            for task, i in list(active.items()):          # step 3: completed searches
                if r.poll(task):
                    r.result(task)
                    s = st[i]
                    t_fin = s.pop("t_fin", time.perf_counter() - t0)
                    ret_lat.append(t_fin - s["t_sub"])
                    s.update(state="waiting", t_ready=time.perf_counter() - t0, R=s["R"] + 1,
                             ctx=s["ctx"] + args.k * 100, done_step=steps)
                    del active[task]
            waiting = [i for i, s in enumerate(st) if s["state"] == "waiting"]
            if waiting:                                    # line 23: priority scheduling
                now = time.perf_counter() - t0
                us = lambda x: int(x * 1e6)  # noqa: E731
                order, _ = sa.sa_priority_order([st[i]["R"] for i in waiting],
                                                [us(now - st[i]["t_arr"]) for i in waiting],
                                                [st[i]["ctx"] for i in waiting],
                                                [us(now - st[i]["t_ready"]) for i in waiting],
                                                waiting, 6)
                batch = [waiting[j] for j in order[:args.batch]]
            else:
                batch = []
            # engine step (timing stand-in)
            t_step = time.perf_counter()
            while time.perf_counter() - t_step < args.step_ms / 1e3:
                for task, i in active.items():             # completion timestamps only
                    if "t_fin" not in st[i] and r.poll(task):
                        st[i]["t_fin"] = time.perf_counter() - t0
            steps += 1
            for i in batch:
                s = st[i]
                if "done_step" in s:
                    stall_steps.append(steps - 1 - s.pop("done_step"))
                s["left"] -= 1
                s["ctx"] += 1
                if s["left"] > 0:
                    continue
                s["seg"] += 1
                if s["seg"] == len(traces[i]):             # <answer>
                    s["state"] = "done"
                    e2e[i] = time.perf_counter() - t0
                    continue
                s["left"] = traces[i][s["seg"]]            # <search>: async retrieval
                s["state"] = "retrieving"
                s["t_sub"] = time.perf_counter() - t0
                q = Qh[qnext:qnext + 1]
                qnext += 1
                if mode == "exact":
                    task = r.submit(q, args.k, 0)
                elif mode == "fixed":
                    task = r.submit(q, args.k, args.nprobe)
                elif mode == "graph":
                    task = r.submit_graph(q, args.k, args.search_range)
                elif mode == "graph_mature":
                    task = r.submit_graph(q, args.k, 256, mature=True, tau=args.graph_tau,
                                          window=4, check_every=1)
                else:
                    task = r.submit(q, args.k, 128, mature=True, tau=3.0, window=32,
                                    check_every=8)
                active[task] = i
        r.free()
        out["modes"][mode] = {
            "engine_steps": steps,
            "retrieval_ms_p50": 1e3 * float(np.percentile(ret_lat, 50)),
            "retrieval_ms_p99": 1e3 * float(np.percentile(ret_lat, 99)),
            "stall_steps_mean": float(np.mean(stall_steps)) if stall_steps else 0.0,
            "stalled_fraction": float(np.mean(np.array(stall_steps) > 0)) if stall_steps else 0.0,
            "e2e_s_mean": float(np.mean(list(e2e.values()))),
            "retrievals": len(ret_lat)}
    print(json.dumps(out))
    idx.free()


if __name__ == "__main__":
    main()

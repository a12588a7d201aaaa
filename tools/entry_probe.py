"""tools/entry_probe.py -- the graph search's entry-point probe (the E best IVF lists per query:
score dump on the tensor cores + exact select) against the flat kernel's fused top-k mode over
the same centroids (a flat index built from them), and the kernel split, at nq = 512, E = 16,
nlist = 16384, d = 768.

  python tools/entry_probe.py [--n 2000000]
"""
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


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2_000_000)
    ap.add_argument("--nq", type=int, default=512)
    ap.add_argument("--E", type=int, default=16)
    args = ap.parse_args()
    cfg = CONFIGS["c3"]
    d = cfg["d"]
    mix = make_mixture(d, cfg["C"], cfg["r"], cfg["s_sub"], cfg["s_n"], CORPUS_SEED, "cuda")
    X = torch.empty(args.n, d, dtype=torch.bfloat16, device="cuda")
    draw_rows_into(mix, X, CORPUS_SEED, 0)
    idx = sa.Index.build(X, 16384, kmeans_iters=4)
    C = torch.from_numpy(idx.export_centroids()).cuda().to(torch.bfloat16).contiguous()
    cflat = sa.Index.build(C)
    Q = torch.empty(args.nq, d, dtype=torch.bfloat16, device="cuda")
    draw_rows_into(mix, Q, QUERY_SEED, 0)
    out = {"nq": args.nq, "E": args.E, "nlist": C.shape[0]}
    torch.cuda.nvtx.range_push("probe")
    out["probe_dump_select_ms"] = timeit(lambda: idx.probes(Q, args.E))
    torch.cuda.nvtx.range_pop()
    torch.cuda.nvtx.range_push("flat")
    out["flat_topk_ms"] = timeit(lambda: cflat.search(Q, args.E))
    torch.cuda.nvtx.range_pop()
    sa.profile_enable(True)
    for _ in range(10):
        idx.probes(Q, args.E)
    torch.cuda.synchronize()
    out["probe_kernels_ms"] = {k: round(sa.profile_read(k)[0] / 10, 4) for k in sa.KERNEL_KINDS
                               if sa.profile_read(k)[1]}
    sa.profile_enable(False)
    sa.profile_enable(True)
    for _ in range(10):
        cflat.search(Q, args.E)
    torch.cuda.synchronize()
    out["flat_kernels_ms"] = {k: round(sa.profile_read(k)[0] / 10, 4) for k in sa.KERNEL_KINDS
                              if sa.profile_read(k)[1]}
    sa.profile_enable(False)
    a = idx.probes(Q, args.E).cpu().numpy()
    b = cflat.search(Q, args.E)[0].cpu().numpy()
    out["same_sets"] = float(np.mean([set(x) == set(y) for x, y in zip(a, b)]))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

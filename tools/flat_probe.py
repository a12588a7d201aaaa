"""Timing probe of the exact flat scan at one shape (tuning experiments; not a benchmark).

  SA_LIBRARY=tuning SA_EXPERIMENT=1 python tools/flat_probe.py --n 1000000 --nq 256

Prints one JSON line: mean ms per search, the flat-scan kernel's mean ms, and the TFLOP/s
that implies.  With the tuning library (build.py --tuning) the timing switches apply
(SA_EXPERIMENT 1: skip score processing, 3: 64-way max only; SA_SEED_ROWS: seed the pruning
bound from that many rows).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2505_12065_b200 as sa  # noqa: E402
from datagen import CORPUS_SEED, QUERY_SEED, draw_rows_into, make_mixture  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--d", type=int, default=768)
    ap.add_argument("--nq", type=int, default=256)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--fp8", type=int, default=0, help="n_cand > 0: fp8 scan + re-rank")
    a = ap.parse_args()
    mix = make_mixture(a.d, 128, 32, 1.0, 0.7, CORPUS_SEED, "cuda")
    X = torch.empty(a.n, a.d, dtype=torch.bfloat16, device="cuda")
    draw_rows_into(mix, X, CORPUS_SEED, 0)
    Q = torch.empty(a.nq, a.d, dtype=torch.bfloat16, device="cuda")
    draw_rows_into(mix, Q, QUERY_SEED, 0)
    idx = sa.Index.build(X)
    if a.fp8:
        idx.build_fp8()
    run = (lambda: idx.search_fp8(Q, a.k, a.fp8)) if a.fp8 else (lambda: idx.search(Q, a.k))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    sa.profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    prof = {k: sa.profile_read(k) for k in sa.KERNEL_KINDS}
    counts = None
    if sa.TUNING and os.environ.get("COUNT"):
        cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
        os.environ["SA_FS_COUNT"] = str(cnt.data_ptr())
        run()
        torch.cuda.synchronize()
        del os.environ["SA_FS_COUNT"]
        counts = cnt.tolist()
    sa.profile_enable(False)
    ms = e0.elapsed_time(e1) / a.reps
    fs_ms, fs_n = prof["flat_scan"]
    kms = fs_ms / max(fs_n, 1)
    flop = 2.0 * a.nq * a.n * a.d
    print(json.dumps({"n": a.n, "d": a.d, "nq": a.nq, "k": a.k, "fp8": a.fp8,
                      "env": {v: os.environ[v] for v in ("SA_LIBRARY", "SA_EXPERIMENT",
                                                         "SA_SEED_ROWS", "SA_NO_SEED")
                              if v in os.environ},
                      "ms_per_search": ms, "flat_kernel_ms": kms,
                      "counts_pass_ins_boundrounds": counts,
                      "other_ms": prof["other"][0] / a.reps,
                      "tflops_kernel": flop / (kms / 1e3) / 1e12,
                      "tflops_search": flop / (ms / 1e3) / 1e12}))
    idx.free()


if __name__ == "__main__":
    main()

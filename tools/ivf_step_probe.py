"""tools/ivf_step_probe.py -- where an IVF batch spends its time at a per-rank shard size (the
w = 8 row shard of C3 by default): ms per batch over back-to-back calls, the library's per-kind
kernel times, and an NVTX range "ivf_step" around the timed calls for an ncu launch list.

  python tools/ivf_step_probe.py [--n 2626916] [--nq 512] [--nprobe 48]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2505_12065_b200 as sa  # noqa: E402
from datagen import CONFIGS, CORPUS_SEED, QUERY_SEED, make_mixture, draw_rows_into  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2_626_916)
    ap.add_argument("--nq", type=int, default=512)
    ap.add_argument("--nprobe", type=int, default=48)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    cfg = CONFIGS["c3"]
    d = cfg["d"]
    mix = make_mixture(d, cfg["C"], cfg["r"], cfg["s_sub"], cfg["s_n"], CORPUS_SEED, "cuda")
    X = torch.empty(args.n, d, dtype=torch.bfloat16, device="cuda")
    draw_rows_into(mix, X, CORPUS_SEED, 0)
    idx = sa.Index.build(X, 16384)
    del X
    Q = torch.empty(args.nq, d, dtype=torch.bfloat16, device="cuda")
    draw_rows_into(mix, Q, QUERY_SEED, 0)
    for _ in range(3):
        idx.search(Q, 10, args.nprobe)
    torch.cuda.synchronize()
    sa.profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.nvtx.range_push("ivf_step")
    e0.record()
    for _ in range(args.reps):
        idx.search(Q, 10, args.nprobe)
    e1.record()
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    prof = {k: sa.profile_read(k) for k in sa.KERNEL_KINDS}
    sa.profile_enable(False)
    print(json.dumps({"n": args.n, "nq": args.nq, "nprobe": args.nprobe,
                      "ms_per_batch": e0.elapsed_time(e1) / args.reps,
                      "kernel_ms": {k: round(v[0] / args.reps, 4) for k, v in prof.items() if v[1]},
                      "launches": {k: v[1] / args.reps for k, v in prof.items() if v[1]}}))
    idx.free()


if __name__ == "__main__":
    main()

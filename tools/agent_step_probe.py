"""Per-kernel picture of one small-batch IVF search (agent step) on the C3 corpus.
Usage: python tools/agent_step_probe.py [batch] [nprobe]   (run under ncu for a launch list)"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_12065_b200 as sa  # noqa: E402
from datagen import CONFIGS, CORPUS_SEED, QUERY_SEED, make_mixture, draw_rows_into  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 1
nprobe = int(sys.argv[2]) if len(sys.argv) > 2 else 48
cfg = CONFIGS["c3"]
mix = make_mixture(cfg["d"], cfg["C"], cfg["r"], cfg["s_sub"], cfg["s_n"], CORPUS_SEED, "cuda")
X = torch.empty(cfg["n"], cfg["d"], dtype=torch.bfloat16, device="cuda")
draw_rows_into(mix, X, CORPUS_SEED, 0)
idx = sa.Index.build(X, 16384)
del X
Q = torch.empty(64, cfg["d"], dtype=torch.bfloat16, device="cuda")
draw_rows_into(mix, Q, QUERY_SEED, 0)
qh = Q[:b].float().cpu().pin_memory()
for _ in range(10):
    idx.search_host(qh, 5, nprobe)
ts = []
for _ in range(50):
    t0 = time.perf_counter()
    idx.search_host(qh, 5, nprobe)
    ts.append(time.perf_counter() - t0)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("agent")
for _ in range(3):
    idx.search_host(qh, 5, nprobe)
torch.cuda.nvtx.range_pop()
print(f"batch {b} nprobe {nprobe}: p50 {1e3*np.median(ts):.3f} ms  p99 {1e3*np.percentile(ts, 99):.3f} ms")

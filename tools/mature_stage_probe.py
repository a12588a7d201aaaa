"""Per-stage timeline of the one-launch maturity-exit search on the C3 IVF index (debug
timestamps, sa_debug_mature_stages).  Usage: python tools/mature_stage_probe.py [batch] [g]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_12065_b200 as sa  # noqa: E402
from datagen import CONFIGS, CORPUS_SEED, QUERY_SEED, make_mixture, draw_rows_into  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 1
g = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = CONFIGS["c3"]
mix = make_mixture(cfg["d"], cfg["C"], cfg["r"], cfg["s_sub"], cfg["s_n"], CORPUS_SEED, "cuda")
X = torch.empty(cfg["n"], cfg["d"], dtype=torch.bfloat16, device="cuda")
draw_rows_into(mix, X, CORPUS_SEED, 0)
idx = sa.Index.build(X, 16384)
del X
Q = torch.empty(64, cfg["d"], dtype=torch.bfloat16, device="cuda")
draw_rows_into(mix, Q, QUERY_SEED, 0)
Qd = Q[:b].contiguous()
for rep in range(4):
    _, _, t, ns = idx.debug_mature_stages(Qd, 5, 32, tau=float("inf"), window=8, check_every=g)
nst = (32 + g - 1) // g
st = ns[:nst]
t0 = st[0, 0]
print(f"batch {b}, g {g}: {nst} stages, total {(st[nst - 1, 3] - t0) / 1e3:.1f} us from the first stage start")
for i in range(nst):
    a0, a1, a2, a3 = (st[i] - t0) / 1e3
    print(f"  stage {i:2d}: start {a0:7.1f}  CTA0 scan done +{a1 - a0:5.1f}  last arrival "
          f"+{a2 - a0:5.1f}  release +{a3 - a0:5.1f}  (closure {a3 - a2:4.1f})")

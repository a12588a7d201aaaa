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
if b <= 8:
    # device-side phase breakdown of the one-launch path (per-CTA %globaltimer stamps)
    Qd = Q[:b].contiguous()
    rows = []
    for _ in range(20):
        _, _, ns = idx.debug_small_phases(Qd, 5, nprobe)
        t0 = ns[:, 0].min()
        last = ns[:, 5].max()
        rows.append([ns[:, 0].max() - t0, np.median(ns[:, 6] - t0), np.median(ns[:, 7] - ns[:, 3]),
                     np.median(ns[:, 1] - t0), ns[:, 1].max() - t0, ns[:, 2].max() - t0,
                     np.median(ns[:, 3] - t0), ns[:, 3].max() - t0, np.median(ns[:, 4] - t0),
                     ns[:, 4].max() - t0, last - t0])
    r = np.median(np.array(rows), axis=0) / 1e3
    print(f"batch {b} phases (us from the first CTA start, median of 20): start spread {r[0]:.1f} | "
          f"first centroid piece {r[1]:.1f} | A med {r[3]:.1f} max {r[4]:.1f} | B fast max {r[5]:.1f} "
          f"| probes known med {r[6]:.1f} max {r[7]:.1f} (first list piece +{r[2]:.1f}) | scan done "
          f"med {r[8]:.1f} max {r[9]:.1f} | final merge {r[10]:.1f}")
# device-path timing: CUDA events around each call (bf16 queries already on the device)
Qd = Q[:b].contiguous()
for _ in range(5):
    idx.search(Qd, 5, nprobe)
st = torch.cuda.current_stream()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(30)]
for e0, e1 in ev:
    e0.record(st)
    idx.search(Qd, 5, nprobe)
    e1.record(st)
    torch.cuda.synchronize()
one = sorted(e0.elapsed_time(e1) for e0, e1 in ev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(50):
    idx.search(Qd, 5, nprobe)
e1.record(st)
torch.cuda.synchronize()
print(f"batch {b} device path: one call (events, synced) p50 {1e3 * one[15]:.1f} us; "
      f"50 back-to-back {1e3 * e0.elapsed_time(e1) / 50:.1f} us per call")
# host path: GPU span of the replayed graph (events around it on the same stream) vs wall time
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(30)]
wall = []
for e0, e1 in ev:
    e0.record(st)
    t0 = time.perf_counter()
    idx.search_host(qh, 5, nprobe, stream=st)
    wall.append(time.perf_counter() - t0)
    e1.record(st)
    torch.cuda.synchronize()
span = sorted(e0.elapsed_time(e1) for e0, e1 in ev)
t0 = time.perf_counter()
for _ in range(2000):
    sa.lib().sa_status_string(0)
ct = (time.perf_counter() - t0) / 2000
print(f"batch {b} host path: wall p50 {1e6 * sorted(wall)[15]:.1f} us, GPU span of the replay "
      f"p50 {1e3 * span[15]:.1f} us; one ctypes call {1e6 * ct:.2f} us")

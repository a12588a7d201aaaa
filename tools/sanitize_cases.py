"""Small invocations of every hot kernel, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck).  Usage:

  compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]

Cases: flat1 (cta_group 1, C1 shape), flat2 (cta_group 2, nq 300), flatk (k = 100, global
heaps), ivf, ivfsmall (agent-step batch), mature, graph, graph_mature, fp8, merge, host
(agent-step host-buffer calls: one-launch IVF search, persistent scratch, pinned results).
Every case checks its result against the exact mode so a sanitizer-perturbed run that
returns garbage fails loudly too.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2505_12065_b200 as sa  # noqa: E402
from datagen import make_mixture, draw_rows  # noqa: E402


def recall(a, b):
    a, b = a.cpu().tolist(), b.cpu().tolist()
    return sum(len(set(x) & set(y)) for x, y in zip(a, b)) / max(1, sum(len(y) for y in b))


def main(cases):
    torch.cuda.set_device(0)
    mix = make_mixture(d=128, C=16, r=16)
    X = draw_rows(mix, 10000, row_seed=1234).cuda().to(torch.bfloat16)
    Q = draw_rows(mix, 300, row_seed=5678).cuda().to(torch.bfloat16)
    flat = sa.Index.build(X)
    ivf = None
    gt10 = flat.search(Q, 10)[0]
    out = {}
    for c in cases:
        if c == "flat1":
            out[c] = recall(flat.search(Q[:100].contiguous(), 10)[0], gt10[:100])
        elif c == "flat2":
            out[c] = recall(flat.search(Q, 10)[0], gt10)
        elif c == "flatk":
            out[c] = recall(flat.search(Q[:64].contiguous(), 100)[0][:, :10], gt10[:64])
        elif c in ("ivf", "ivfsmall", "mature", "graph", "graph_mature", "fp8", "host"):
            if ivf is None:
                ivf = sa.Index.build(X, 64, kmeans_iters=3)
            if c == "ivf":
                out[c] = recall(ivf.search(Q, 10, 64)[0], gt10)
            elif c == "ivfsmall":
                out[c] = recall(ivf.search(Q[:4].contiguous(), 10, 64)[0], gt10[:4])
            elif c == "mature":
                ids = ivf.search_mature(Q[:8].contiguous(), 10, 64, tau=1e9, window=4)[0]
                out[c] = recall(ids, gt10[:8])
            elif c == "graph":
                ivf.build_graph(knn_k=24, degree=16, nprobe_build=4)
                out[c] = recall(ivf.search_graph(Q[:64].contiguous(), 10, 128, search_width=2,
                                                 n_entries=8)[0], gt10[:64])
            elif c == "graph_mature":
                ivf.build_graph(knn_k=24, degree=16, nprobe_build=4)
                ids = ivf.search_graph_mature(Q[:16].contiguous(), 10, 128, tau=1e9, window=4,
                                              search_width=2, n_entries=8)[0]
                out[c] = recall(ids, gt10[:16])
            elif c == "host":
                qh = Q[:8].float().cpu().contiguous()
                got = torch.cat([ivf.search_host(qh[i:i + 1].contiguous(), 10, 64)[0]
                                 for i in range(8)] + [ivf.search_host(qh, 10, 64)[0]])
                out[c] = recall(got, torch.cat([gt10[:8].cpu(), gt10[:8].cpu()]))
            elif c == "fp8":
                ivf.build_fp8()
                out[c] = recall(ivf.search_fp8(Q[:128].contiguous(), 10, 64)[0], gt10[:128])
        elif c == "merge":
            # three row shards of the corpus, their key lists merged (the sharded a9 merge)
            shards = []
            for r in range(3):
                off, ln = sa.shard_range(X.shape[0], r, 3)
                shards.append(sa.Index.build(X[off:off + ln].contiguous(), row_offset=off,
                                             n_total=X.shape[0]))
            ks = torch.stack([s.search_keys(Q[:32].contiguous(), 10) for s in shards])
            out[c] = recall(sa.sa_merge_keys(ks)[0], gt10[:32])
        torch.cuda.synchronize()
    print("sanitize cases:", out, flush=True)
    bad = {c: r for c, r in out.items() if r < (0.9 if c.startswith(("ivf", "mature", "graph"))
                                               else 0.99)}
    if bad:
        raise SystemExit(f"low recall under the sanitizer: {bad}")


if __name__ == "__main__":
    main(sys.argv[1:] or ["flat1", "flat2", "flatk", "merge", "ivf", "ivfsmall", "mature",
                          "graph", "graph_mature", "fp8", "host"])

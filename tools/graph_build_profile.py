import sys, time, json, torch
sys.path.insert(0, '.')
import paper_2505_12065_b200 as sa
from datagen import CONFIGS, CORPUS_SEED, make_mixture, draw_rows_into
cfg = CONFIGS["c3"]; n, d = cfg["n"], cfg["d"]
mix = make_mixture(d, cfg["C"], cfg["r"], cfg["s_sub"], cfg["s_n"], CORPUS_SEED, "cuda")
X = torch.empty(n, d, dtype=torch.bfloat16, device="cuda"); draw_rows_into(mix, X, CORPUS_SEED, 0)
idx = sa.Index.build(X, 16384); del X; torch.cuda.synchronize()
sa.profile_enable(True)
t0 = time.perf_counter(); idx.build_graph(knn_k=64, degree=48, nprobe_build=8); torch.cuda.synchronize()
print(json.dumps({"build_s": time.perf_counter() - t0, "kernels": {k: sa.profile_read(k) for k in sa.KERNEL_KINDS}}))

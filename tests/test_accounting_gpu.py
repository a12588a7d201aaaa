"""Kernel accounting (sa_profile_*) and the bounded captured-search caches.

Every launch is counted under the kind of the outermost open region, and every outermost
region is timed: a kind has launches exactly when it has time (the graph path
once reported flat-scan launches with 0 ms and probe time with 0 launches).
"""
import numpy as np
import pytest
import torch

from datagen import draw_rows, make_mixture

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def small_index(sa):
    mix = make_mixture(d=128, C=16, r=16)
    X = draw_rows(mix, 20000, row_seed=1234).cuda().to(torch.bfloat16)
    Q = draw_rows(mix, 300, row_seed=5678).cuda().to(torch.bfloat16)
    idx = sa.Index.build(X, 64, kmeans_iters=3)
    idx.build_graph(knn_k=24, degree=16, nprobe_build=4)
    yield idx, Q
    idx.free()


def _profile(sa, fn):
    torch.cuda.synchronize()
    sa.profile_enable(True)
    fn()
    torch.cuda.synchronize()
    out = {k: sa.profile_read(k) for k in sa.KERNEL_KINDS}
    sa.profile_enable(False)
    return out


@pytest.mark.parametrize("mode", ["exact", "ivf", "graph"])
def test_time_and_launches_agree(sa, small_index, mode):
    idx, Q = small_index
    call = {"exact": lambda: idx.search(Q, 10, 0),
            "ivf": lambda: idx.search(Q, 10, 16),
            "graph": lambda: idx.search_graph(Q, 10, 64, search_width=2, n_entries=8)}[mode]
    prof = _profile(sa, call)
    for kind, (ms, n) in prof.items():
        if kind == "other":
            continue          # OTHER also holds launches made outside any timed region
        assert (ms > 0) == (n > 0), (mode, kind, ms, n)
    main = {"exact": "flat_scan", "ivf": "ivf_scan", "graph": "graph_search"}[mode]
    assert prof[main][1] >= 1 and prof[main][0] > 0
    if mode == "graph":
        # the entry-point score dump and select belong to the probe, not to flat_scan / merge
        assert prof["ivf_probe"][1] == 2 and prof["flat_scan"][1] == 0


def test_host_cache_is_bounded_and_correct(sa, small_index):
    """sa_search_host keeps at most 32 captured shapes (LRU); evicted shapes recapture."""
    idx, Q = small_index
    Qh = Q.float().cpu()
    ref = {}
    for nq in range(1, 41):     # 40 distinct shapes > the 32-entry cap
        qb = Qh[:nq].contiguous().pin_memory()
        ids, _ = idx.search_host(qb, 5, 8)
        ref[nq] = ids.clone()
    for nq in (1, 2, 40):       # 1 and 2 were evicted: recaptured, same result
        ids, _ = idx.search_host(Qh[:nq].contiguous().pin_memory(), 5, 8)
        assert torch.equal(ids, ref[nq])
        dev, _ = idx.search(Q[:nq].contiguous(), 5, 8)
        assert np.array_equal(ids.numpy(), dev.cpu().numpy())

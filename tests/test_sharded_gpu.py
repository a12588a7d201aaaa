"""Row-sharded search on one GPU (P8-iii): w shard indexes (row_offset,
n_total) searched with sa_search_keys, stacked rank-major [w, nq, k] exactly as
ncclAllGather lays them out, merged with sa_merge_keys -> bit-identical to the unsharded
index, for the exact mode and for IVF (shards built with the full index's centroids)."""
import numpy as np
import pytest
import torch

from datagen import make_mixture, draw_rows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def data():
    mix = make_mixture(d=256, C=16, r=16)
    X = draw_rows(mix, 60_001, row_seed=41, device="cuda").to(torch.bfloat16)
    Q = draw_rows(mix, 300, row_seed=42, device="cuda").to(torch.bfloat16)
    return X, Q


@pytest.mark.parametrize("w", [2, 3, 4])
def test_exact_sharded_equals_unsharded(sa, data, w):
    X, Q = data
    n = X.shape[0]
    full = sa.Index.build(X)
    ids, sc = full.search(Q, 10)
    keys = []
    for r in range(w):
        off, ln = sa.shard_range(n, r, w)
        idx = sa.Index.build(X[off:off + ln].contiguous(), row_offset=off, n_total=n)
        keys.append(idx.search_keys(Q, 10))
        idx.free()
    mi, ms = sa.sa_merge_keys(torch.stack(keys))
    assert torch.equal(mi, ids) and torch.equal(ms, sc)
    full.free()


@pytest.mark.parametrize("w,nprobe", [(2, 8), (4, 32)])
def test_ivf_sharded_equals_unsharded(sa, data, w, nprobe):
    X, Q = data
    n = X.shape[0]
    full = sa.Index.build(X, 64, kmeans_iters=8)
    ids, sc = full.search(Q, 10, nprobe=nprobe)
    C = torch.from_numpy(full.export_centroids()).cuda()
    keys = []
    for r in range(w):
        off, ln = sa.shard_range(n, r, w)
        idx = sa.Index.build(X[off:off + ln].contiguous(), 64, row_offset=off, n_total=n,
                             centroids=C)
        assert np.array_equal(idx.export_centroids(), full.export_centroids())
        keys.append(idx.search_keys(Q, 10, nprobe=nprobe))
        idx.free()
    mi, ms = sa.sa_merge_keys(torch.stack(keys))
    assert torch.equal(mi, ids) and torch.equal(ms, sc)
    full.free()


def test_merge_keys_pads_and_orders(sa):
    # two "ranks", one empty: the merge must keep the order and pad with (-1, -inf)
    k = 4
    sc = torch.tensor([[0.5, 0.25, 0.0, -1.0]])
    ids = torch.tensor([[7, 3, 9, 2]])
    X = torch.zeros(10, 64)
    for i, s in zip(ids[0].tolist(), sc[0].tolist()):
        X[i, 0] = s
    idx = sa.Index.build(X.cuda())
    q = torch.zeros(1, 64, device="cuda")
    q[0, 0] = 1.0
    kk = idx.search_keys(q, k)
    empty = torch.zeros_like(kk)
    mi, ms = sa.sa_merge_keys(torch.stack([empty, kk]))
    assert mi[0].tolist() == [7, 3, 0, 1] and ms[0, :2].tolist() == [0.5, 0.25]
    mi2, ms2 = sa.sa_merge_keys(torch.stack([empty, empty]))
    assert mi2[0].tolist() == [-1] * k and torch.isinf(ms2).all()
    idx.free()

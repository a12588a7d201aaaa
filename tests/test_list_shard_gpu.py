"""List-sharded IVF (sa_build_opts.list_shard_*): every rank
holds the full corpus, trains the same quantiser, and keeps the whole lists l % w == r.  Driven
on one B200 through the in-process communicator group (one host thread per rank): the sharded
search (rank-local keys -> all-gather -> merge) must equal the unsharded index bit for bit,
exact and IVF, and pass the oracle band rule; without a communicator the ranks' lists
partition the unsharded index's lists.
"""
import threading

import numpy as np
import pytest
import torch

from datagen import draw_rows, make_mixture, to_bf16_bits
from parity import check_against_rows

pytestmark = pytest.mark.gpu

N, D, NQ, K, NLIST = 24_007, 128, 120, 10, 48


@pytest.fixture(scope="module")
def data():
    mix = make_mixture(d=D, C=16, r=16)
    X = draw_rows(mix, N, row_seed=81).to(torch.bfloat16)
    Q = draw_rows(mix, NQ, row_seed=82).to(torch.bfloat16)
    return X.cuda(), Q.cuda()


def run_ranks(world, fn):
    out, err = [None] * world, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                out[r] = fn(r)
                torch.cuda.current_stream().synchronize()
        except BaseException as e:  # noqa: BLE001 -- re-raised below
            err.append((r, e))

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    if err:
        raise err[0][1]
    assert not any(t.is_alive() for t in ts), "a rank hung"
    return out


def test_lists_partition_the_unsharded_index(sa, data):
    X, _ = data
    full = sa.Index.build(X, NLIST, kmeans_iters=4)
    f_off, f_ids = full.export_lists()
    cents = full.export_centroids()
    full.free()
    w = 3
    seen = np.zeros(N, dtype=np.int64)
    for r in range(w):
        idx = sa.Index.build(X, NLIST, kmeans_iters=4, list_shard=(r, w))
        assert np.array_equal(idx.export_centroids().view(np.uint32), cents.view(np.uint32))
        off, ids = idx.export_lists()
        for l in range(NLIST):
            got = np.sort(ids[off[l]:off[l + 1]])
            want = np.sort(f_ids[f_off[l]:f_off[l + 1]]) if l % w == r else np.zeros(0, ids.dtype)
            assert np.array_equal(got, want), (r, l)
        seen[ids] += 1
        idx.free()
    assert (seen == 1).all()


@pytest.mark.parametrize("world", [2, 3])
def test_list_sharded_search_equals_unsharded(sa, data, world):
    X, Q = data
    plain = sa.Index.build(X, NLIST, kmeans_iters=4)
    want = {p: [t.cpu() for t in plain.search(Q, K, p)] for p in (0, 6, NLIST)}
    plain.free()
    comms = sa.Comm.local_group(world)

    def rank(r):
        idx = sa.Index.build(X, NLIST, kmeans_iters=4, comm=comms[r], list_shard=(r, world))
        res = {p: [t.cpu() for t in idx.search(Q, K, p)] for p in (0, 6, NLIST)}
        idx.free()
        return res

    outs = run_ranks(world, rank)
    for c in comms:
        c.free()
    for p in (0, 6, NLIST):
        for r in range(world):
            ids, sc = outs[r][p]
            assert torch.equal(ids, want[p][0]), (world, r, p)
            assert np.array_equal(sc.numpy().view(np.uint32), want[p][1].numpy().view(np.uint32))
    ids, sc = outs[0][0]
    rep = check_against_rows(ids.numpy(), sc.numpy(), to_bf16_bits(X.cpu()), to_bf16_bits(Q.cpu()), K)
    assert rep["ok"], rep


def test_list_shard_argument_errors(sa, data):
    X, _ = data
    with pytest.raises(sa.SAError):
        sa.Index.build(X, 0, list_shard=(0, 2))                   # needs nlist >= 1
    with pytest.raises(sa.SAError):
        sa.Index.build(X, NLIST, list_shard=(2, 2))               # rank out of range
    with pytest.raises(sa.SAError):
        sa.Index.build(X[:1000].contiguous(), NLIST, row_offset=5, n_total=2000,
                       list_shard=(0, 2))                          # not the full corpus

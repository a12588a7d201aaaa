"""The NCCL transport of the sharded path, executed on one B200 (
VERDICT r1 "the ncclAllGather branch has never been executed").

An NCCL communicator of ONE rank (sa_comm_unique_id + sa_comm_init, world 1) with
sa_comm_set_collectives on takes exactly the code path of a multi-GPU job -- the sharded IVF
build assembles its training sample with ncclBroadcast, every search runs rank-local keys ->
ncclAllGather -> k-way merge, and the cross-rank argument check all-gathers its header -- with
no second GPU and no rank waiting on another.  Results must equal the unsharded index bit for
bit (P8-iii) and pass the oracle band rule.
"""
import numpy as np
import pytest
import torch

from datagen import draw_rows, make_mixture, to_bf16_bits
from parity import check_against_rows

pytestmark = pytest.mark.gpu

N, D, NQ, K = 20_011, 128, 150, 10


@pytest.fixture(scope="module")
def data():
    mix = make_mixture(d=D, C=16, r=16)
    X = draw_rows(mix, N, row_seed=4242)
    Q = draw_rows(mix, NQ, row_seed=2424)
    return X, Q


@pytest.fixture(scope="module")
def comm(sa):
    c = sa.Comm.nccl_single().set_collectives(True).set_checks(True)
    info = c.info()
    assert info["world"] == 1 and info["nccl_nranks"] == 1
    yield c
    c.free()


def _run(idx, Q, k, nprobe):
    ids, sc = idx.search(Q, k, nprobe)
    torch.cuda.synchronize()
    return ids.cpu().numpy(), sc.cpu().numpy()


def test_nccl_sharded_exact_equals_unsharded_and_oracle(sa, data, comm):
    X, Q = data
    Xd, Qd = X.cuda().to(torch.bfloat16), Q.cuda().to(torch.bfloat16)
    plain = sa.Index.build(Xd)
    shard = sa.Index.build(Xd, row_offset=0, n_total=N, comm=comm)
    a, sa_ = _run(plain, Qd, K, 0)
    b, sb = _run(shard, Qd, K, 0)
    assert np.array_equal(a, b) and np.array_equal(sa_.view(np.uint32), sb.view(np.uint32))
    rep = check_against_rows(b, sb, to_bf16_bits(X), to_bf16_bits(Q), K)
    assert rep["ok"], rep
    # the host-buffer call takes the same sharded path (no captured graph when sharded)
    hi, hs = shard.search_host(Q.float().contiguous(), K, 0)
    assert np.array_equal(hi.numpy(), b) and np.array_equal(hs.numpy().view(np.uint32),
                                                            sb.view(np.uint32))
    plain.free()
    shard.free()


def test_nccl_sharded_ivf_build_and_search(sa, data, comm):
    X, Q = data
    Xd, Qd = X.cuda().to(torch.bfloat16), Q.cuda().to(torch.bfloat16)
    plain = sa.Index.build(Xd, 32, kmeans_iters=4)
    shard = sa.Index.build(Xd, 32, kmeans_iters=4, row_offset=0, n_total=N, comm=comm)
    # the sample assembled by ncclBroadcast trains the same centroids
    assert np.array_equal(plain.export_centroids().view(np.uint32),
                          shard.export_centroids().view(np.uint32))
    for nprobe in (4, 32):
        a, sa_ = _run(plain, Qd, K, nprobe)
        b, sb = _run(shard, Qd, K, nprobe)
        assert np.array_equal(a, b) and np.array_equal(sa_.view(np.uint32), sb.view(np.uint32))
    rep = check_against_rows(b, sb, to_bf16_bits(X), to_bf16_bits(Q), K)   # nprobe = nlist
    assert rep["ok"], rep
    plain.free()
    shard.free()


def test_nccl_argument_check_rejects_bad_call(sa, data, comm):
    X, Q = data
    shard = sa.Index.build(X.cuda().to(torch.bfloat16), row_offset=0, n_total=N, comm=comm)
    ids = torch.full((NQ, K), 7, dtype=torch.int64, device="cuda")
    sc = torch.full((NQ, K), 7.0, dtype=torch.float32, device="cuda")
    with pytest.raises(sa.SAError):
        shard.search(Q.cuda().to(torch.bfloat16), 0, 0, out=(ids, sc))   # k = 0: invalid
    torch.cuda.synchronize()
    assert bool((ids == 7).all()) and bool((sc == 7.0).all())       # outputs untouched
    shard.free()

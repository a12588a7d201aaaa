"""Parity of the exact flat path (tcgen05 scan + fused top-k + merge) against the
fp64 oracle, through the C ABI.  SURVEY.md §8(c) pins P1-P8; band rule in
tests/parity.py."""
import numpy as np
import pytest
import torch

import oracle
from datagen import make_mixture, draw_rows, to_bf16_bits, planted_corpus
from parity import check_against_rows

pytestmark = pytest.mark.gpu


def _bf16(x):
    return torch.as_tensor(x, dtype=torch.float32).to(torch.bfloat16)


def _search(sa, X, Q, k, qdtype=torch.bfloat16):
    idx = sa.Index.build(X.cuda().contiguous())
    ids, sc = idx.search(Q.cuda().to(qdtype).contiguous(), k)
    torch.cuda.synchronize()
    idx.free()
    return ids.cpu().numpy(), sc.cpu().numpy()


# ------------------------------------------------------------ tensor-core layout
@pytest.mark.parametrize("n,d,nq", [(200, 64, 5), (1000, 128, 130), (777, 768, 129), (333, 100, 3),
                                    (5003, 256, 515)])   # > 148 tiles: several per CTA
def test_debug_scores_match_oracle(sa, n, d, nq):
    g = torch.Generator().manual_seed(n + d)
    X = torch.randn(n, d, generator=g)
    Q = torch.randn(nq, d, generator=g)
    idx = sa.Index.build(X.cuda())
    S = idx.debug_scores(Q.cuda().to(torch.bfloat16)).cpu().numpy().astype(np.float64)
    idx.free()
    Xb, Qb = to_bf16_bits(X), to_bf16_bits(Q)
    qi, ri = np.meshgrid(np.arange(nq), np.arange(n), indexing="ij")
    want = oracle.pair_scores(Xb, Qb, qi.ravel(), ri.ravel()).reshape(nq, n)
    scale = np.sqrt((oracle.bf16_to_f64(Qb) ** 2).sum(1))[:, None] * np.sqrt(
        (oracle.bf16_to_f64(Xb) ** 2).sum(1))[None, :]
    err = np.abs(S - want) / scale
    assert err.max() < 1e-5, err.max()


# ------------------------------------------------------------ C1 (BASELINE config 1)
def test_c1_full_parity(sa):
    mix = make_mixture(d=128, C=16, r=16)
    X = draw_rows(mix, 10_000, row_seed=1234)          # fp32 corpus, rounded by the library
    Q = draw_rows(mix, 100, row_seed=5678)
    ids, sc = _search(sa, X, Q, 10, qdtype=torch.float32)
    rep = check_against_rows(ids, sc, to_bf16_bits(X), to_bf16_bits(Q), 10)
    assert rep["ok"], rep
    rep5 = check_against_rows(ids, sc, to_bf16_bits(X), to_bf16_bits(Q), 10, rtol=1e-5)
    assert rep5["ok"], rep5          # diagnostic band


@pytest.mark.parametrize("n,d,nq,k", [
    (1, 64, 1, 1), (63, 64, 2, 5), (64, 128, 128, 10), (65, 128, 129, 10),
    (4097, 384, 127, 32), (4097, 384, 127, 33), (3000, 768, 200, 256), (500, 96, 300, 100),
    (20000, 768, 513, 10),
])
def test_shapes_and_k(sa, n, d, nq, k):
    g = torch.Generator().manual_seed(n * 7 + nq)
    X = torch.randn(n, d, generator=g)
    Q = torch.randn(nq, d, generator=g)
    ids, sc = _search(sa, X, Q, k)
    rep = check_against_rows(ids, sc, to_bf16_bits(X), to_bf16_bits(Q), k)
    assert rep["ok"], rep


def test_p3_k_greater_than_n_pads(sa):
    g = torch.Generator().manual_seed(3)
    X = torch.randn(7, 64, generator=g)
    Q = torch.randn(3, 64, generator=g)
    ids, sc = _search(sa, X, Q, 12)
    assert np.all(ids[:, 7:] == -1) and np.all(np.isneginf(sc[:, 7:]))
    for qi in range(3):
        assert sorted(ids[qi, :7].tolist()) == list(range(7))


def test_p1_spec_example_exact(sa):
    X = torch.tensor([[0.0, 0.0], [1.0, 0.0], [0.0, 2.0]])
    Q = torch.tensor([[0.9, 0.0]])
    ids, sc = _search(sa, X, Q, 2)
    assert ids[0].tolist() == [1, 0]
    assert sc[0].tolist() == [0.8984375, 0.0]


def test_p4_orthonormal_exact_ties(sa):
    d = 128
    X = torch.eye(d)
    Q = X[[0, 5, 127]]
    ids, sc = _search(sa, X, Q, 6)
    for r, j in enumerate([0, 5, 127]):
        assert ids[r].tolist() == [j] + [i for i in range(d) if i != j][:5]
        assert sc[r].tolist() == [1.0] + [0.0] * 5


def test_p5_duplicates_across_tiles(sa):
    g = torch.Generator().manual_seed(5)
    X = torch.randn(5000, 128, generator=g)
    for dup in (63, 64, 2047, 4999):
        X[dup] = X[10]
    Q = X[10:11] + 0.01 * torch.randn(1, 128, generator=g)
    ids, sc = _search(sa, X, Q, 5)
    assert ids[0].tolist() == [10, 63, 64, 2047, 4999]
    assert len(set(sc[0].tolist())) == 1          # bit-identical scores


def test_p6_all_negative(sa):
    g = torch.Generator().manual_seed(6)
    q = torch.randn(1, 256, generator=g)
    scale = torch.rand(3000, 1, generator=g) + 0.1
    X = -scale * _bf16(q).float()
    ids, sc = _search(sa, X, q, 10)
    rep = check_against_rows(ids, sc, to_bf16_bits(X), to_bf16_bits(q), 10)
    assert rep["ok"], rep
    assert np.all(sc < 0)


def test_p7_planted_tile_edges(sa):
    n = 70_001
    winners = [0, 63, 64, 127, 128, 255, 256, 4095, 4096, n // 2, n - 2, n - 1]
    X, Q = planted_corpus(n, 384, winners)
    ids, sc = _search(sa, X, Q, 3)
    assert ids[:, 0].tolist() == winners
    rep = check_against_rows(ids, sc, to_bf16_bits(X), to_bf16_bits(Q), 3)
    assert rep["ok"], rep


def test_p8_batch_invariance_and_pow2_scaling(sa):
    mix = make_mixture(d=768, C=128, r=32)
    X = draw_rows(mix, 30_000, row_seed=11)
    Q = draw_rows(mix, 512, row_seed=12)
    idx = sa.Index.build(X.cuda().to(torch.bfloat16))
    Qd = Q.cuda().to(torch.bfloat16)
    ids, sc = idx.search(Qd, 10)
    for j in (0, 200, 511):
        i1, s1 = idx.search(Qd[j:j + 1].contiguous(), 10)
        assert torch.equal(i1[0], ids[j]) and torch.equal(s1[0], sc[j])
    i4, s4 = idx.search((Qd * 4).contiguous(), 10)
    assert torch.equal(i4, ids) and torch.equal(s4, sc * 4)
    idx.free()


def test_search_host_matches_device(sa):
    g = torch.Generator().manual_seed(9)
    X = torch.randn(9000, 256, generator=g)
    Q = torch.randn(33, 256, generator=g)
    idx = sa.Index.build(X.cuda())
    i_d, s_d = idx.search(Q.cuda(), 7)
    i_h, s_h = idx.search_host(Q.contiguous(), 7)
    assert torch.equal(i_d.cpu(), i_h) and torch.equal(s_d.cpu(), s_h)
    idx.free()


# ------------------------------------------------------------ C2 (BASELINE config 2)
@pytest.mark.slow
def test_c2_parity(sa):
    mix = make_mixture(d=768, C=128, r=32)
    X = torch.empty(1_000_000, 768, dtype=torch.bfloat16, device="cuda")
    from datagen import draw_rows_into
    draw_rows_into(mix, X, row_seed=1234)
    Q = draw_rows(mix, 256, row_seed=5678, device="cuda").to(torch.bfloat16)
    idx = sa.Index.build(X)
    ids, sc = idx.search(Q, 10)
    torch.cuda.synchronize()
    Xb = X.cpu().view(torch.int16).numpy().view(np.uint16)
    Qb = Q.cpu().view(torch.int16).numpy().view(np.uint16)
    sub = np.arange(0, 256, 4)                # 64 of the 256 queries through the oracle
    rep = check_against_rows(ids.cpu().numpy()[sub], sc.cpu().numpy()[sub], Xb, Qb[sub], 10)
    idx.free()
    assert rep["ok"], rep


def test_search_host_graph_replay_matches_device(sa):
    """The small-batch host path replays a captured CUDA graph; results must equal the
    device path for repeated calls with new data and for several shapes (exact + IVF)."""
    g = torch.Generator().manual_seed(19)
    X = torch.randn(20_000, 128, generator=g)
    idx = sa.Index.build(X.cuda(), 16, kmeans_iters=4)
    for nq, k, nprobe in [(1, 5, 0), (7, 5, 4), (64, 10, 16), (7, 5, 4)]:
        for rep in range(3):
            Q = torch.randn(nq, 128, generator=g)
            i_d, s_d = idx.search(Q.cuda(), k, nprobe)
            i_h, s_h = idx.search_host(Q.contiguous(), k, nprobe)
            assert torch.equal(i_d.cpu(), i_h) and torch.equal(s_d.cpu(), s_h), (nq, k, nprobe, rep)
    idx.free()

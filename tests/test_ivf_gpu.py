"""IVF build + search on the GPU against the IVF oracle (oracle/ivf.py) and the IVF
invariants of SURVEY.md §8(c) (P10-P14)."""
import numpy as np
import pytest
import torch

import oracle
from oracle import ivf
from datagen import make_mixture, draw_rows, to_bf16_bits
from parity import check, check_against_rows

pytestmark = pytest.mark.gpu


def bits(x):
    return oracle.bf16_round(np.asarray(x, dtype=np.float32))


def bits_to_tensor(b):
    return torch.from_numpy(b.view(np.int16).copy()).view(torch.bfloat16)


def blocks_corpus(n_per, d=32, nblk=4, noise=0.01, seed=0):
    g = np.random.default_rng(seed)
    X = noise * g.standard_normal((n_per * nblk, d))
    for b in range(nblk):
        X[b * n_per:(b + 1) * n_per, b] += 1.0
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    return bits(X)


def lists_of(idx):
    off, ids = idx.export_lists()
    return [ids[off[j]:off[j + 1]] for j in range(len(off) - 1)], off, ids


@pytest.mark.parametrize("n_per", [1000, 10000])
def test_p14_planted_blocks_match_oracle(sa, n_per):
    X = blocks_corpus(n_per)
    C, Cb, assign, lists = ivf.build(X, 4, iters=5)
    idx = sa.Index.build(bits_to_tensor(X).cuda(), 4, kmeans_iters=5)
    glists, off, ids = lists_of(idx)
    for j in range(4):
        assert np.array_equal(glists[j], lists[j])
    Cg = idx.export_centroids()
    assert np.abs(Cg - C).max() < 1e-5
    # queries near block 2: nprobe=1 returns only block-2 ids; 300 queries -> 3 query blocks
    g = np.random.default_rng(5)
    Q = np.zeros((300, 32))
    Q[:, 2] = 1.0
    Q += 0.05 * g.standard_normal(Q.shape)
    Qb = bits(Q)
    gi, gs = idx.search(bits_to_tensor(Qb).cuda(), 10, nprobe=1)
    gi, gs = gi.cpu().numpy(), gs.cpu().numpy()
    oi, osc, P = ivf.search(X, lists, Cb, Qb, 10, 1)
    assert np.all((gi >= 2 * n_per) & (gi < 3 * n_per))
    rows = lists[2]
    rep = check(gi, gs, oi, osc,
                lambda qi, ids_: oracle.pair_scores(X, Qb, np.full(len(ids_), qi), ids_), 10)
    assert rep["ok"], rep
    idx.free()


def test_r10_empty_list_repair_matches_oracle(sa):
    g = np.random.default_rng(3)
    X = 0.01 * g.standard_normal((4000, 16))
    for b, axis in enumerate([0, 1, 2, 2]):
        X[b * 1000:(b + 1) * 1000, axis] += 1.0
    X[2000:4000] = X[2000]
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    Xb = bits(X)
    C1, _, _ = ivf.kmeans(Xb, 4, iters=1)
    idx = sa.Index.build(bits_to_tensor(Xb).cuda(), 4, kmeans_iters=1)
    Cg = idx.export_centroids()
    assert np.abs(Cg - C1).max() < 1e-5
    idx.free()


@pytest.fixture(scope="module")
def mixture_index(sa):
    mix = make_mixture(d=128, C=16, r=16, s_n=0.7)
    X = draw_rows(mix, 50_000, row_seed=21)
    Q = draw_rows(mix, 64, row_seed=22)
    Xb, Qb = to_bf16_bits(X), to_bf16_bits(Q)
    idx = sa.Index.build(bits_to_tensor(Xb).cuda(), 64, kmeans_iters=10)
    yield idx, Xb, Qb
    idx.free()


def test_p13_lists_partition_and_assignment(sa, mixture_index):
    idx, Xb, Qb = mixture_index
    glists, off, ids = lists_of(idx)
    assert off[0] == 0 and off[-1] == Xb.shape[0] and np.all(np.diff(off) >= 0)
    assert np.array_equal(np.sort(ids), np.arange(Xb.shape[0]))
    for l in glists:
        assert np.all(np.diff(l) > 0)                     # ascending id inside a list
    Cg = idx.export_centroids()
    Cb = oracle.bf16_to_f64(bits(Cg))
    sc = oracle.bf16_to_f64(Xb) @ Cb.T
    assigned = np.empty(Xb.shape[0], dtype=np.int64)
    for j, l in enumerate(glists):
        assigned[l] = j
    best = sc.max(1)
    got = sc[np.arange(len(assigned)), assigned]
    assert np.all(got >= best - 1e-5)                     # argmax within fp32 rounding
    assert np.mean(assigned == sc.argmax(1)) > 0.999
    assert np.allclose(np.linalg.norm(Cg, axis=1), 1.0, atol=1e-5)


def test_build_is_deterministic(sa, mixture_index):
    idx, Xb, _ = mixture_index
    idx2 = sa.Index.build(bits_to_tensor(Xb).cuda(), 64, kmeans_iters=10)
    assert np.array_equal(idx.export_centroids(), idx2.export_centroids())
    o1, i1 = idx.export_lists()
    o2, i2 = idx2.export_lists()
    assert np.array_equal(o1, o2) and np.array_equal(i1, i2)
    idx2.free()


def test_p10_nprobe_nlist_is_exact(sa, mixture_index):
    idx, Xb, Qb = mixture_index
    gi, gs = idx.search(bits_to_tensor(Qb).cuda(), 10, nprobe=64)
    rep = check_against_rows(gi.cpu().numpy(), gs.cpu().numpy(), Xb, Qb, 10)
    assert rep["ok"], rep
    # exact mode on the (list-major) IVF index is exact too
    gi0, gs0 = idx.search(bits_to_tensor(Qb).cuda(), 10, nprobe=0)
    rep0 = check_against_rows(gi0.cpu().numpy(), gs0.cpu().numpy(), Xb, Qb, 10)
    assert rep0["ok"], rep0


@pytest.mark.parametrize("nprobe,k", [(1, 10), (4, 10), (8, 50), (16, 5)])
def test_p11_result_is_exact_over_probed_lists(sa, mixture_index, nprobe, k):
    idx, Xb, Qb = mixture_index
    glists, _, _ = lists_of(idx)
    Qd = bits_to_tensor(Qb).cuda()
    P = idx.probes(Qd, nprobe).cpu().numpy()
    # probe set = top-nprobe centroids by fp64 score over the stored bf16 centroids (band)
    Cb_bits = bits(idx.export_centroids())
    pids, psc = oracle.flat_topk(Cb_bits, Qb, min(64, nprobe + 8))
    pc = oracle.bf16_to_f64(Qb) @ oracle.bf16_to_f64(Cb_bits).T
    for qi in range(len(Qb)):
        thr = psc[qi, nprobe - 1]
        must = set(pids[qi][psc[qi] > thr + 1e-5].tolist())
        assert must <= set(P[qi].tolist())
        assert np.all(pc[qi, P[qi]] >= thr - 1e-5)
    gi, gs = idx.search(Qd, k, nprobe=nprobe)
    gi, gs = gi.cpu().numpy(), gs.cpu().numpy()
    for qi in range(len(Qb)):
        rows = np.sort(np.concatenate([glists[j] for j in P[qi]]))
        oi, osc = oracle.flat_topk(Xb[rows], Qb[qi:qi + 1], k + 8)
        oi = np.where(oi >= 0, rows[np.maximum(oi, 0)], -1)
        r = check(gi[qi:qi + 1], gs[qi:qi + 1], oi, osc,
                  lambda _q, ids_: oracle.pair_scores(Xb, Qb[qi:qi + 1], np.zeros(len(ids_), int), ids_),
                  k, n_avail=min(k, len(rows)))
        assert r["ok"], (qi, r)


def test_p12_recall_monotone(sa, mixture_index):
    idx, Xb, Qb = mixture_index
    Qd = bits_to_tensor(Qb).cuda()
    ei, _ = oracle.flat_topk(Xb, Qb, 10)
    prev = np.zeros(len(Qb))
    for nprobe in (1, 2, 4, 8, 16, 32, 64):
        gi, _ = idx.search(Qd, 10, nprobe=nprobe)
        gi = gi.cpu().numpy()
        rec = np.array([len(set(gi[i]) & set(ei[i])) / 10 for i in range(len(Qb))])
        assert np.all(rec >= prev - 1e-9)
        prev = rec
    assert prev.mean() == 1.0

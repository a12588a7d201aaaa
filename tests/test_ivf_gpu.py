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


def test_kmeans_mixture_steps_match_oracle(sa):
    """k-means on realistic data: on a 40k-row mixture, the GPU's
    initial centroids equal the oracle's bit for bit, and each of the first two Lloyd
    iterations, started from the GPU's own previous centroids, equals the oracle's step
    (oracle/ivf.lloyd_step) on every list no ambiguous row touches.  A row is ambiguous when
    its best and second-best centroid scores are closer than twice the fp32 accumulation
    bound of both, 2 * (d - 1) * 2^-24 * sum_j |x_j c_j| (the GPU decides on fp32 tensor-core
    scores of exact bf16 products, the oracle in fp64); decisions with larger margins must
    agree.  Unaffected centroids agree within 1e-5 (fp32 member sums); at least 3/4 of the
    lists are compared in each iteration."""
    mx = make_mixture(d=128, C=16, r=16, s_n=0.7)
    Xb = to_bf16_bits(draw_rows(mx, 40_000, row_seed=91))
    nlist = 64
    Xd = bits_to_tensor(Xb).cuda()
    rows = ivf.sample_rows(Xb.shape[0], nlist)
    S = oracle.bf16_to_f64(Xb[rows])
    C0_or = ivf.kmeans(Xb, nlist, iters=0)[0]
    prev = None
    touched_total = 0
    for it in range(3):
        idx = sa.Index.build(Xd, nlist, kmeans_iters=it)
        Cg = idx.export_centroids().astype(np.float64)
        idx.free()
        if it == 0:
            assert np.array_equal(Cg, C0_or)          # R9 init: sample rows, widened exactly
        else:
            C_or, a, margin = ivf.lloyd_step(S, prev)
            Cb = oracle.bf16_to_f64(ivf.centroids_bf16(prev))
            second = np.argsort(-(S @ Cb.T), axis=1)[:, 1]
            d = S.shape[1]
            absum = np.abs(S) @ np.abs(Cb).T
            eb = 2 * (d - 1) * 2.0 ** -24 * (absum[np.arange(len(S)), a] +
                                             absum[np.arange(len(S)), second])
            amb = np.nonzero(margin <= eb)[0]
            touched = set(a[amb].tolist()) | set(second[amb].tolist())
            empty = [j for j in range(nlist) if not np.any(a == j)]
            if empty:   # the repair depends on every row's score: compare only when unambiguous
                assert amb.size == 0
            ok = [j for j in range(nlist) if j not in touched]
            assert len(ok) >= 3 * nlist // 4, (it, len(touched), amb.size)
            assert np.abs(Cg[ok] - C_or[ok]).max() < 1e-5, it
            touched_total += len(touched)
        prev = Cg
    print(f"k-means steps: {touched_total} list(s) touched by ambiguous rows over 2 iterations")


def test_t1_error_paths_on_live_index(sa):
    """SURVEY §8(b) conventions on a LIVE index (not just a null handle): each invalid call
    returns its status and leaves the outputs untouched (validation is synchronous and side-
    effect free); nprobe > 0 on a flat index is SA_ERR_STATE; k beyond the candidates is legal
    and padded."""
    mx = make_mixture(d=64, C=4, r=8, s_n=0.7)
    X = draw_rows(mx, 3000, row_seed=93).cuda().to(torch.bfloat16)
    Q = draw_rows(mx, 5, row_seed=94).cuda().to(torch.bfloat16)
    flat = sa.Index.build(X)
    ivfi = sa.Index.build(X, 8, kmeans_iters=2)
    L = sa.lib()
    ids = torch.full((5, 300), 123, dtype=torch.int64, device="cuda")
    sc = torch.full((5, 300), 4.5, device="cuda")
    st = sa._stream_ptr(None)

    def call(idx, q, nq, k, nprobe, qdt=sa.SA_BF16):
        r = L.sa_search_ex(idx.handle, q, qdt, nq, k, nprobe, sa._ptr(ids), sa._ptr(sc), st)
        torch.cuda.synchronize()
        return r

    cases = [(flat, sa._ptr(Q), 5, 0, 0, sa.SA_ERR_INVALID_ARG),     # k = 0
             (flat, sa._ptr(Q), 5, 257, 0, sa.SA_ERR_INVALID_ARG),   # k > 256
             (flat, sa._ptr(Q), 0, 10, 0, sa.SA_ERR_INVALID_ARG),    # nq = 0
             (flat, sa._ptr(Q), -3, 10, 0, sa.SA_ERR_INVALID_ARG),   # nq < 0
             (flat, None, 5, 10, 0, sa.SA_ERR_INVALID_ARG),          # null queries
             (flat, sa._ptr(Q), 5, 10, 1, sa.SA_ERR_STATE),          # nprobe > 0 on a flat index
             (ivfi, sa._ptr(Q), 5, 10, 9, sa.SA_ERR_INVALID_ARG),    # nprobe > nlist
             (ivfi, sa._ptr(Q), 5, 10, -1, sa.SA_ERR_INVALID_ARG),   # nprobe < 0
             (ivfi, sa._ptr(Q), 5, 10, 4, sa.SA_ERR_INVALID_ARG, 7)]  # bad dtype code
    for c in cases:
        idx, q, nq, k, nprobe, want = c[:6]
        qdt = c[6] if len(c) > 6 else sa.SA_BF16
        assert call(idx, q, nq, k, nprobe, qdt) == want, c
        assert sa.last_error() != ""
        assert bool((ids == 123).all()) and bool((sc == 4.5).all()), c   # outputs untouched
    # host-buffer and fp8 entry points validate the same way
    hq = Q.cpu()
    hi = torch.full((5, 10), 9, dtype=torch.int64)
    hs = torch.zeros(5, 10)
    assert L.sa_search_host(flat.handle, sa._ptr(hq), sa.SA_BF16, 5, 0, 0, sa._ptr(hi),
                            sa._ptr(hs), st) == sa.SA_ERR_INVALID_ARG
    assert bool((hi == 9).all())
    assert L.sa_search_fp8(flat.handle, sa._ptr(Q), sa.SA_BF16, 5, 10, 0, 16, sa._ptr(ids),
                           sa._ptr(sc), st) == sa.SA_ERR_STATE          # no fp8 copy built
    assert bool((ids == 123).all())
    # legal edge: k > n_local pads with (-1, -inf); k = n returns every row once
    small = sa.Index.build(X[:7].contiguous())
    gi, gs = small.search(Q, 12)
    assert (gi[:, 7:] == -1).all() and torch.isinf(gs[:, 7:]).all()
    assert all(sorted(r) == list(range(7)) for r in gi[:, :7].cpu().tolist())
    for i in (flat, ivfi, small):
        i.free()

"""Robustness variants of SURVEY.md §8(d) (correctness, not timed): adversarial ascending-
score row order, duplicated rows across tiles / slices / lists, a skewed giant IVF list,
and the largest k."""
import numpy as np
import pytest
import torch

import oracle
from datagen import make_mixture, draw_rows, to_bf16_bits
from parity import check, check_against_rows

pytestmark = pytest.mark.gpu


def _bits_t(b):
    return torch.from_numpy(b.view(np.int16).copy()).view(torch.bfloat16)


def test_adversarial_ascending_scores(sa):
    """Rows sorted so every query's score rises with the row id: every row of the scan is
    a new best, the heaps take an insertion per candidate (worst case for the epilogue)."""
    mix = make_mixture(d=256, C=8, r=8)
    X = draw_rows(mix, 40_000, row_seed=51)
    Q = draw_rows(mix, 300, row_seed=52)
    q0 = Q[0:1].to(torch.bfloat16).float()
    order = torch.argsort((X.to(torch.bfloat16).float() @ q0.T).squeeze(1))   # ascending
    X = X[order].contiguous()
    Q[1:5] = Q[0]                                             # several queries share the order
    idx = sa.Index.build(X.cuda())
    ids, sc = idx.search(Q.cuda().to(torch.bfloat16), 16)
    rep = check_against_rows(ids.cpu().numpy(), sc.cpu().numpy(), to_bf16_bits(X),
                             to_bf16_bits(Q), 16)
    idx.free()
    assert rep["ok"], rep


def test_duplicated_rows_tie_order(sa):
    """1% of rows duplicated at random positions (across tiles and corpus slices): ties must
    come back lowest id first, bit-identical scores, and parity holds."""
    g = np.random.default_rng(7)
    mix = make_mixture(d=128, C=8, r=8)
    X = draw_rows(mix, 60_000, row_seed=61)
    src = g.integers(0, 60_000, 600)
    dst = g.integers(0, 60_000, 600)
    X[dst] = X[src]
    Q = torch.cat([X[src[:40]] + 0.001, draw_rows(mix, 24, row_seed=62)])
    idx = sa.Index.build(X.cuda())
    ids, sc = idx.search(Q.cuda().to(torch.bfloat16), 10)
    ids, sc = ids.cpu().numpy(), sc.cpu().numpy()
    rep = check_against_rows(ids, sc, to_bf16_bits(X), to_bf16_bits(Q), 10)
    assert rep["ok"], rep
    for q in range(ids.shape[0]):
        for j in range(9):
            if sc[q, j] == sc[q, j + 1]:
                assert ids[q, j] < ids[q, j + 1]
    idx.free()


def test_skewed_giant_list_ivf(sa):
    """One mixture component with 40% of the rows (a giant list split into many chunks) plus
    noise components: IVF result == exact search over the probed lists; nprobe=nlist exact."""
    mix = make_mixture(d=128, C=16, r=4, s_sub=0.3, s_n=0.2)
    big = draw_rows(make_mixture(d=128, C=1, r=2, s_sub=0.1, s_n=0.05, struct_seed=99),
                    20_000, row_seed=71)
    rest = draw_rows(mix, 30_000, row_seed=72)
    X = torch.cat([big, rest])
    Xb = to_bf16_bits(X)
    Q = torch.cat([big[:8] + 0.01, rest[:8]])
    Qb = to_bf16_bits(Q)
    idx = sa.Index.build(_bits_t(Xb).cuda(), 32, kmeans_iters=6)
    off, gid = idx.export_lists()
    assert np.diff(off).max() > 4096          # at least one list spans several scan chunks
    Qd = _bits_t(Qb).cuda()
    gi, gs = idx.search(Qd, 10, nprobe=4)
    gi, gs = gi.cpu().numpy(), gs.cpu().numpy()
    P = idx.probes(Qd, 4).cpu().numpy()
    for q in range(len(Qb)):
        rows = np.sort(np.concatenate([gid[off[l]:off[l + 1]] for l in P[q]]))
        oi, osc = oracle.flat_topk(Xb[rows], Qb[q:q + 1], 18)
        oi = np.where(oi >= 0, rows[np.maximum(oi, 0)], -1)
        r = check(gi[q:q + 1], gs[q:q + 1], oi, osc,
                  lambda _q, ids_: oracle.pair_scores(Xb, Qb[q:q + 1], np.zeros(len(ids_), int), ids_),
                  10)
        assert r["ok"], (q, r)
    ai, asc = idx.search(Qd, 10, nprobe=32)
    rep = check_against_rows(ai.cpu().numpy(), asc.cpu().numpy(), Xb, Qb, 10)
    assert rep["ok"], rep
    idx.free()


@pytest.mark.parametrize("nprobe", [0, 16])
def test_k256(sa, nprobe):
    mix = make_mixture(d=192, C=8, r=8)
    X = draw_rows(mix, 30_000, row_seed=81)
    Q = draw_rows(mix, 20, row_seed=82)
    idx = sa.Index.build(X.cuda(), 16, kmeans_iters=4)
    # nprobe = 16 = nlist: exhaustive through the IVF path
    ids, sc = idx.search(Q.cuda().to(torch.bfloat16), 256, nprobe=nprobe)
    rep = check_against_rows(ids.cpu().numpy(), sc.cpu().numpy(), to_bf16_bits(X),
                             to_bf16_bits(Q), 256)
    idx.free()
    assert rep["ok"], rep

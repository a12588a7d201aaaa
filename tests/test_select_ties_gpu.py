"""The probe's exact top-nprobe select under heavy ties (readings R5, R11: keys (score desc,
list id asc)).  With a supplied quantiser whose centroids are duplicated, many centroid scores
are exactly equal (same bf16 data, same fp32 arithmetic), which drives the stream select
(nprobe <= 32) through its ranking path (<= 1024 survivors) and its radix fallback (more), and
the cached select (nprobe > 32) through its tie handling.  Expected: the oracle's order of the
fp64 scores with ties by lowest list id -- decided exactly where the fp64 margins are clear.
"""
import numpy as np
import pytest
import torch

from datagen import draw_rows, make_mixture

pytestmark = pytest.mark.gpu

D = 128


def _probe_case(sa, C, Q, nprobe):
    X = C.repeat(2, 1).contiguous()   # the rows do not matter for the probe
    idx = sa.Index.build(X.cuda().to(torch.bfloat16), C.shape[0], centroids=C.cuda().float())
    got = idx.probes(Q.cuda().to(torch.bfloat16), nprobe).cpu().numpy()
    cb = idx.export_centroids()        # the index's fp32 centroids (bf16 copies score)
    idx.free()
    return got, cb


def _expected(Cb, Qb, nprobe):
    S = Qb.astype(np.float64) @ Cb.astype(np.float64).T
    order = np.lexsort((np.arange(Cb.shape[0])[None, :].repeat(len(Qb), 0), -S), axis=1)
    return S, order[:, :nprobe]


@pytest.mark.parametrize("nlist,nprobe", [(512, 16), (2048, 16), (2048, 32), (2048, 48)])
def test_all_centroids_equal(sa, nlist, nprobe):
    """Every score ties: the probe set is lists 0..nprobe-1 for every query."""
    mix = make_mixture(d=D, C=4, r=8)
    c = draw_rows(mix, 1, row_seed=7)
    C = c.repeat(nlist, 1)
    Q = draw_rows(mix, 37, row_seed=8)
    got, _ = _probe_case(sa, C, Q, nprobe)
    assert (got == np.arange(nprobe)[None, :]).all(), got[:2]


@pytest.mark.parametrize("nprobe", [8, 32, 48])
def test_duplicated_centroids(sa, nprobe):
    """64 distinct centroids, each repeated 8 times (nlist 512, interleaved): 8-way exact ties."""
    mix = make_mixture(d=D, C=16, r=16)
    base = draw_rows(mix, 64, row_seed=9)
    C = base.repeat(8, 1)                     # centroid j = base[j % 64]
    Q = draw_rows(mix, 53, row_seed=10)
    got, cb = _probe_case(sa, C, Q, nprobe)
    Cb = torch.from_numpy(cb).to(torch.bfloat16).float().numpy()
    Qb = Q.to(torch.bfloat16).float().numpy()
    S, want = _expected(Cb, Qb, nprobe)
    checked = 0
    for q in range(len(Q)):
        s_sorted = np.sort(np.unique(S[q]))[::-1]
        # distinct score levels must be separated well beyond fp32 rounding to compare exactly
        if len(s_sorted) > 1 and np.min(-np.diff(s_sorted[: nprobe // 8 + 2])) < 1e-4 * np.abs(S[q]).max():
            continue
        assert np.array_equal(got[q], want[q]), (q, got[q], want[q])
        checked += 1
    assert checked >= len(Q) // 2

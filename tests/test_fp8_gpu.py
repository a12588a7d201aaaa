"""fp8 flat scan + bf16 re-rank on the GPU (sa_index_build_fp8 / sa_search_fp8) against
oracle/fp8.py (readings R30-R33).

  * quantisation (R30): the e4m3 bytes and the scale exponent the index keeps equal the
    oracle's bit for bit (flat index and list-major IVF index);
  * candidates (R32): with k = n_cand every candidate comes back (re-scored); the set is the
    oracle's fp8 top-n_cand under the band rule on the fp8 scores (must-include above the
    boundary + tol, must-exclude below it);
  * re-rank (R33): the result is the exact top-k over the GPU's own candidate set (band rule
    against oracle.c), scores within tol of the fp64 bf16 scores;
  * end to end: equal to the exact search (band rule) for every query whose exact top-k lies
    among the oracle's candidates; edge shapes (nq 1 / 129 / 300, n_cand >= n, k > n).
"""
import numpy as np
import pytest
import torch

import oracle
from oracle import fp8
from datagen import make_mixture, draw_rows, to_bf16_bits
from parity import check, check_against_rows, tol_of

pytestmark = pytest.mark.gpu


def bits_to_tensor(b):
    return torch.from_numpy(np.ascontiguousarray(b).view(np.int16).copy()).view(torch.bfloat16)


@pytest.fixture(scope="module")
def data():
    mx = make_mixture(d=128, C=16, r=16, s_n=0.7)
    Xb = to_bf16_bits(draw_rows(mx, 20_011, row_seed=91))
    Qb = to_bf16_bits(draw_rows(mx, 300, row_seed=92))
    return Xb, Qb


@pytest.mark.parametrize("nlist", [0, 32])
def test_quantised_bytes_bit_exact(sa, data, nlist):
    Xb, _ = data
    idx = sa.Index.build(bits_to_tensor(Xb).cuda(), nlist, kmeans_iters=4).build_fp8()
    codes, e = idx.export_fp8()
    X8, oe = fp8.quantize_corpus(Xb)
    assert e == oe
    assert np.array_equal(codes, fp8.e4m3_bits(X8))
    idx.free()


def cand_check(gi, Xb, Qb, n_cand):
    """The GPU candidate ids vs the oracle's fp8 scores with the band rule."""
    X8, _ = fp8.quantize_corpus(Xb)
    Q8, _ = fp8.quantize_queries(Qb)
    Xc, Qc = fp8._as_bf16_bits(X8), fp8._as_bf16_bits(Q8)
    oi, osc = oracle.flat_topk(Xc, Qc, min(n_cand + 16, Xb.shape[0]))
    bad = []
    for q in range(len(Qb)):
        navail = min(n_cand, Xb.shape[0])
        sk = osc[q][navail - 1]
        t = tol_of(sk, 1e-3)
        g = set(gi[q][:navail].tolist())
        must = set(oi[q][osc[q] > sk + t].tolist())
        s_g = oracle.pair_scores(Xc, Qc, np.full(navail, q), gi[q][:navail])
        if must - g or np.any(s_g < sk - t) or len(g) != navail:
            bad.append(q)
    return bad


@pytest.mark.parametrize("nlist", [0, 32])
def test_candidates_and_rerank(sa, data, nlist):
    Xb, Qb = data
    idx = sa.Index.build(bits_to_tensor(Xb).cuda(), nlist, kmeans_iters=4).build_fp8()
    Qd = bits_to_tensor(Qb).cuda()
    n_cand = 48
    ci, cs = idx.search_fp8(Qd, n_cand, n_cand)      # every candidate, re-scored
    ci, cs = ci.cpu().numpy(), cs.cpu().numpy()
    assert cand_check(ci, Xb, Qb, n_cand) == []
    gi, gs = idx.search_fp8(Qd, 10, n_cand)
    gi, gs = gi.cpu().numpy(), gs.cpu().numpy()
    # R33: the top-10 of the GPU's own candidates -- bit-identical to the k = n_cand call,
    # and the exact top-10 over those rows (band rule against oracle.c)
    assert np.array_equal(gi, ci[:, :10]) and np.array_equal(gs, cs[:, :10])
    for q in range(len(Qb)):
        rows = np.sort(ci[q])
        oi, osc = oracle.flat_topk(Xb[rows], Qb[q:q + 1], 16)
        oi = np.where(oi >= 0, rows[np.maximum(oi, 0)], -1)
        r = check(gi[q:q + 1], gs[q:q + 1], oi, osc,
                  lambda _q, ids_: oracle.pair_scores(Xb, Qb[q:q + 1], np.zeros(len(ids_), int),
                                                      ids_), 10)
        assert r["ok"], (q, r)
    # end to end vs the exact search, wherever the exact top-10 is among the candidates
    _, _, orows = fp8.search(Xb, Qb, 10, n_cand)
    ei, _ = oracle.flat_topk(Xb, Qb, 10)
    covered = [q for q in range(len(Qb)) if set(ei[q]) <= set(orows[q])]
    assert len(covered) >= 0.97 * len(Qb)
    r = check_against_rows(gi[covered], gs[covered], Xb, Qb[covered], 10)
    assert r["ok"], r
    idx.free()


@pytest.mark.parametrize("nq", [1, 129])
def test_edges(sa, data, nq):
    Xb, Qb = data
    small = Xb[:250]
    idx = sa.Index.build(bits_to_tensor(small).cuda(), 0).build_fp8()
    Qd = bits_to_tensor(Qb[:nq]).cuda()
    # n_cand >= n: every row is a candidate -> the exact search
    gi, gs = idx.search_fp8(Qd, 10, 256)
    r = check_against_rows(gi.cpu().numpy(), gs.cpu().numpy(), small, Qb[:nq], 10)
    assert r["ok"], r
    tiny = sa.Index.build(bits_to_tensor(Xb[:7]).cuda(), 0).build_fp8()
    ti, ts = tiny.search_fp8(Qd, 10, 16)              # k > n: 7 rows then (-1, -inf)
    r = check_against_rows(ti.cpu().numpy(), ts.cpu().numpy(), Xb[:7], Qb[:nq], 10)
    assert r["ok"], r
    assert (ti[:, 7:] == -1).all() and torch.isinf(ts[:, 7:]).all()
    tiny.free()
    idx.free()


def test_errors(sa, data):
    Xb, Qb = data
    idx = sa.Index.build(bits_to_tensor(Xb[:1000]).cuda(), 0)
    Qd = bits_to_tensor(Qb[:4]).cuda()
    with pytest.raises(sa.SAError) as e:
        idx.search_fp8(Qd, 10, 32)
    assert e.value.status == sa.SA_ERR_STATE
    idx.build_fp8()
    with pytest.raises(sa.SAError):
        idx.search_fp8(Qd, 10, 257)
    with pytest.raises(sa.SAError):
        idx.search_fp8(Qd, 33, 32)
    idx.free()


def test_ivf_fp8_candidates_and_rerank(sa, data):
    """R35: with nprobe > 0 the e4m3 candidates come from the rows of the nprobe best lists
    (probed on the bf16 query, as sa_search): the GPU's candidate set = the oracle's e4m3
    top-n_cand over exactly those rows (band rule on fp8 scores), the result = the exact
    top-k over the GPU's candidates, and nprobe = nlist gives the flat fp8 candidates."""
    Xb, Qb = data
    idx = sa.Index.build(bits_to_tensor(Xb).cuda(), 32, kmeans_iters=4).build_fp8()
    Qd = bits_to_tensor(Qb).cuda()
    off, gid = idx.export_lists()
    X8, _ = fp8.quantize_corpus(Xb)
    Q8, _ = fp8.quantize_queries(Qb)
    Xc, Qc = fp8._as_bf16_bits(X8), fp8._as_bf16_bits(Q8)
    n_cand, nprobe = 16, 6
    P = idx.probes(Qd, nprobe).cpu().numpy()
    ci, cs = idx.search_fp8(Qd, n_cand, n_cand, nprobe=nprobe)
    ci = ci.cpu().numpy()
    gi, gs = idx.search_fp8(Qd, 10, n_cand, nprobe=nprobe)
    gi, gs = gi.cpu().numpy(), gs.cpu().numpy()
    assert np.array_equal(gi, ci[:, :10])
    for q in range(0, len(Qb), 3):
        rows = np.sort(np.concatenate([gid[off[l]:off[l + 1]] for l in P[q]]))
        oi, osc = oracle.flat_topk(Xc[rows], Qc[q:q + 1], min(n_cand + 8, rows.size))
        navail = min(n_cand, rows.size)
        sk = osc[0][navail - 1]
        t = tol_of(sk, 1e-3)
        must = set(rows[oi[0][(oi[0] >= 0) & (osc[0] > sk + t)]].tolist())
        got = set(ci[q][:navail].tolist())
        assert must <= got and len(got) == navail and got <= set(rows.tolist()), q
        s_g = oracle.pair_scores(Xc, Qc[q:q + 1], np.zeros(navail, int), ci[q][:navail])
        assert np.all(s_g >= sk - t), q
        # re-rank: exact top-10 over the GPU's candidates
        cr = np.sort(ci[q][:navail])
        ei, es = oracle.flat_topk(Xb[cr], Qb[q:q + 1], 10)
        ei = np.where(ei >= 0, cr[np.maximum(ei, 0)], -1)
        r = check(gi[q:q + 1], gs[q:q + 1], ei, es,
                  lambda _q, ids_: oracle.pair_scores(Xb, Qb[q:q + 1], np.zeros(len(ids_), int),
                                                      ids_), 10)
        assert r["ok"], (q, r)
    # nprobe = nlist: every row is probed -> the flat fp8 candidates
    fi, fsc = idx.search_fp8(Qd, n_cand, n_cand)
    ai, asc = idx.search_fp8(Qd, n_cand, n_cand, nprobe=32)
    same = np.mean([set(fi[q].tolist()) == set(ai[q].tolist()) for q in range(len(Qb))])
    assert same >= 0.97, same     # differ only where fp32 sums reorder the n_cand boundary
    with pytest.raises(sa.SAError):
        idx.search_fp8(Qd, 10, 16, nprobe=33)
    idx.free()


def test_power_of_two_scaling_is_exact(sa, data):
    """P8-ii for the fp8 modes: scaling a query by 2^j leaves its e4m3 codes unchanged (R31's
    per-row exponent absorbs it), so the candidates are identical and the re-ranked scores are
    the originals times 2^j exactly (flat and IVF)."""
    Xb, Qb = data
    idx = sa.Index.build(bits_to_tensor(Xb).cuda(), 32, kmeans_iters=4).build_fp8()
    Qd = bits_to_tensor(Qb).cuda()
    for nprobe in (0, 6):
        gi, gs = idx.search_fp8(Qd, 10, 16, nprobe=nprobe)
        for j in (-2, 3):
            qj = (Qd.float() * 2.0 ** j).to(torch.bfloat16)
            si, ss = idx.search_fp8(qj, 10, 16, nprobe=nprobe)
            assert torch.equal(si, gi) and torch.equal(ss, gs * 2.0 ** j), (nprobe, j)
    idx.free()

"""Parity at BASELINE.json's full size (C3: 21,015,324 x 768 bf16, batch 512, top-10) in the
launch configuration bench.py times, on sampled outputs the oracle computes one by one
(tests/parity.py band rule), plus IVF (nlist=16384) properties at full size."""
import numpy as np
import pytest
import torch

import oracle
from datagen import CONFIGS, CORPUS_SEED, QUERY_SEED, make_mixture, draw_rows_into
from parity import check

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SAMPLE_Q = [0, 1, 77, 255, 256, 300, 511]        # both query groups, both CTA halves, ragged


def _bits(t):
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


@pytest.fixture(scope="module")
def c3(sa):
    cfg = CONFIGS["c3"]
    n, d, nq = cfg["n"], cfg["d"], cfg["nq"]
    mix = make_mixture(d, cfg["C"], cfg["r"], cfg["s_sub"], cfg["s_n"], CORPUS_SEED, "cuda")
    X = torch.empty(n, d, dtype=torch.bfloat16, device="cuda")
    draw_rows_into(mix, X, CORPUS_SEED, 0)
    Q = torch.empty(nq, d, dtype=torch.bfloat16, device="cuda")
    draw_rows_into(mix, Q, QUERY_SEED, 0)
    flat = sa.Index.build(X)
    ids, sc = flat.search(Q, 10)
    torch.cuda.synchronize()
    # oracle over the whole corpus for the sampled queries, streamed in 2^21-row chunks
    Qb = _bits(Q)[SAMPLE_Q]
    top = oracle.TopK(Qb, 10 + 16)
    chunk = 1 << 21
    for lo in range(0, n, chunk):
        top.update(_bits(X[lo:lo + chunk]), lo)
    flat.free()
    yield dict(X=X, Q=Q, ids=ids.cpu().numpy(), sc=sc.cpu().numpy(), top=top, Qb=Qb)


def test_c3_exact_sampled_parity(c3):
    X, Qb, top = c3["X"], c3["Qb"], c3["top"]
    gi, gs = c3["ids"][SAMPLE_Q], c3["sc"][SAMPLE_Q]

    def score_of(qi, ids):
        rows = _bits(X[torch.as_tensor(ids, device="cuda")])
        return oracle.pair_scores(rows, Qb[qi:qi + 1], np.zeros(len(ids), int), np.arange(len(ids)))

    rep = check(gi, gs, top.ids, top.scores, score_of, 10)
    assert rep["ok"], rep
    rep5 = check(gi, gs, top.ids, top.scores, score_of, 10, rtol=1e-5)
    assert rep5["ok"], rep5


def test_c3_exact_properties_all_queries(c3):
    ids, sc = c3["ids"], c3["sc"]
    n = CONFIGS["c3"]["n"]
    assert np.all((ids >= 0) & (ids < n))
    for q in range(ids.shape[0]):
        assert len(set(ids[q].tolist())) == 10
        for j in range(9):   # strict (score desc, id asc)
            assert sc[q, j] > sc[q, j + 1] or (sc[q, j] == sc[q, j + 1] and ids[q, j] < ids[q, j + 1])


def test_c3_ivf_full_size(sa, c3):
    X, Q = c3["X"], c3["Q"]
    idx = sa.Index.build(X, 16384)
    off, gid = idx.export_lists()
    n = X.shape[0]
    assert off[-1] == n and np.array_equal(np.sort(gid), np.arange(n))
    # nprobe = 48 (bench's calibrated point): recall vs the exact result over all 512 queries
    ii, isc = idx.search(Q, 10, nprobe=48)
    ii = ii.cpu().numpy()
    rec = np.mean([len(set(ii[q]) & set(c3["ids"][q])) / 10 for q in range(len(ii))])
    assert rec >= 0.95, rec
    # P11 on sampled queries: result == exact top-k over the rows of the probed lists
    P = idx.probes(Q, 48).cpu().numpy()
    Qb_all = _bits(Q)
    Xl = idx  # rows of a list = stored rows off[l]:off[l+1] -> global ids gid[...]
    for q in SAMPLE_Q:
        rows = np.sort(np.concatenate([gid[off[l]:off[l + 1]] for l in P[q]]))
        Xr = _bits(X[torch.as_tensor(rows, device="cuda")])
        oi, osc = oracle.flat_topk(Xr, Qb_all[q:q + 1], 10 + 8)
        oi = np.where(oi >= 0, rows[np.maximum(oi, 0)], -1)
        rep = check(ii[q:q + 1], isc.cpu().numpy()[q:q + 1], oi, osc,
                    lambda _q, ids_: oracle.pair_scores(
                        _bits(X[torch.as_tensor(ids_, device="cuda")]), Qb_all[q:q + 1],
                        np.zeros(len(ids_), int), np.arange(len(ids_))), 10)
        assert rep["ok"], (q, rep)
    # exact mode on the IVF (list-major) index == exact mode on the flat index, bit-exact
    ei, es = idx.search(Q, 10, nprobe=0)
    assert np.array_equal(ei.cpu().numpy(), c3["ids"]) and np.array_equal(es.cpu().numpy(), c3["sc"])
    del Xl
    idx.free()


def test_c3_graph_and_fp8_full_size(sa, c3):
    """The headline graph mode (degree 48, L = 104, w = 4, 16 entry lists: bench.py's
    calibrated point) and the fp8 scan + re-rank at full size: recall against the exact result
    over all 512 queries, returned scores = the fp64 oracle's scores of the returned ids (band
    rule) on the sampled queries, strict order, batch invariance of the graph search."""
    X, Q = c3["X"], c3["Q"]
    idx = sa.Index.build(X, 16384)
    idx.build_graph(knn_k=64, degree=48, nprobe_build=8)
    idx.build_fp8()
    Qb_all = _bits(Q)
    exact = c3["ids"]

    def scores_ok(ids, sc, q):
        rows = _bits(X[torch.as_tensor(ids, device="cuda")])
        ps = oracle.pair_scores(rows, Qb_all[q:q + 1], np.zeros(len(ids), int), np.arange(len(ids)))
        return np.all(np.abs(ps - sc) <= 1e-3 * np.maximum(np.abs(ps), 1e-3))

    gi, gs = idx.search_graph(Q, 10, 104, search_width=4, n_entries=16)
    gi, gs = gi.cpu().numpy(), gs.cpu().numpy()
    rec = np.mean([len(set(gi[q]) & set(exact[q])) / 10 for q in range(len(gi))])
    assert rec >= 0.95, rec
    for q in SAMPLE_Q:
        assert scores_ok(gi[q], gs[q], q), q
        assert len(set(gi[q].tolist())) == 10
        for j in range(9):
            assert gs[q, j] > gs[q, j + 1] or (gs[q, j] == gs[q, j + 1] and gi[q, j] < gi[q, j + 1])
    for q in (0, 300):   # alone (1024-thread shape) == inside the 512 batch (256-thread shape)
        si, ss = idx.search_graph(Q[q:q + 1].contiguous(), 10, 104, search_width=4, n_entries=16)
        assert np.array_equal(si.cpu().numpy()[0], gi[q]) and np.array_equal(ss.cpu().numpy()[0], gs[q])
    fi, fs = idx.search_fp8(Q, 10, 16)
    fi, fs = fi.cpu().numpy(), fs.cpu().numpy()
    same = np.mean([np.array_equal(fi[q], exact[q]) for q in range(len(fi))])
    assert same >= 0.99, same
    for q in SAMPLE_Q:
        assert scores_ok(fi[q], fs[q], q), q
    # IVF on the e4m3 copy (R35) at bench.py's point: recall vs exact, returned scores
    vi, vs = idx.search_fp8(Q, 10, 16, nprobe=48)
    vi, vs = vi.cpu().numpy(), vs.cpu().numpy()
    rec8 = np.mean([len(set(vi[q]) & set(exact[q])) / 10 for q in range(len(vi))])
    assert rec8 >= 0.95, rec8
    for q in SAMPLE_Q:
        assert scores_ok(vi[q], vs[q], q), q
    idx.free()


def test_c3_agent_step_shapes(sa, c3):
    """BASELINE config 5 shapes at full size (batches of 1 and 64, top-5): the exact and IVF
    results of a small batch equal the first 5 entries of the same queries' batch-512 top-10
    bit for bit (P8-i: each query's scores do not depend on the batch it is in)."""
    X, Q = c3["X"], c3["Q"]
    flat = sa.Index.build(X)
    for b in (1, 64):
        qi, qs = flat.search(Q[:b].contiguous(), 5)
        assert np.array_equal(qi.cpu().numpy(), c3["ids"][:b, :5])
        assert np.array_equal(qs.cpu().numpy(), c3["sc"][:b, :5])
    flat.free()
    idx = sa.Index.build(X, 16384)
    bi, bs = idx.search(Q, 10, nprobe=48)
    for b in (1, 64):
        qi, qs = idx.search(Q[:b].contiguous(), 5, nprobe=48)
        assert np.array_equal(qi.cpu().numpy(), bi.cpu().numpy()[:b, :5])
        assert np.array_equal(qs.cpu().numpy(), bs.cpu().numpy()[:b, :5])
    idx.free()

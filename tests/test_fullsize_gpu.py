"""Parity at BASELINE.json's full size (C3: 21,015,324 x 768 bf16, batch 512, top-10) in the
launch configuration bench.py times, on sampled outputs the oracle computes one by one
(tests/parity.py band rule): queries 0-63 of the seed-5678 stream plus tile / CTA-half edge
queries, and P7 planted winners at rows {0, 127, 128, 255, 256, n-1} and at every shard
boundary +-1 of w = 2, 4, 8.  The row-sharded library path (w = 2 and 8
in-process ranks, bench.py's per-rank launch configuration at N = 8) equals the unsharded
result bit for bit.  Plus IVF (nlist=16384), graph and fp8 properties at full size."""
import numpy as np
import pytest
import torch

import oracle
from datagen import CONFIGS, CORPUS_SEED, QUERY_SEED, make_mixture, draw_rows_into
from parity import check

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SAMPLE_Q = [0, 1, 77, 255, 256, 300, 511]        # both query groups, both CTA halves, ragged
PARITY_Q = list(range(64)) + [77, 255, 256, 300, 511]  # oracle parity over these


def planted_rows(n):
    """P7: tile edges, the last row, and every shard boundary +-1 for w = 2, 4, 8."""
    rows = {0, 127, 128, 255, 256, n - 1}
    for w in (2, 4, 8):
        for r in range(1, w):
            off = r * (n // w) + min(r, n % w)
            rows.update({off - 1, off, off + 1})
    return sorted(rows)


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
    # P7 planted winners: query j of a separate seeded stream is planted (x 2, exact in bf16)
    # at row planted[j]; it beats every unit-norm row for its own query
    planted = planted_rows(n)
    Qp = torch.empty(len(planted), d, dtype=torch.bfloat16, device="cuda")
    draw_rows_into(mix, Qp, QUERY_SEED + 4321, 0)
    X[torch.as_tensor(planted, device="cuda")] = (Qp.float() * 2.0).to(torch.bfloat16)
    flat = sa.Index.build(X)
    ids, sc = flat.search(Q, 10)
    pid, psc = flat.search(Qp, 10)
    torch.cuda.synchronize()
    # oracle over the whole corpus for the parity queries, streamed in 2^21-row chunks
    Qb = np.concatenate([_bits(Q)[PARITY_Q], _bits(Qp)])
    top = oracle.TopK(Qb, 10 + 16)
    chunk = 1 << 21
    for lo in range(0, n, chunk):
        top.update(_bits(X[lo:lo + chunk]), lo)
    flat.free()
    yield dict(X=X, Q=Q, Qp=Qp, planted=planted, ids=ids.cpu().numpy(), sc=sc.cpu().numpy(),
               pid=pid.cpu().numpy(), psc=psc.cpu().numpy(), top=top, Qb=Qb)


def test_c3_exact_parity_queries_0_63_and_planted(c3):
    X, Qb, top = c3["X"], c3["Qb"], c3["top"]
    gi = np.concatenate([c3["ids"][PARITY_Q], c3["pid"]])
    gs = np.concatenate([c3["sc"][PARITY_Q], c3["psc"]])

    def score_of(qi, ids):
        rows = _bits(X[torch.as_tensor(ids, device="cuda")])
        return oracle.pair_scores(rows, Qb[qi:qi + 1], np.zeros(len(ids), int), np.arange(len(ids)))

    rep = check(gi, gs, top.ids, top.scores, score_of, 10)
    assert rep["ok"], rep
    rep5 = check(gi, gs, top.ids, top.scores, score_of, 10, rtol=1e-5)
    assert rep5["ok"], rep5
    assert c3["pid"][:, 0].tolist() == c3["planted"]          # P7: every planted winner first
    print(f"C3 parity: {len(gi)} queries, band median {rep['band_median']}, "
          f"max {rep['band_max']}, max rel score err {rep['max_rel_score_err']:.2e}")


def _run_ranks(world, fn):
    import threading
    out, err = [None] * world, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                out[r] = fn(r)
                torch.cuda.current_stream().synchronize()
        except BaseException as e:  # noqa: BLE001 -- re-raised below
            err.append(e)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=1200)
    if err:
        raise err[0]
    return out


@pytest.mark.parametrize("world", [2, 8])
def test_c3_row_sharded_library_path(sa, c3, world):
    """sa_search on w row shards (in-process communicator: the library's own all-gather +
    merge branch, each rank in bench.py's per-rank launch configuration) == the unsharded
    result bit for bit, for the 512-query batch and the planted queries (P8-iii at C3)."""
    X, Q, Qp = c3["X"], c3["Q"], c3["Qp"]
    n = X.shape[0]
    comms = sa.Comm.local_group(world)

    def rank(r):
        off, ln = sa.shard_range(n, r, world)
        idx = sa.Index.build(X[off:off + ln], row_offset=off, n_total=n, comm=comms[r])
        a = [t.cpu().numpy() for t in idx.search(Q, 10)]
        b = [t.cpu().numpy() for t in idx.search(Qp, 10)]
        idx.free()
        return a, b

    res = _run_ranks(world, rank)
    for c in comms:
        c.free()
    for a, b in res:
        assert np.array_equal(a[0], c3["ids"]) and np.array_equal(a[1], c3["sc"])
        assert np.array_equal(b[0], c3["pid"]) and np.array_equal(b[1], c3["psc"])


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
    bi, bs = bi.cpu().numpy(), bs.cpu().numpy()
    qi, qs = idx.search(Q[:64].contiguous(), 5, nprobe=48)      # batch path: bit for bit
    assert np.array_equal(qi.cpu().numpy(), bi[:64, :5])
    assert np.array_equal(qs.cpu().numpy(), bs[:64, :5])
    # batches of <= 8 take the one-launch path (CUDA-core sums): the same ids except at
    # near-ties of the 5th score, scores within fp32 rounding
    for b in (1, 8):
        si, ss = idx.search(Q[:b].contiguous(), 5, nprobe=48)
        si, ss = si.cpu().numpy(), ss.cpu().numpy()
        assert np.allclose(ss, bs[:b, :5], rtol=1e-5, atol=1e-7)
        for q in range(b):
            for i in set(si[q].tolist()) ^ set(bi[q, :5].tolist()):
                s = float(ss[q][list(si[q]).index(i)]) if i in si[q] else float(bs[q][list(bi[q]).index(i)])
                assert abs(s - bs[q, 4]) <= 1e-5 * max(abs(bs[q, 4]), 1e-3), (b, q, i)
    idx.free()

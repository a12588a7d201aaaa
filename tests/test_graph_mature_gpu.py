"""Non-stall maturity exit on the GPU beam search (sa_search_graph_mature) against
oracle/graph.py's search(tau=...).

PAPER.md §3.3 P:167-177 (RQ_t, EMA, "exceeds a threshold tau and the LLM engine is ready"),
App. B.2; readings R27-R29.
  * golden: GR5's hand-evaluated path-graph trace (tests/test_graph_oracle.py) bit-exactly on
    the GPU -- RQ / EMA per step, exit step and result for tau = inf / 0 / never ready / g = 3
    (scores there are exact in fp32, so both sides compute the same bits);
  * mixture: on the GPU's own graph and entry points, for the queries whose plain beam search
    equals the oracle's, the per-step RQ / EMA agree within the error propagated from fp32
    scores, and the exit step equals the oracle's unless the oracle's EMA sits within that
    error of tau at a checkpoint;
  * prefix property: the result of a search that exits at step t is bit-identical to the plain
    search capped at t iterations; engine never ready -> the plain search, bit-exactly.
"""
import math

import numpy as np
import pytest
import torch

from oracle import graph
from datagen import make_mixture, draw_rows, to_bf16_bits
from test_graph_oracle import path_graph
from test_graph_gpu import bits_to_tensor, entries_of

pytestmark = pytest.mark.gpu


def flag(v, device=False):
    f = torch.full((1,), v, dtype=torch.int32)
    return f.cuda() if device else f.pin_memory()


def test_gr5_golden_trace_bit_exact(sa):
    X, nbr, q = path_graph()
    idx = sa.Index.build(bits_to_tensor(X).cuda(), 1,
                         centroids=torch.ones(1, X.shape[1], dtype=torch.float32).cuda())
    idx.import_graph(nbr)
    assert np.array_equal(idx.export_graph(), nbr)
    Qd = bits_to_tensor(q).cuda()
    kw = dict(search_width=1, n_entries=1)
    gi, gs, st, rq, ema = idx.search_graph_mature(Qd, 2, 2, tau=math.inf, window=3,
                                                  trace_cols=6, **kw)
    torch.cuda.synchronize()
    o = graph.search(X, nbr, q[0], 2, L=2, w=1, entries=[0], T=100, tau=math.inf, window=3)
    assert int(st[0]) == o["iterations"] == 4
    rq, ema = rq.cpu().numpy()[0], ema.cpu().numpy()[0]
    assert rq[:4].tolist() == o["rq"].tolist() == [0.0, 0.0, 0.0, 1.0]
    assert ema[:4].tolist() == o["ema"].tolist() == [0.0, 0.0, 0.0, 0.5]
    assert np.isnan(rq[4:]).all() and np.isnan(ema[4:]).all()
    assert gi.cpu().tolist()[0] == [3, 2] and gs.cpu().tolist()[0] == [0.5, 0.375]
    # (tau, g, ready) -> (steps, ids): GR5's exit lines
    for tau, g, ready, steps, ids in ((0.0, 1, True, 1, [1, 0]), (0.0, 1, False, 4, [3, 2]),
                                      (0.0, 3, True, 3, [3, 2]), (0.5, 1, True, 4, [3, 2]),
                                      (0.6, 1, True, 4, [3, 2])):
        for dev in (False, True):
            gi, gs, st = idx.search_graph_mature(Qd, 2, 2, tau=tau, window=3, check_every=g,
                                                 engine_ready=flag(1 if ready else 0, dev), **kw)
            torch.cuda.synchronize()
            o = graph.search(X, nbr, q[0], 2, L=2, w=1, entries=[0], T=100, tau=tau, window=3,
                             g=g, ready=ready)
            assert int(st[0]) == o["iterations"] == steps, (tau, g, ready)
            assert gi.cpu().tolist()[0] == o["ids"].tolist() == ids
    idx.free()


@pytest.fixture(scope="module")
def mixture(sa):
    mx = make_mixture(d=128, C=16, r=16, s_n=0.7)
    X = draw_rows(mx, 12_000, row_seed=81)
    Q = draw_rows(mx, 64, row_seed=82)
    Xb, Qb = to_bf16_bits(X), to_bf16_bits(Q)
    idx = sa.Index.build(bits_to_tensor(Xb).cuda(), 16, kmeans_iters=8)
    idx.build_graph(knn_k=24, degree=16, nprobe_build=3)
    nbr = idx.export_graph()
    yield idx, Xb, Qb, nbr, entries_of(idx, Qb, 4)
    idx.free()


def test_trace_and_exit_match_oracle(sa, mixture):
    idx, Xb, Qb, nbr, ent = mixture
    Qd = bits_to_tensor(Qb).cuda()
    L, w, W, T = 64, 2, 8, 200
    pi, ps, px, _ = idx.search_graph(Qd, 10, L, search_width=w, n_entries=4, expanded=True)
    gi, gs, st, rq, ema = idx.search_graph_mature(Qd, 10, L, tau=math.inf, window=W,
                                                  search_width=w, n_entries=4, trace_cols=T)
    pi, px, st = pi.cpu().numpy(), px.cpu().numpy(), st.cpu().numpy()
    rq, ema = rq.cpu().numpy(), ema.cpu().numpy()
    # tau = inf never exits: the plain search, bit-exactly
    assert np.array_equal(gi.cpu().numpy(), pi) and torch.equal(gs, ps)
    taus, certified, err = [], set(), 0.0
    for q in range(len(Qb)):
        o = graph.search(Xb, nbr, Qb[q], 10, L=L, w=w, entries=ent[q], T=10_000,
                         tau=math.inf, window=W)
        same = np.array_equal(pi[q], o["ids"]) and px[q] == o["expanded"]
        # identical path unless the oracle's path crosses a near-tie the fp32 error bound
        # cannot separate (oracle/graph.py `certified`); only then may traces differ
        assert same or not o["certified"], q
        if not o["certified"]:
            continue
        certified.add(q)
        n = o["iterations"]
        assert st[q] == n
        assert np.all(np.abs(rq[q, :n] - o["rq"]) <= 2e-3), q
        assert np.all(np.abs(ema[q, :n] - o["ema"]) <= 2e-3), q
        assert np.isnan(rq[q, n:]).all()
        err = max(err, float(np.abs(ema[q, :n] - o["ema"]).max()))
        taus.append(np.median(o["ema"]))
    print(f"graph maturity: {len(certified)} of {len(Qb)} paths certified, max EMA error {err:.2e}")
    # a finite tau: on certified paths the exit step equals the oracle's unless its EMA at a
    # checkpoint lies within the measured GPU-vs-oracle EMA error (x4) of tau
    band = 4 * max(err, 1e-9)
    tau = float(np.median(taus))
    for g in (1, 3):
        gi, gs, st = idx.search_graph_mature(Qd, 10, L, tau=tau, window=W, check_every=g,
                                             search_width=w, n_entries=4)
        st = st.cpu().numpy()
        agree = checked = 0
        for q in sorted(certified):
            o = graph.search(Xb, nbr, Qb[q], 10, L=L, w=w, entries=ent[q], T=10_000,
                             tau=tau, window=W, g=g)
            e = o["ema"]
            if any(abs(e[t - 1] - tau) <= band for t in range(g, len(e) + 1, g)):
                continue
            checked += 1
            agree += st[q] == o["iterations"]
        assert agree == checked and checked >= len(certified) - 2, (g, agree, checked)


def test_prefix_property_and_readiness(sa, mixture):
    idx, Xb, Qb, nbr, ent = mixture
    Qd = bits_to_tensor(Qb).cuda()
    L, w = 64, 2
    gi, gs, st = idx.search_graph_mature(Qd, 10, L, tau=0.5, window=4, search_width=w,
                                         n_entries=4)
    st = st.cpu()
    assert int(st.min()) >= 1
    for t in sorted(set(st.tolist()))[:6]:
        rows = (st == t).nonzero().flatten().tolist()
        ci, cs = idx.search_graph(Qd, 10, L, search_width=w, n_entries=4, max_iters=t)
        for r in rows:
            assert torch.equal(gi[r], ci[r]) and torch.equal(gs[r], cs[r]), (t, r)
    # never ready: the natural stop, i.e. the plain search
    pi, ps = idx.search_graph(Qd, 10, L, search_width=w, n_entries=4)
    for dev in (False, True):
        ni, ns, _ = idx.search_graph_mature(Qd, 10, L, tau=0.0, window=4, search_width=w,
                                            n_entries=4, engine_ready=flag(0, dev))
        assert torch.equal(ni, pi) and torch.equal(ns, ps)
    # tau = 0 with the engine ready: every query stops after its first step
    _, _, s0 = idx.search_graph_mature(Qd, 10, L, tau=0.0, window=4, search_width=w,
                                       n_entries=4)
    assert torch.all(s0 == 1)


def test_errors(sa, mixture):
    idx, Xb, Qb, nbr, ent = mixture
    Qd = bits_to_tensor(Qb).cuda()
    with pytest.raises(sa.SAError):
        idx.search_graph_mature(Qd, 10, 64, tau=0.5, window=0)
    with pytest.raises(sa.SAError):
        idx.search_graph_mature(Qd, 10, 64, tau=float("nan"), window=4)
    with pytest.raises(sa.SAError):
        idx.search_graph_mature(Qd, 10, 64, tau=0.5, window=4, check_every=0)
    with pytest.raises(sa.SAError):
        idx.import_graph(np.full((Xb.shape[0], 4), Xb.shape[0] + 5, dtype=np.int64))

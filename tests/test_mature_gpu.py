"""Non-stall maturity exit on the GPU (sa_search_mature) against oracle/maturity.py.

PAPER.md §3.3, App. B.2; readings R14-R19.
  * golden: the hand-evaluated 5-list trace (tests/golden/maturity_trace.txt) bit-exactly,
    every exit line (tau, g, engine ready or not);
  * mixture (50k x 128, nlist 64): per-step RQ / EMA within the error propagated from the
    fp32 scores, exit step equal to the oracle's unless the oracle's EMA sits within that
    error of tau, results = exact top-k over the first t_exit probed lists (band rule);
  * engine readiness: flag 0 -> natural stop; a flag raised while the search runs stops it
    early, and the result is still the exact prefix result.
"""
import math
import time

import numpy as np
import pytest
import torch

import oracle
from oracle import ivf, maturity
from datagen import make_mixture, draw_rows, to_bf16_bits
from parity import check
from test_maturity_oracle import golden_geometry, load_golden

pytestmark = pytest.mark.gpu


def bits_to_tensor(b):
    return torch.from_numpy(np.ascontiguousarray(b).view(np.int16).copy()).view(torch.bfloat16)


def pinned_flag(v):
    f = torch.zeros(1, dtype=torch.int32).pin_memory()
    f[0] = v
    return f


def test_golden_trace_bit_exact(sa):
    X, lists, C, Q, k, window = golden_geometry()
    _, _, _, _, steps, exits = load_golden()
    idx = sa.Index.build(bits_to_tensor(X).cuda(), 5,
                         centroids=torch.from_numpy(C.astype(np.float32)).cuda())
    off, ids = idx.export_lists()
    for j in range(5):
        assert list(ids[off[j]:off[j + 1]]) == list(lists[j])
    Qd = bits_to_tensor(Q).cuda()
    gi, gs, gt, rq, ema = idx.search_mature(Qd, k, 5, tau=math.inf, window=window, trace=True)
    torch.cuda.synchronize()
    assert int(gt[0]) == 5
    rq, ema = rq.cpu().numpy()[0], ema.cpu().numpy()[0]
    for (t, l, s_t, r, e) in steps:
        assert rq[t - 1] == r and ema[t - 1] == e, (t, rq, ema)
    never = pinned_flag(0)
    for tau, g, ready, t_exit, want in exits:
        gi, gs, gt = idx.search_mature(Qd, k, 5, tau=tau, window=window, check_every=g,
                                       engine_ready=None if ready else never)
        torch.cuda.synchronize()
        assert int(gt[0]) == t_exit, (tau, g, ready)
        assert gi.cpu().tolist()[0] == want
    idx.free()


@pytest.fixture(scope="module")
def mix(sa):
    mx = make_mixture(d=128, C=16, r=16, s_n=0.7)
    X = draw_rows(mx, 50_000, row_seed=31)
    Q = draw_rows(mx, 24, row_seed=32)
    Xb, Qb = to_bf16_bits(X), to_bf16_bits(Q)
    idx = sa.Index.build(bits_to_tensor(Xb).cuda(), 64, kmeans_iters=8)
    off, ids = idx.export_lists()
    lists = [ids[off[j]:off[j + 1]] for j in range(64)]
    yield idx, Xb, Qb, lists
    idx.free()


def ema_error_bound(o, window, delta, k):
    """|GPU - oracle| bounds of RQ_t / EMA_t when every score is off by <= delta."""
    a = 2.0 / (window + 1)
    brq, bema = [], []
    for t in range(len(o["rq"])):
        den = o["s_best"][t] - o["s_worst"][t]
        if not np.isfinite(o["s_t"][t]) or k == 1:
            b = 0.0                     # empty list / single-entry list: RQ = 1 on both sides
        elif den <= 4 * delta:
            b = math.inf                # s_best ~ s_worst: the ratio is ill-conditioned
        else:
            b = 2 * delta * (1 + abs(o["rq"][t])) / (den - 2 * delta)
        brq.append(b)
        bema.append(b if t == 0 else a * b + (1 - a) * bema[-1])
    return np.array(brq), np.array(bema)


def check_prefix_result(gi, gs, Xb, Qb, qi, rows, k):
    oi, osc = oracle.flat_topk(Xb[rows], Qb[qi:qi + 1], k + 8)
    oi = np.where(oi >= 0, rows[np.maximum(oi, 0)], -1)
    r = check(gi[qi:qi + 1], gs[qi:qi + 1], oi, osc,
              lambda _q, ids_: oracle.pair_scores(Xb, Qb[qi:qi + 1], np.zeros(len(ids_), int), ids_),
              k, n_avail=min(k, len(rows)))
    assert r["ok"], (qi, r)


@pytest.mark.parametrize("k,P,tau,window,g", [
    (10, 24, 2.0, 8, 1),
    (10, 24, 1.0, 4, 3),
    (5, 32, 3.0, 16, 2),
    (1, 12, 0.9, 4, 1),
    (50, 16, 1.5, 8, 4),
    (10, 20, math.inf, 8, 5),
])
@pytest.mark.parametrize("nq", [24, 8])
def test_matches_oracle_on_mixture(sa, mix, k, P, tau, window, g, nq):
    """nq = 24: the captured-graph stage loop; nq = 8 (and k <= 32, 8 g <= 64): the one-launch
    kernel whose stages are closed on the device (ivf_small.cu).  The oracle walks the probe
    order of the batch probe; a query whose first P + 1 probe ranks hold an fp32 near-tie may
    be ordered differently by the one-launch path's CUDA-core probe and is skipped."""
    idx, Xb, Qb, lists = mix
    Qb = Qb[:nq]
    Qd = bits_to_tensor(Qb).cuda()
    C = oracle.bf16_to_f64(oracle.bf16_round(np.asarray(idx.export_centroids(), np.float32)))
    Q64 = oracle.bf16_to_f64(Qb)
    pc = Q64 @ C.T
    eb = 2 * (Q64.shape[1] - 1) * 2.0 ** -24 * (np.abs(Q64) @ np.abs(C).T)
    probes = idx.probes(Qd, P).cpu().numpy()
    gi, gs, gt, grq, gema = idx.search_mature(Qd, k, P, tau=tau, window=window, check_every=g,
                                              trace=True)
    torch.cuda.synchronize()
    gi, gs, gt = gi.cpu().numpy(), gs.cpu().numpy(), gt.cpu().numpy()
    grq, gema = grq.cpu().numpy(), gema.cpu().numpy()
    delta = 1e-5
    exits = []
    skipped = 0
    for qi in range(len(Qb)):
        ranked = probes[qi][:P].tolist() + [int(j) for j in np.argsort(-pc[qi]) if j not in
                                            set(probes[qi][:P].tolist())][:1]
        gaps = [pc[qi, ranked[i]] - pc[qi, ranked[i + 1]] - eb[qi, ranked[i]] - eb[qi, ranked[i + 1]]
                for i in range(len(ranked) - 1)]
        if min(gaps) <= 0:
            skipped += 1
            continue
        o = maturity.search_query(Xb, lists, probes[qi], Qb[qi], k, tau=math.inf, window=window)
        brq, bema = ema_error_bound(o, window, delta, k)
        t = int(gt[qi])
        assert 1 <= t <= P
        assert np.all(np.isnan(grq[qi, t:])) and not np.any(np.isnan(grq[qi, :t]))
        assert np.all(np.abs(grq[qi, :t] - o["rq"][:t]) <= brq[:t] + 1e-12), qi
        assert np.all(np.abs(gema[qi, :t] - o["ema"][:t]) <= bema[:t] + 1e-12), qi
        # the oracle's exit with the same rule; a different step only where EMA ~ tau
        t_or = maturity.maturity_point(o["ema"], tau, g) or P
        if t != t_or:
            tt = min(t, t_or)
            assert abs(o["ema"][tt - 1] - tau) <= bema[tt - 1] + 1e-12, (qi, t, t_or)
        if t < P:
            assert t % g == 0 and gema[qi, t - 1] >= tau
        # earlier checkpoints did not pass on the GPU's own signal
        for c in range(g, t, g):
            assert gema[qi, c - 1] < tau
        rows = np.sort(np.concatenate([lists[j] for j in probes[qi][:t]]))
        check_prefix_result(gi, gs, Xb, Qb, qi, rows, k)
        exits.append(t)
    assert skipped <= max(2, len(Qb) // 6), skipped
    if tau == math.inf:
        assert all(t == P for t in exits)


def test_engine_flag_gates_the_exit(sa, mix):
    idx, Xb, Qb, lists = mix
    Qd = bits_to_tensor(Qb).cuda()
    never = pinned_flag(0)
    _, _, gt = idx.search_mature(Qd, 10, 16, tau=0.0, window=4, check_every=2, engine_ready=never)
    torch.cuda.synchronize()
    assert np.all(gt.cpu().numpy() == 16)             # never ready: natural stop
    ready = pinned_flag(1)
    _, _, gt = idx.search_mature(Qd, 10, 16, tau=0.0, window=4, check_every=2, engine_ready=ready)
    torch.cuda.synchronize()
    assert np.all(gt.cpu().numpy() == 2)              # ready and EMA >= 0: first checkpoint
    dev_flag = torch.ones(1, dtype=torch.int32, device="cuda")
    _, _, gt = idx.search_mature(Qd, 10, 16, tau=0.0, window=4, check_every=4,
                                 engine_ready=dev_flag)
    torch.cuda.synchronize()
    assert np.all(gt.cpu().numpy() == 4)


def test_flag_raised_mid_search_stops_it(sa, mix):
    """The host raises the flag while the device loop runs (Alg. 1 line 10-11)."""
    idx, Xb, Qb, lists = mix
    Qd = bits_to_tensor(Qb[:4]).cuda()
    flag = pinned_flag(0)
    P = 64
    args = dict(tau=0.0, window=4, check_every=1, engine_ready=flag)
    idx.search_mature(Qd, 10, P, **args)               # capture the graph first
    torch.cuda.synchronize()
    flag[0] = 0
    gi, gs, gt = idx.search_mature(Qd, 10, P, **args)
    time.sleep(0.0002)
    flag[0] = 1
    torch.cuda.synchronize()
    gt = gt.cpu().numpy()
    assert np.all((gt >= 1) & (gt < P)), gt
    gi, gs = gi.cpu().numpy(), gs.cpu().numpy()
    probes = idx.probes(Qd, P).cpu().numpy()
    for qi in range(4):
        rows = np.sort(np.concatenate([lists[j] for j in probes[qi][:gt[qi]]]))
        check_prefix_result(gi, gs, Xb, Qb[:4], qi, rows, 10)


def test_k256_and_single_query(sa, mix):
    idx, Xb, Qb, lists = mix
    Qd = bits_to_tensor(Qb[:1]).cuda()
    probes = idx.probes(Qd, 8).cpu().numpy()
    gi, gs, gt = idx.search_mature(Qd, 256, 8, tau=1.0, window=4, check_every=2)
    torch.cuda.synchronize()
    t = int(gt.cpu()[0])
    rows = np.sort(np.concatenate([lists[j] for j in probes[0][:t]]))
    check_prefix_result(gi.cpu().numpy(), gs.cpu().numpy(), Xb, Qb[:1], 0, rows, 256)


def test_invalid_and_unsupported(sa, mix):
    idx, Xb, Qb, lists = mix
    Qd = bits_to_tensor(Qb[:4]).cuda()
    with pytest.raises(sa.SAError) as e:
        idx.search_mature(Qd, 10, 65, tau=1.0, window=4)
    assert e.value.status == sa.SA_ERR_INVALID_ARG
    with pytest.raises(sa.SAError) as e:
        idx.search_mature(Qd, 10, 8, tau=1.0, window=0)
    assert e.value.status == sa.SA_ERR_INVALID_ARG
    big = torch.zeros(4097, 128, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(sa.SAError) as e:
        idx.search_mature(big, 10, 8, tau=1.0, window=4)
    assert e.value.status == sa.SA_ERR_UNSUPPORTED
    flat = sa.Index.build(bits_to_tensor(Xb[:1000]).cuda(), 0)
    with pytest.raises(sa.SAError) as e:
        flat.search_mature(Qd, 10, 8, tau=1.0, window=4)
    assert e.value.status == sa.SA_ERR_STATE
    flat.free()

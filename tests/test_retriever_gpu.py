"""Asynchronous retrieval tasks (sa_retriever_*, Alg. 1) on the GPU: results equal the
synchronous calls bit for bit, slots are bounded, the engine-ready flag reaches running
maturity searches."""
import time

import numpy as np
import pytest
import torch

from datagen import make_mixture, draw_rows, to_bf16_bits

pytestmark = pytest.mark.gpu


def bits_to_tensor(b):
    return torch.from_numpy(np.ascontiguousarray(b).view(np.int16).copy()).view(torch.bfloat16)


@pytest.fixture(scope="module")
def setup(sa):
    mx = make_mixture(d=128, C=16, r=16, s_n=0.7)
    X = draw_rows(mx, 50_000, row_seed=41)
    Q = draw_rows(mx, 16, row_seed=42)
    idx = sa.Index.build(bits_to_tensor(to_bf16_bits(X)).cuda(), 64, kmeans_iters=8)
    yield idx, Q.numpy().astype(np.float32)
    idx.free()


def wait(r, t, timeout=10.0):
    t0 = time.time()
    while not r.poll(t):
        assert time.time() - t0 < timeout
    return r.result(t)


def test_tasks_match_synchronous_calls(sa, setup):
    idx, Q = setup
    r = sa.Retriever(idx, streams=2, slots=4, max_nq=16, max_k=10)
    Qd = torch.from_numpy(Q).cuda()
    t_ivf = r.submit(Q[:8], 10, 8)
    t_ex = r.submit(Q[8:], 5, 0)
    r.set_engine_ready(True)
    t_m = r.submit(Q[:4], 10, 16, mature=True, tau=1.0, window=4, check_every=2)
    ids, sc, lists = wait(r, t_ivf)
    gi, gs = idx.search(Qd[:8].contiguous(), 10, 8)
    assert np.array_equal(ids, gi.cpu().numpy()) and np.array_equal(sc, gs.cpu().numpy())
    assert np.all(lists == 8)
    ids, sc, _ = wait(r, t_ex)
    gi, gs = idx.search(Qd[8:].contiguous(), 5, 0)
    assert np.array_equal(ids, gi.cpu().numpy()) and np.array_equal(sc, gs.cpu().numpy())
    ids, sc, lists = wait(r, t_m)
    gi, gs, gt = idx.search_mature(Qd[:4].contiguous(), 10, 16, tau=1.0, window=4, check_every=2)
    assert np.array_equal(ids, gi.cpu().numpy()) and np.array_equal(lists, gt.cpu().numpy())
    r.free()


def test_slots_are_bounded_and_tasks_known(sa, setup):
    idx, Q = setup
    r = sa.Retriever(idx, streams=1, slots=2, max_nq=4, max_k=5)
    a = r.submit(Q[:4], 5, 4)
    b = r.submit(Q[:4], 5, 4)
    with pytest.raises(sa.SAError) as e:
        r.submit(Q[:4], 5, 4)
    assert e.value.status == sa.SA_ERR_STATE
    with pytest.raises(sa.SAError):
        r.submit(Q[:5], 5, 4)                          # nq > max_nq
    wait(r, a)
    wait(r, b)
    with pytest.raises(sa.SAError) as e:
        r.poll(a)                                      # already collected
    assert e.value.status == sa.SA_ERR_STATE
    c = r.submit(Q[:4], 5, 4)                          # slot freed
    wait(r, c)
    r.free()


def test_engine_ready_stops_running_maturity_search(sa, setup):
    idx, Q = setup
    r = sa.Retriever(idx, streams=1, slots=2, max_nq=4, max_k=10)
    r.set_engine_ready(False)
    t = r.submit(Q[:4], 10, 64, mature=True, tau=0.0, window=4, check_every=1)
    _, _, lists = wait(r, t)
    assert np.all(lists == 64)                         # never ready: natural stop
    t = r.submit(Q[:4], 10, 64, mature=True, tau=0.0, window=4, check_every=1)
    time.sleep(0.0002)
    r.set_engine_ready(True)
    _, _, lists = wait(r, t)
    assert np.all((lists >= 1) & (lists < 64)), lists
    r.free()


def test_graph_tasks_match_synchronous_calls(sa, setup):
    """Alg. 1 over the proximity graph (the paper's own retriever): plain and maturity-exit
    graph tasks equal the synchronous calls bit for bit; the engine flag (never raised) keeps
    the maturity search running to its natural stop, which equals the plain search."""
    idx, Q = setup
    idx.build_graph(knn_k=24, degree=16, nprobe_build=4)
    r = sa.Retriever(idx, streams=2, slots=4, max_nq=16, max_k=10)
    Qd = torch.from_numpy(Q).cuda()
    r.set_engine_ready(True)
    t_g = r.submit_graph(Q[:8], 10, 64, search_width=2, n_entries=4)
    t_m = r.submit_graph(Q[8:], 10, 64, search_width=2, n_entries=4, mature=True, tau=0.9,
                         window=4, check_every=1)
    ids, sc, it = wait(r, t_g)
    gi, gs = idx.search_graph(Qd[:8].contiguous(), 10, 64, search_width=2, n_entries=4)
    assert np.array_equal(ids, gi.cpu().numpy()) and np.array_equal(sc, gs.cpu().numpy())
    assert np.all(it == -1)
    ids, sc, it = wait(r, t_m)
    mi, ms, mt = idx.search_graph_mature(Qd[8:].contiguous(), 10, 64, tau=0.9, window=4,
                                         check_every=1, search_width=2, n_entries=4)
    assert np.array_equal(ids, mi.cpu().numpy()) and np.array_equal(it, mt.cpu().numpy())
    r.set_engine_ready(False)
    t_n = r.submit_graph(Q[8:], 10, 64, search_width=2, n_entries=4, mature=True, tau=0.0,
                         window=4, check_every=1)
    ids, sc, it = wait(r, t_n)
    pi, ps = idx.search_graph(Qd[8:].contiguous(), 10, 64, search_width=2, n_entries=4)
    assert np.array_equal(ids, pi.cpu().numpy()) and np.array_equal(sc, ps.cpu().numpy())
    r.free()

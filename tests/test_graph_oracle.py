"""Pins for the graph-index oracle (oracle/graph.py) -- CPU only.  DESIGN.md R22-R27.

GR1  hand-evaluated detour counts / pruning / reverse merge on a 5-node kNN graph (below):
     node 2 keeps [1, 3] because its neighbour 0 is reachable 1 -> 0 at ranks (0, 0) < 1
     (detour 1), node 4 drops 0 (detours via 1 and 3); final lists mix forward and reverse
     edges as R26 orders them
GR2  hand-traced beam search on a 4-node path graph (iterations, expansions, T cut-off)
GR3  exhaustive search (L >= n) == brute force over the nodes reachable from the entry (oracle.c)
GR4  knn() == brute force top-K without self (oracle.c), ties by id on duplicated rows
"""
import numpy as np

import oracle
from oracle import graph


def bits(x):
    return oracle.bf16_round(np.asarray(x, dtype=np.float32))


KNN5 = np.array([[1, 2, 3], [0, 2, 4], [1, 0, 3], [2, 0, 4], [1, 3, 0]])


def test_gr1_prune_and_reverse_by_hand():
    fwd = graph.prune(KNN5, 2)
    assert fwd.tolist() == [[1, 2], [0, 2], [1, 3], [2, 0], [1, 3]]
    nbr = graph.reverse_merge(fwd)
    assert nbr.tolist() == [[1, 3], [0, 2], [1, 3], [2, 4], [1, 3]]
    # R >= K keeps every kNN entry, reordered by (detour, rank)
    assert graph.prune(KNN5, 3)[2].tolist() == [1, 3, 0]
    assert graph.prune(KNN5, 3)[4].tolist() == [1, 3, 0]


def path_graph():
    s = [0.125, 0.25, 0.375, 0.5]
    X = np.zeros((4, 8))
    for i, v in enumerate(s):
        X[i, 0] = v
        X[i, 1 + i] = 0.5
    q = np.zeros((1, 8))
    q[0, 0] = 1.0
    nbr = np.array([[1, -1], [0, 2], [1, 3], [2, -1]])
    return bits(X), nbr, bits(q)


def test_gr2_beam_search_by_hand():
    X, nbr, q = path_graph()
    r = graph.search(X, nbr, q[0], 2, L=2, w=1, entries=[0], T=100)
    assert r["ids"].tolist() == [3, 2] and r["scores"].tolist() == [0.5, 0.375]
    assert r["iterations"] == 4 and r["expanded"] == 4
    r = graph.search(X, nbr, q[0], 2, L=2, w=1, entries=[0], T=2)
    assert r["ids"].tolist() == [2, 1] and r["iterations"] == 2
    r = graph.search(X, nbr, q[0], 3, L=4, w=2, entries=[0, 0, -1], T=100)
    # w=2: it1 expands {0} only (one unexpanded), it2 {1}, it3 {2}, it4 {3}
    assert r["ids"].tolist() == [3, 2, 1] and r["iterations"] == 4


def mixture(n=300, d=32, seed=1):
    g = np.random.default_rng(seed)
    c = g.standard_normal((6, d))
    X = c[g.integers(0, 6, n)] + 0.5 * g.standard_normal((n, d))
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    return bits(X)


def test_gr3_exhaustive_search_is_exact():
    Xb = mixture()
    nbr, _ = graph.build(Xb, 16, 8)
    g = np.random.default_rng(2)
    Q = g.standard_normal((10, 32))
    Q /= np.linalg.norm(Q, axis=1, keepdims=True)
    Qb = bits(Q)
    ids, sc = oracle.flat_topk(Xb, Qb, 10)
    # nodes reachable from entry 0 (BFS); L >= n means the beam never drops one of them
    seen, todo = {0}, [0]
    while todo:
        u = todo.pop()
        for v in nbr[u]:
            if v >= 0 and int(v) not in seen:
                seen.add(int(v))
                todo.append(int(v))
    reach = np.array(sorted(seen))
    assert reach.size > 30
    ids, sc = oracle.flat_topk(Xb[reach], Qb, 10)
    for i in range(10):
        r = graph.search(Xb, nbr, Qb[i], 10, L=300, w=4, entries=[0], T=10_000)
        assert r["ids"].tolist() == reach[ids[i]].tolist()
        assert np.allclose(r["scores"], sc[i], rtol=0, atol=1e-12)
        assert r["expanded"] == reach.size


def test_gr4_knn_is_brute_force_without_self():
    Xb = mixture(120)
    Xb[7] = Xb[3]                       # duplicate: 3 and 7 are each other's best neighbour
    kn = graph.knn(Xb, 5)
    ids, _ = oracle.flat_topk(Xb, Xb, 6)
    for i in range(120):
        want = [int(x) for x in ids[i] if x != i][:5]
        assert kn[i].tolist() == want
    assert kn[3][0] == 7 and kn[7][0] == 3


def test_gr5_maturity_on_beam_search_by_hand():
    """Maturity exit on the beam search (R28-R29) on the path graph of GR2, by hand:
    L=2, w=1, entry 0; step 1 scores {1: 0.25} -> list (0.25, 0.125), s_t = s_best -> RQ 0;
    step 2 scores {2: 0.375} -> list (0.375, 0.25), RQ 0; step 3 scores {3: 0.5}, RQ 0;
    step 4 scores nothing -> RQ 1.  W=3 (alpha 0.5): EMA 0, 0, 0, 0.5."""
    X, nbr, q = path_graph()
    r = graph.search(X, nbr, q[0], 2, L=2, w=1, entries=[0], T=100, tau=float("inf"), window=3)
    assert r["rq"].tolist() == [0.0, 0.0, 0.0, 1.0]
    assert r["ema"].tolist() == [0.0, 0.0, 0.0, 0.5]
    assert r["iterations"] == 4
    # tau = 0 stops after the first step with the engine ready; never ready -> natural stop
    r = graph.search(X, nbr, q[0], 2, L=2, w=1, entries=[0], T=100, tau=0.0, window=3)
    assert r["iterations"] == 1 and r["ids"].tolist() == [1, 0]
    r = graph.search(X, nbr, q[0], 2, L=2, w=1, entries=[0], T=100, tau=0.0, window=3,
                     ready=False)
    assert r["iterations"] == 4 and r["ids"].tolist() == [3, 2]
    r = graph.search(X, nbr, q[0], 2, L=2, w=1, entries=[0], T=100, tau=0.0, window=3, g=3)
    assert r["iterations"] == 3 and r["ids"].tolist() == [3, 2]


def test_gr6_fp8_navigation_exact_on_e4m3_grid():
    """R34 on the GR2 path graph: every value is on the e4m3 grid after the power-of-two
    scaling (0.125..0.5 -> 64..256), so the fp8 scores are the bf16 scores times 2^17 and the
    fp8-navigated search equals the bf16 one, ids and (re-ranked) scores."""
    X, nbr, q = path_graph()
    a = graph.search(X, nbr, q[0], 2, L=2, w=1, entries=[0], T=100)
    b = graph.search_fp8(X, nbr, q[0], 2, L=2, w=1, entries=[0], T=100)
    assert b["ids"].tolist() == a["ids"].tolist() == [3, 2]
    assert b["scores"].tolist() == [0.5, 0.375] and b["iterations"] == a["iterations"]


def test_gr7_fp8_exhaustive_is_bf16_brute_force_over_reachable():
    """L >= n keeps every reachable node in the list whatever the (fp8) scores, so the bf16
    re-rank returns the exact bf16 top-k of the reachable set (oracle.c)."""
    Xb = mixture()
    nbr, _ = graph.build(Xb, 16, 8)
    g = np.random.default_rng(3)
    Q = g.standard_normal((6, 32))
    Q /= np.linalg.norm(Q, axis=1, keepdims=True)
    Qb = bits(Q)
    seen, todo = {0}, [0]
    while todo:
        u = todo.pop()
        for v in nbr[u]:
            if v >= 0 and int(v) not in seen:
                seen.add(int(v))
                todo.append(int(v))
    reach = np.array(sorted(seen))
    ids, sc = oracle.flat_topk(Xb[reach], Qb, 10)
    for i in range(6):
        r = graph.search_fp8(Xb, nbr, Qb[i], 10, L=300, w=4, entries=[0], T=10_000)
        assert r["ids"].tolist() == reach[ids[i]].tolist()
        assert np.allclose(r["scores"], sc[i], rtol=0, atol=1e-12)


def test_gr8_certified_paths():
    """The oracle's certification of its own search path (used by the GPU parity tests to tell
    legitimate fp32-vs-fp64 near-tie divergence from a defect): GR2's path separates every
    decision by >= 0.125 >> the fp32 error bound -> certified; two identical rows (different
    ids) competing for the result order tie exactly -> not certified."""
    X, nbr, q = path_graph()
    assert graph.search(X, nbr, q[0], 2, L=2, w=1, entries=[0], T=100)["certified"]
    Xd = bits([[0.25, 0.0], [0.5, 0.25], [0.5, 0.25]])
    nb = np.array([[1, 2], [0, -1], [0, -1]])
    r = graph.search(Xd, nb, bits([[1.0, 1.0]])[0], 2, L=2, w=1, entries=[0], T=100)
    assert r["ids"].tolist() == [1, 2] and not r["certified"] and r["near_tie"] == 0.0
    # a gap above the bound is certified even when tiny in absolute terms
    Xg = bits([[0.25, 0.0], [0.5, 0.25], [0.5, 0.2421875]])
    r = graph.search(Xg, nb, bits([[1.0, 1.0]])[0], 2, L=2, w=1, entries=[0], T=100)
    assert r["ids"].tolist() == [1, 2] and r["certified"]

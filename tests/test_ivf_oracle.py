"""Pins for the IVF oracle (oracle/ivf.py) -- CPU only.
and the readings R8-R11 of DESIGN.md."""
import numpy as np

import oracle
from oracle import ivf


def bits(x):
    return oracle.bf16_round(np.asarray(x, dtype=np.float32))


def blocks_corpus(n_per=1000, d=32, nblk=4, noise=0.01, seed=0):
    """Rows in contiguous blocks, block b near e_b (orthogonal cluster centres)."""
    g = np.random.default_rng(seed)
    X = noise * g.standard_normal((n_per * nblk, d))
    for b in range(nblk):
        X[b * n_per:(b + 1) * n_per, b] += 1.0
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    return bits(X)


def test_splitmix64_reference_vectors():
    # SplitMix64 reference output sequence from state 0 (Steele, Lea, Flood 2014)
    z, out = 0, []
    for _ in range(3):
        out.append(ivf.splitmix64(z))
        z = (z + 0x9E3779B97F4A7C15) & ivf.MASK64
    assert out == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_sample_rows_strided_by_global_id():
    r = ivf.sample_rows(4000, 4, 256)
    assert r.shape == (1024,) and r[0] == 0 and r[-1] == (1023 * 4000) // 1024
    assert np.all(np.diff(r) > 0)
    assert np.array_equal(ivf.sample_rows(100, 4, 256), np.arange(100))   # n_train = n_total


def test_p14_planted_blocks_recovered():
    X = blocks_corpus()
    C, Cb, assign, lists = ivf.build(X, 4, iters=5)
    for b in range(4):
        assert np.array_equal(lists[b], np.arange(b * 1000, (b + 1) * 1000))
        # centroid = normalised sum of its training-sample members (closed form of the update)
        rows = ivf.sample_rows(4000, 4)
        m = oracle.bf16_to_f64(X[rows[(rows >= b * 1000) & (rows < (b + 1) * 1000)]]).sum(0)
        assert np.allclose(C[b], m / np.linalg.norm(m), atol=1e-12)
    q = bits(np.eye(32)[2:3] + 0.05)
    ids, sc, P = ivf.search(X, lists, Cb, q, 5, 1)
    assert P[0, 0] == 2 and np.all((ids[0] >= 2000) & (ids[0] < 3000))


def test_p10_nprobe_all_equals_exact():
    g = np.random.default_rng(1)
    X = bits(g.standard_normal((3000, 48)))
    Q = bits(g.standard_normal((9, 48)))
    _, Cb, _, lists = ivf.build(X, 16, iters=4)
    ids, sc, _ = ivf.search(X, lists, Cb, Q, 10, 16)
    eids, esc = oracle.flat_topk(X, Q, 10)
    assert np.array_equal(ids, eids) and np.array_equal(sc, esc)


def test_p12_recall_monotone_in_nprobe():
    g = np.random.default_rng(2)
    X = bits(g.standard_normal((4000, 32)))
    Q = bits(g.standard_normal((20, 32)))
    _, Cb, _, lists = ivf.build(X, 32, iters=4)
    eids, _ = oracle.flat_topk(X, Q, 10)
    prev = np.zeros(20)
    for nprobe in (1, 2, 4, 8, 16, 32):
        ids, _, _ = ivf.search(X, lists, Cb, Q, 10, nprobe)
        rec = np.array([len(set(ids[i]) & set(eids[i])) / 10 for i in range(20)])
        assert np.all(rec >= prev)          # nested probe sets
        prev = rec
    assert np.all(prev == 1.0)


def test_r10_empty_list_repair():
    # Blocks 2 and 3 are copies of one row: the two centroids initialised there are equal,
    # tie on every row, the lower id wins them all (R8), list 3 is empty after the first
    # assignment and must take the sample row with the lowest assigned score (R10).
    g = np.random.default_rng(3)
    X = 0.01 * g.standard_normal((4000, 16))
    for b, axis in enumerate([0, 1, 2, 2]):
        X[b * 1000:(b + 1) * 1000, axis] += 1.0
    X[2000:4000] = X[2000]
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    Xb = bits(X)
    rows = ivf.sample_rows(4000, 4)
    S = oracle.bf16_to_f64(Xb[rows])
    # one iteration by hand from the same init
    stride = len(rows) // 4
    o = ivf.splitmix64(0x5A2505) % stride
    C0 = S[np.arange(4) * stride + o]
    sc = S @ oracle.bf16_to_f64(ivf.centroids_bf16(C0)).T
    a = np.argmax(sc, 1)
    best = sc[np.arange(len(rows)), a]
    C1, a1, _ = ivf.kmeans(Xb, 4, iters=1)
    assert np.array_equal(a1, a)
    empty = [j for j in range(4) if not np.any(a == j)]
    assert empty, "construction must produce an empty list"
    worst = np.lexsort((np.arange(len(rows)), best))
    for r, j in zip(worst, empty):
        assert np.array_equal(C1[j], S[r])

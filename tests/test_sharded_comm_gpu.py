"""The library's own sharded branch, end to end on one B200 (
VERDICT r1 "no test drives the library's own sharded branch").

`world` ranks live in threads of this process, each with its shard index (row_offset,
n_total) and an in-process communicator (sa_comm_init_local).  Every rank calls the public
sa_index_build_ex / sa_search / sa_search_host / sa_search_fp8 exactly as a one-process-per-GPU
NCCL job would: the sharded IVF build assembles the training sample from every rank's part,
the search all-gathers every rank's [nq, k] keys and merges them.  Results are compared with
the fp64 oracle (band rule), and with the unsharded index bit for bit (P8-iii).
"""
import threading

import numpy as np
import pytest
import torch

import oracle
from datagen import draw_rows, make_mixture, to_bf16_bits
from parity import check, check_against_rows

pytestmark = pytest.mark.gpu

N, D = 30_011, 128


def run_ranks(world, fn):
    """fn(rank) on `world` threads (each on its own stream); returns the per-rank results."""
    out, err = [None] * world, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                out[r] = fn(r)
                torch.cuda.current_stream().synchronize()
        except BaseException as e:  # noqa: BLE001 -- re-raised in the main thread
            err.append((r, e))

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    if err:
        raise err[0][1]
    assert not any(t.is_alive() for t in ts), "a rank hung"
    return out


@pytest.fixture(scope="module")
def data():
    mix = make_mixture(d=D, C=16, r=16)
    X = draw_rows(mix, N, row_seed=71).to(torch.bfloat16)
    Q = draw_rows(mix, 160, row_seed=72).to(torch.bfloat16)
    # P7 planted winners at every shard boundary (w = 2, 3): query j's winner is a scaled copy
    # of itself placed at row off_r - 1, off_r or off_r + 1; P5 duplicates across a boundary
    plant_rows = set()
    for w in (2, 3):
        for r in range(1, w):
            off = r * (N // w) + min(r, N % w)
            plant_rows.update({off - 1, off, off + 1})
    plant_rows = sorted(plant_rows)
    for j, row in enumerate(plant_rows):
        X[row] = (Q[j].float() * 2.0).to(torch.bfloat16)
    off2 = N // 2 + (N % 2 > 0)
    X[off2 + 5] = X[off2 - 7]            # duplicate pair straddling the w=2 boundary
    return X.cuda(), Q.cuda(), plant_rows


def shard(X, world, r):
    import paper_2505_12065_b200 as sa
    off, ln = sa.shard_range(X.shape[0], r, world)
    return X[off:off + ln].contiguous(), off


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_exact_search_vs_oracle(sa, data, world):
    X, Q, planted = data
    comms = sa.Comm.local_group(world)

    def rank(r):
        Xs, off = shard(X, world, r)
        idx = sa.Index.build(Xs, row_offset=off, n_total=X.shape[0], comm=comms[r])
        ids, sc = idx.search(Q, 10)
        keys = idx.search_keys(Q, 10)
        idx.free()
        return ids.cpu().numpy(), sc.cpu().numpy(), keys

    res = run_ranks(world, rank)
    for c in comms:
        c.free()
    for r in range(1, world):       # every rank receives the same global result
        assert np.array_equal(res[r][0], res[0][0]) and np.array_equal(res[r][1], res[0][1])
    ids, sc = res[0][0], res[0][1]
    rep = check_against_rows(ids, sc, to_bf16_bits(X.cpu()), to_bf16_bits(Q.cpu()), 10)
    assert rep["ok"], rep
    for j, row in enumerate(planted):            # P7: planted winners at shard boundaries
        assert ids[j, 0] == row, (j, row, ids[j, :3])
    # bit-identical to the unsharded index (P8-iii) and to the caller-driven composition
    full = sa.Index.build(X)
    fi, fs = full.search(Q, 10)
    full.free()
    assert np.array_equal(ids, fi.cpu().numpy()) and np.array_equal(sc, fs.cpu().numpy())
    mi, ms = sa.sa_merge_keys(torch.stack([res[r][2] for r in range(world)]))
    assert np.array_equal(mi.cpu().numpy(), ids) and np.array_equal(ms.cpu().numpy(), sc)


def test_sharded_duplicate_pair_across_boundary(sa, data):
    """P5 across shards: the duplicate rows straddling the w=2 boundary tie bit-exactly and the
    lower global id comes first."""
    X, Q, _ = data
    off2 = X.shape[0] // 2 + (X.shape[0] % 2 > 0)
    q = X[off2 - 7:off2 - 6].contiguous()
    comms = sa.Comm.local_group(2)

    def rank(r):
        Xs, off = shard(X, 2, r)
        idx = sa.Index.build(Xs, row_offset=off, n_total=X.shape[0], comm=comms[r])
        ids, sc = idx.search(q, 12)
        idx.free()
        return ids.cpu().numpy(), sc.cpu().numpy()

    (ids, sc), _ = run_ranks(2, rank)
    for c in comms:
        c.free()
    ids, sc = ids[0].tolist(), sc[0]
    # (a planted boundary row may outscore the self-match; the pair itself must be adjacent)
    j = ids.index(off2 - 7)
    assert ids[j + 1] == off2 + 5 and sc[j] == sc[j + 1]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_ivf_build_and_search_vs_oracle(sa, data, world):
    """Sharded IVF build (sample assembled through the communicator) -> centroids identical to
    the unsharded build; nprobe = nlist equals exact search (P10, band rule vs the oracle);
    nprobe < nlist equals the unsharded IVF result bit for bit and the oracle's exact search
    over the union of the probed lists (P11)."""
    X, Q, _ = data
    nlist = 32
    full = sa.Index.build(X, nlist, kmeans_iters=6)
    C_full = full.export_centroids()
    fi8, fs8 = full.search(Q, 10, 8)
    loff, lids = full.export_lists()
    P = full.probes(Q, 8).cpu().numpy()
    full.free()
    comms = sa.Comm.local_group(world)

    def rank(r):
        Xs, off = shard(X, world, r)
        idx = sa.Index.build(Xs, nlist, kmeans_iters=6, row_offset=off, n_total=X.shape[0],
                             comm=comms[r])
        C = idx.export_centroids()
        a = idx.search(Q, 10, nlist)
        b = idx.search(Q, 10, 8)
        idx.free()
        return C, [t.cpu().numpy() for t in a + b]

    res = run_ranks(world, rank)
    for c in comms:
        c.free()
    for r in range(world):
        assert np.array_equal(res[r][0], C_full), r        # w-invariant quantiser
    ai, asc, bi, bsc = res[0][1]
    Xb, Qb = to_bf16_bits(X.cpu()), to_bf16_bits(Q.cpu())
    rep = check_against_rows(ai, asc, Xb, Qb, 10)          # P10
    assert rep["ok"], rep
    assert np.array_equal(bi, fi8.cpu().numpy()) and np.array_equal(bsc, fs8.cpu().numpy())
    for qi in range(0, Q.shape[0], 4):                      # P11 on a sample of queries
        rows = np.sort(np.concatenate([lids[loff[l]:loff[l + 1]] for l in P[qi]]))
        oi, osc = oracle.flat_topk(Xb[rows], Qb[qi:qi + 1], 18)
        oi = np.where(oi >= 0, rows[np.maximum(oi, 0)], -1)
        r = check(bi[qi:qi + 1], bsc[qi:qi + 1], oi, osc,
                  lambda _q, ids_: oracle.pair_scores(Xb, Qb[qi:qi + 1],
                                                      np.zeros(len(ids_), int), ids_),
                  10, n_avail=min(10, len(rows)))
        assert r["ok"], (qi, r)


def test_sharded_fp8_and_host_path(sa, data):
    """sa_search_fp8 (global power-of-two scale through the communicator) and sa_search_host
    on a 2-rank sharded index equal the unsharded results bit for bit."""
    X, Q, _ = data
    full = sa.Index.build(X)
    full.build_fp8()
    f8 = [t.cpu().numpy() for t in full.search_fp8(Q, 10, 32)]
    fh = [t.numpy() for t in full.search_host(Q[:7].float().cpu().contiguous(), 5)]
    _, e_full = full.export_fp8()
    full.free()
    comms = sa.Comm.local_group(2)

    def rank(r):
        Xs, off = shard(X, 2, r)
        idx = sa.Index.build(Xs, row_offset=off, n_total=X.shape[0], comm=comms[r])
        idx.build_fp8()
        _, e = idx.export_fp8()
        a = [t.cpu().numpy() for t in idx.search_fp8(Q, 10, 32)]
        h = [t.numpy() for t in idx.search_host(Q[:7].float().cpu().contiguous(), 5)]
        idx.free()
        return e, a, h

    res = run_ranks(2, rank)
    for c in comms:
        c.free()
    for e, a, h in res:
        assert e == e_full
        assert all(np.array_equal(x, y) for x, y in zip(a, f8))
        assert all(np.array_equal(x, y) for x, y in zip(h, fh))


def test_cross_rank_argument_check(sa, data):
    """sa_comm_set_checks: mismatched (nq, k, nprobe) or a rank failing validation makes every
    rank return SA_ERR_INVALID_ARG with its outputs untouched -- nobody hangs."""
    X, Q, _ = data
    comms = [c.set_checks(True) for c in sa.Comm.local_group(2)]
    cases = [dict(nq=(4, 5), k=(10, 10)), dict(nq=(4, 4), k=(10, 0)),
             dict(nq=(4, 4), k=(10, 11)), dict(nq=(4, 4), k=(5, 5))]

    def rank(r):
        Xs, off = shard(X, 2, r)
        idx = sa.Index.build(Xs, row_offset=off, n_total=X.shape[0], comm=comms[r])
        out = []
        for c in cases:
            nq, k = c["nq"][r], c["k"][r]
            ids = torch.full((4, 16), 77, dtype=torch.int64, device="cuda")
            sc = torch.full((4, 16), 7.0, device="cuda")
            st = sa.lib().sa_search_ex(idx.handle, sa._ptr(Q), sa.SA_BF16, nq, k, 0, sa._ptr(ids),
                                       sa._ptr(sc), sa._stream_ptr(None))
            torch.cuda.synchronize()
            out.append((st, bool((ids == 77).all()), bool((sc == 7.0).all())))
        idx.free()
        return out

    res = run_ranks(2, rank)
    for c in comms:
        c.free()
    for r in range(2):
        for ci, (st, ids_untouched, sc_untouched) in enumerate(res[r][:3]):
            assert st == sa.SA_ERR_INVALID_ARG, (r, ci, st)
            assert ids_untouched and sc_untouched, (r, ci)
        assert res[r][3][0] == sa.SA_OK


def test_local_group_lifetime(sa):
    comms = sa.Comm.local_group(2)
    assert comms[1].info() == {"rank": 1, "world": 2, "nccl_nranks": 2}
    g = comms[0]._group.handle
    assert sa.lib().sa_comm_group_free(g) == sa.SA_ERR_STATE     # members alive
    for c in comms:
        c.free()
    assert comms[0]._group.handle is None

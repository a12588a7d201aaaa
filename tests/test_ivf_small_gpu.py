"""The one-launch IVF search of agent-step batches (nq <= 8; kernels/ivf_small.cu) against the
IVF oracle (R11, R36).

  * P10: nprobe = nlist is exact search (band rule vs oracle.c), for every batch size 1..8;
  * P11: the result is the exact top-k over the union of the probed lists -- the oracle's
    probe set (fp64 top-nprobe over the stored bf16 centroids, ties by lowest id), for every
    query whose probe boundary is wider than the fp32 error bound;
  * P8-i within the path: a query alone or inside a batch of 2..8 -> identical bits;
  * the batch path (nq > 8, tensor cores) and this path (CUDA cores) return the same ids
    except at near-ties of the k-th score;
  * fp32 input == its bf16 rounding; padding when the probed lists hold fewer than k rows;
  * a 2-rank sharded search (local communicator) equals the unsharded one bit for bit.
"""
import threading

import numpy as np
import pytest
import torch

import oracle
from datagen import draw_rows, make_mixture, to_bf16_bits
from parity import check, check_against_rows

pytestmark = pytest.mark.gpu


def bits(x):
    return oracle.bf16_round(np.asarray(x, dtype=np.float32))


def t16(b):
    return torch.from_numpy(np.ascontiguousarray(b).view(np.int16).copy()).view(torch.bfloat16)


@pytest.fixture(scope="module")
def setup(sa):
    mix = make_mixture(d=128, C=16, r=16, s_n=0.7)
    Xb = to_bf16_bits(draw_rows(mix, 50_000, row_seed=31))
    Qb = to_bf16_bits(draw_rows(mix, 40, row_seed=32))
    idx = sa.Index.build(t16(Xb).cuda(), 64, kmeans_iters=8)
    off, gid = idx.export_lists()
    lists = [gid[off[j]:off[j + 1]] for j in range(64)]
    Cb = bits(idx.export_centroids())
    yield idx, Xb, Qb, lists, Cb
    idx.free()


def small_search(idx, Qb, k, nprobe, batch):
    """Queries in batches of `batch` (<= 8: the one-launch path)."""
    ids, sc = [], []
    for i in range(0, len(Qb), batch):
        gi, gs = idx.search(t16(Qb[i:i + batch]).cuda(), k, nprobe)
        ids.append(gi.cpu().numpy())
        sc.append(gs.cpu().numpy())
    return np.concatenate(ids), np.concatenate(sc)


@pytest.mark.parametrize("batch", [1, 3, 8])
def test_p10_all_lists_is_exact(sa, setup, batch):
    idx, Xb, Qb, lists, Cb = setup
    gi, gs = small_search(idx, Qb, 10, 64, batch)
    rep = check_against_rows(gi, gs, Xb, Qb, 10)
    assert rep["ok"], rep


def p11_check(gi, gs, Xb, Qb, lists, Cb, nprobe, k):
    """P11 for every query whose probe boundary is wider than the fp32 error bound; returns the
    number of queries skipped at a probe near-tie."""
    nlist = len(lists)
    C = oracle.bf16_to_f64(Cb)
    Q = oracle.bf16_to_f64(Qb)
    pc = Q @ C.T
    eb = 2 * (Q.shape[1] - 1) * 2.0 ** -24 * (np.abs(Q) @ np.abs(C).T)
    skipped = 0
    for qi in range(len(Qb)):
        order = np.lexsort((np.arange(nlist), -pc[qi]))
        P = order[:nprobe]
        if nprobe < nlist:
            a, b = order[nprobe - 1], order[nprobe]
            if pc[qi, a] - pc[qi, b] <= eb[qi, a] + eb[qi, b]:
                skipped += 1       # probe boundary inside the fp32 error: either set is right
                continue
        rows = np.sort(np.concatenate([lists[j] for j in P]))
        oi, osc = oracle.flat_topk(Xb[rows], Qb[qi:qi + 1], k + 8)
        oi = np.where(oi >= 0, rows[np.maximum(oi, 0)], -1)
        r = check(gi[qi:qi + 1], gs[qi:qi + 1], oi, osc,
                  lambda _q, ids_: oracle.pair_scores(Xb, Qb[qi:qi + 1],
                                                      np.zeros(len(ids_), int), ids_),
                  k, n_avail=min(k, len(rows)))
        assert r["ok"], (nprobe, k, qi, r)
    return skipped


@pytest.mark.parametrize("nprobe,k", [(1, 10), (5, 1), (8, 32), (16, 5), (48, 10)])
def test_p11_exact_over_oracle_probe_set(sa, setup, nprobe, k):
    idx, Xb, Qb, lists, Cb = setup
    gi, gs = small_search(idx, Qb, k, nprobe, 8)
    skipped = p11_check(gi, gs, Xb, Qb, lists, Cb, nprobe, k)
    assert skipped <= 2, skipped
    print(f"P11 small path nprobe={nprobe} k={k}: {skipped} probe near-ties skipped")


@pytest.mark.parametrize("nprobe", [16, 48, 256])
def test_p11_many_centroids_per_cta_correlated_slices(sa, nprobe):
    """nlist = 6000 > 32 x grid: every CTA scores several 32-row centroid pieces.  The centroids
    are ordered by descending score against query 0, so each CTA's slice is a contiguous score
    band: the probe threshold T' taken from the per-CTA best keys lies far below the nprobe-th
    key and the candidate set is large -- counted ranks at nprobe = 16 (~600 candidates), the
    radix-select branch at 48 and 256 (> 1024 candidates).  P11 against the oracle's probe set."""
    mix = make_mixture(d=128, C=16, r=16, s_n=0.7)
    Xb = to_bf16_bits(draw_rows(mix, 60_000, row_seed=41))
    Qb = to_bf16_bits(draw_rows(mix, 4, row_seed=42))
    rng = np.random.default_rng(43)
    C = rng.standard_normal((6000, 128)).astype(np.float32)
    C /= np.linalg.norm(C, axis=1, keepdims=True)
    s0 = oracle.bf16_to_f64(bits(C)) @ oracle.bf16_to_f64(Qb[0])
    C = np.ascontiguousarray(C[np.lexsort((np.arange(6000), -s0))])
    idx = sa.Index.build(t16(Xb).cuda(), 6000, centroids=torch.from_numpy(C).cuda())
    off, gid = idx.export_lists()
    lists = [gid[off[j]:off[j + 1]] for j in range(6000)]
    Cb = bits(idx.export_centroids())
    gi, gs = small_search(idx, Qb, 10, nprobe, 4)
    skipped = p11_check(gi, gs, Xb, Qb, lists, Cb, nprobe, 10)
    assert skipped <= 1, skipped
    # a query alone == inside the batch
    si, ss = small_search(idx, Qb, 10, nprobe, 1)
    assert np.array_equal(si, gi) and np.array_equal(ss, gs)
    idx.free()


def test_batch_invariance_and_input_dtype(sa, setup):
    idx, Xb, Qb, lists, Cb = setup
    Q8 = t16(Qb[:8]).cuda()
    bi, bs = idx.search(Q8, 10, 16)
    for n in (1, 2, 5):
        for j in range(0, 8, n):
            if j + n > 8:
                break
            si, ss = idx.search(Q8[j:j + n].contiguous(), 10, 16)
            assert torch.equal(si, bi[j:j + n]) and torch.equal(ss, bs[j:j + n]), (n, j)
    # fp32 input is rounded to bf16 inside the kernel (R3): identical to the bf16 call
    fi, fs = idx.search(Q8.float(), 10, 16)
    assert torch.equal(fi, bi) and torch.equal(fs, bs)
    # host-buffer call (captured graph) == device call
    hi, hs = idx.search_host(Q8.float().cpu().contiguous(), 10, 16)
    assert torch.equal(hi, bi.cpu()) and torch.equal(hs, bs.cpu())


def test_matches_batch_path_except_near_ties(sa, setup):
    idx, Xb, Qb, lists, Cb = setup
    k, nprobe = 10, 16
    si, ss = small_search(idx, Qb, k, nprobe, 8)               # one-launch path
    bi, bs = idx.search(t16(Qb).cuda(), k, nprobe)           # 40 queries: batch path
    bi, bs = bi.cpu().numpy(), bs.cpu().numpy()
    for q in range(len(Qb)):
        assert np.allclose(ss[q], bs[q], rtol=1e-5, atol=1e-7), q
        diff = set(si[q].tolist()) ^ set(bi[q].tolist())
        if diff:   # only ids within fp32 rounding of the k-th score may differ
            s = oracle.pair_scores(Xb, Qb[q:q + 1], np.zeros(len(diff), int), np.array(sorted(diff)))
            assert np.all(np.abs(s - bs[q, k - 1]) <= 1e-5 * max(abs(bs[q, k - 1]), 1e-3)), q


def test_padding_when_lists_are_short(sa):
    mix = make_mixture(d=64, C=4, r=8, s_n=0.7)
    Xb = to_bf16_bits(draw_rows(mix, 40, row_seed=33))
    Qb = to_bf16_bits(draw_rows(mix, 3, row_seed=34))
    idx = sa.Index.build(t16(Xb).cuda(), 8, kmeans_iters=3)
    off, gid = idx.export_lists()
    P = idx.probes(t16(Qb).cuda(), 1).cpu().numpy()
    gi, gs = idx.search(t16(Qb).cuda(), 32, 1)
    gi, gs = gi.cpu().numpy(), gs.cpu().numpy()
    for q in range(3):
        n = int(off[P[q, 0] + 1] - off[P[q, 0]])
        assert n < 32
        assert np.all(gi[q, n:] == -1) and np.all(np.isneginf(gs[q, n:]))
        assert sorted(gi[q, :n].tolist()) == sorted(gid[off[P[q, 0]]:off[P[q, 0] + 1]].tolist())
    idx.free()


def test_sharded_small_batch_equals_unsharded(sa, setup):
    idx, Xb, Qb, lists, Cb = setup
    Q4 = t16(Qb[:4]).cuda()
    ui, us = idx.search(Q4, 10, 16)
    X = t16(Xb).cuda()
    C = torch.from_numpy(idx.export_centroids()).cuda()
    comms = sa.Comm.local_group(2)
    out = [None, None]

    def rank(r):
        torch.cuda.set_device(0)
        off, ln = sa.shard_range(X.shape[0], r, 2)
        s_idx = sa.Index.build(X[off:off + ln], 64, row_offset=off, n_total=X.shape[0],
                               comm=comms[r], centroids=C)
        out[r] = [t.cpu() for t in s_idx.search(Q4, 10, 16)]
        s_idx.free()

    ts = [threading.Thread(target=rank, args=(r,)) for r in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    for c in comms:
        c.free()
    for r in range(2):
        assert torch.equal(out[r][0], ui.cpu()) and torch.equal(out[r][1], us.cpu())

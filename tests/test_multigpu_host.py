"""Host-side logic of the row-sharded (N > 1) path, on CPU with world_size-2 gloo process
groups: the balanced shard split, shard-invariant synthetic rows, the NCCL
unique-id exchange, and the decomposition the sharded search relies on -- per-shard exact
top-k with global ids, all-gathered rank-major [w, nq, k], merged -- equals the global top-k."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from datagen import make_mixture, draw_rows, to_bf16_bits


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(fn, world, *args):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_entry, args=(fn, r, world, port, q, args)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    errs = [r for r in res if isinstance(r, str)]
    assert not errs, errs
    return sorted(res, key=lambda r: r[0])


def _entry(fn, rank, world, port, q, args):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        out = fn(rank, world, *args)
        dist.destroy_process_group()
        q.put((rank, out))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put(f"rank {rank}: {e}\n{traceback.format_exc()}")


def test_shard_range_balanced_and_complete():
    from paper_2505_12065_b200 import shard_range
    for n in (1, 7, 1000, 21_015_324):
        for w in (1, 2, 3, 4, 8):
            parts = [shard_range(n, r, w) for r in range(w)]
            assert parts[0][0] == 0
            for (o1, l1), (o2, _) in zip(parts, parts[1:]):
                assert o1 + l1 == o2
            assert parts[-1][0] + parts[-1][1] == n
            assert max(l for _, l in parts) - min(l for _, l in parts) <= 1
    # 21,015,324 rows over 8 ranks -> 2,626,915 or 2,626,916 rows each
    assert {shard_range(21_015_324, r, 8)[1] for r in range(8)} == {2_626_915, 2_626_916}


def test_generator_rows_are_shard_invariant():
    from paper_2505_12065_b200 import shard_range
    mix = make_mixture(d=32, C=4, r=4)
    full = draw_rows(mix, 150_000, row_seed=9)
    for w in (2, 3):
        parts = [draw_rows(mix, shard_range(150_000, r, w)[1], row_seed=9,
                           start=shard_range(150_000, r, w)[0]) for r in range(w)]
        assert torch.equal(torch.cat(parts), full)


def _uid(rank, world):
    import paper_2505_12065_b200 as sa
    return sa.Comm.exchange_unique_id()


def test_unique_id_exchange_gloo():
    res = _run(_uid, 2)
    assert res[0][1] == res[1][1] and len(res[0][1]) == 128 and any(res[0][1])


def _sharded_exact(rank, world, n, d, nq, k):
    from paper_2505_12065_b200 import shard_range
    mix = make_mixture(d=d, C=8, r=8)
    off, ln = shard_range(n, rank, world)
    X = to_bf16_bits(draw_rows(mix, ln, row_seed=31, start=off))
    Q = to_bf16_bits(draw_rows(mix, nq, row_seed=32))
    ids, sc = oracle.flat_topk(X, Q, k)
    ids = np.where(ids >= 0, ids + off, -1)
    # all-gather rank-major [w, nq, k] (what ncclAllGather does with the packed keys)
    t_ids = torch.from_numpy(ids)
    t_sc = torch.from_numpy(sc)
    g_ids = [torch.empty_like(t_ids) for _ in range(world)]
    g_sc = [torch.empty_like(t_sc) for _ in range(world)]
    dist.all_gather(g_ids, t_ids)
    dist.all_gather(g_sc, t_sc)
    G_ids = torch.stack(g_ids).numpy()
    G_sc = torch.stack(g_sc).numpy()
    out = np.full((nq, k), -1, dtype=np.int64)
    for qi in range(nq):
        cand = [(s, i) for r in range(world) for s, i in zip(G_sc[r, qi], G_ids[r, qi]) if i >= 0]
        cand.sort(key=lambda t: (-t[0], t[1]))
        for j, (_, i) in enumerate(cand[:k]):
            out[qi, j] = i
    return out


@pytest.mark.parametrize("world", [2])
def test_sharded_exact_decomposition_gloo(world):
    n, d, nq, k = 20_001, 32, 12, 10
    res = _run(_sharded_exact, world, n, d, nq, k)
    mix = make_mixture(d=d, C=8, r=8)
    X = to_bf16_bits(draw_rows(mix, n, row_seed=31))
    Q = to_bf16_bits(draw_rows(mix, nq, row_seed=32))
    want, _ = oracle.flat_topk(X, Q, k)
    for _, got in res:
        assert np.array_equal(got, want)

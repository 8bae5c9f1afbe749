"""CPU: the N>1 decomposition (batch shards for conv, column panels for GEMM)
with two gloo ranks.  Each rank computes its shard with the oracle; rank 0
gathers and must reproduce the single-process result bit for bit (the
partition has no reduction, so exactness is structural)."""
import os
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_shard_ranges_partition():
    sys.path.insert(0, ROOT)
    from paper_1904_05347_b200 import shard
    for total in (1, 7, 32, 256, 1000):
        for world in (1, 2, 3, 8):
            spans = shard.all_shards(total, world)
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    assert shard.all_shards(256, 8) == [(32 * r, 32 * r + 32) for r in range(8)]
    for n in (100, 1024, 8192):
        cols = [shard.panel_range(n, 4, r) for r in range(4)]
        assert cols[0][0] == 0 and cols[-1][1] == n
        assert all(lo % 256 == 0 for lo, _ in cols if lo < n)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch
    import torch.distributed as dist
    import pyoracle as O
    from paper_1904_05347_b200 import shard
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N = 6
        s_full = O.Conv(N, 9, 11, 8, 5, 3, 3, 1, True)
        x = O.fill_random(int(np.prod(s_full.in_shape)), 3).reshape(s_full.in_shape)
        f = O.fill_random(int(np.prod(s_full.filt_shape)), 4).reshape(s_full.filt_shape)
        lo, hi = shard.shard_range(N, world, rank)
        s_loc = O.Conv(hi - lo, 9, 11, 8, 5, 3, 3, 1, True)
        y_loc = O.conv2d_naive(s_loc, x[lo:hi], f)
        full = shard.gather_batch_shards(torch.from_numpy(y_loc), N)
        # GEMM column panels: C = A B with A replicated, B column blocks.
        m, n, k = 40, 700, 33
        a = O.fill_random(m * k, 5)
        b = O.fill_random(k * n, 6).reshape(n, k)  # column-major k x n: column j = b[j]
        c0, c1 = shard.panel_range(n, world, rank, align=64)
        panel = O.gemm_naive(m, c1 - c0, k, 1.0, 0.0, 0, 0, a, b[c0:c1].ravel(), None)
        panels = [None] * world
        dist.all_gather_object(panels, (c0, c1, panel))
        t = shard.max_over_ranks(float(rank + 1))
        if rank == 0:
            want = O.conv2d_naive(s_full, x, f)
            ok_conv = np.array_equal(full.numpy().view(np.uint32), want.view(np.uint32))
            gemm_want = O.gemm_naive(m, n, k, 1.0, 0.0, 0, 0, a, b.ravel(), None)
            got = np.concatenate([p[2] for p in sorted(panels, key=lambda p: p[0])])
            ok_gemm = np.array_equal(got.view(np.uint32), gemm_want.view(np.uint32))
            q.put((ok_conv, ok_gemm, t))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_decomposition():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
        assert p.exitcode == 0
    ok_conv, ok_gemm, t = q.get(timeout=10)
    assert ok_conv and ok_gemm
    assert t == 2.0  # MAX over ranks


def _worker_helpers(rank, world, port, q):
    """The helpers bench.py's multi-GPU leg uses, on gloo: per-rank seeded
    slices of one logical tensor, broadcast of the shared operand, gather to
    rank 0, per-rank scalars."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_1904_05347_b200 import shard
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        per = 3
        lo, hi = rank * per, (rank + 1) * per
        mine = shard.seeded_images((4, 5, 2), lo, hi, 1234, 7, "cpu")
        cols = shard.seeded_columns(6, *shard.panel_range(8, world, rank, 4), 4242, 4, "cpu")
        f = torch.full((3,), float(rank))
        shard.broadcast_(f)  # rank 0's filter everywhere
        parts = shard.gather_to(mine, 0)
        cparts = shard.gather_to(cols, 0)
        ts = shard.all_gather_scalar(10.0 + rank)
        if rank == 0:
            whole = shard.seeded_images((4, 5, 2), 0, per * world, 1234, 7, "cpu")
            wcols = shard.seeded_columns(6, 0, 8, 4242, 4, "cpu")
            q.put((bool(torch.equal(torch.cat(parts), whole)),
                   bool(torch.equal(torch.cat(cparts), wcols)),
                   float(f.sum()), ts))
        else:
            q.put(None)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_bench_helpers():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30600 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker_helpers, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
        assert p.exitcode == 0
    res = [q.get(timeout=10) for _ in range(2)]
    res = [r for r in res if r is not None][0]
    ok_imgs, ok_cols, fsum, ts = res
    assert ok_imgs and ok_cols
    assert fsum == 0.0  # broadcast from rank 0
    assert ts == [10.0, 11.0]

"""The multi-GPU path's host logic on CPU: two gloo ranks (world size 2) shard the config-5 dead-time
sweep with no overlap and full coverage, and agree on the max of their timings."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2509_20500_b200.shard import max_over_ranks, shard, shard_indices


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tds = list(np.linspace(10.0, 500.0, 16 * world))
    mine = shard(tds, rank, world)
    got = [None] * world
    dist.all_gather_object(got, mine)
    t = max_over_ranks([1.0 + rank, 10.0 - rank])
    q.put((rank, got, t))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_indices_cover():
    for n in (0, 1, 7, 16, 64):
        for w in (1, 2, 3, 8):
            parts = [shard_indices(n, r, w) for r in range(w)]
            flat = sorted(i for p in parts for i in p)
            assert flat == list(range(n))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1
    with pytest.raises(ValueError):
        shard_indices(4, 2, 2)


def test_gloo_two_ranks():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    tds = list(np.linspace(10.0, 500.0, 32))
    for rank, got, t in res:
        assert sorted(x for part in got for x in part) == sorted(tds)      # full coverage, no overlap
        assert len(got[0]) == len(got[1]) == 16
        assert t == [2.0, 10.0]                                             # max over ranks


# ------------------------------------------------- one matrix split by rows
from paper_2509_20500_b200.shard import row_block  # noqa: E402


def test_row_block_partition():
    for n in (2, 7, 64, 1000, 32768):
        for w in (1, 2, 3, 8):
            if n < w:
                with pytest.raises(ValueError):
                    row_block(n, 0, w)
                continue
            blocks = [row_block(n, r, w) for r in range(w)]
            assert blocks[0][0] == 0 and sum(b[1] for b in blocks) == n
            for (a0, an), (b0, _) in zip(blocks, blocks[1:]):
                assert a0 + an == b0                                    # contiguous, rank order
            sizes = [b[1] for b in blocks]
            assert min(sizes) >= 1 and max(sizes) - min(sizes) <= 1


def _pi_blockwise(P, l, blocks, iters):
    """Reference: power iteration whose product is summed block by block in rank order -- the order
    the all-reduce of the row-sharded path adds the ranks' partial products (Thm 2)."""
    N = P.shape[0]
    pi = np.full(N, 1.0 / N)
    for _ in range(iters):
        x = pi[(np.arange(N) - l) % N]                 # x_r = pi[(r - l) mod N]: the gathered iterate
        y = None
        for r0, n in blocks:
            part = x[r0:r0 + n] @ P[r0:r0 + n]
            y = part if y is None else y + part
        pi = y / y.sum()
    return pi


def _shard_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(42)
    N, l, iters = 97, 31, 25
    P = rng.uniform(0.1, 1.0, (N, N))
    P /= P.sum(axis=1, keepdims=True)
    r0, n = row_block(N, rank, world)
    mine = P[r0:r0 + n]                                 # this rank stores only its rows
    pi = np.full(N, 1.0 / N)
    for _ in range(iters):
        x = pi[(np.arange(N) - l) % N]                 # replicated iterate, gather offset local
        y = torch.from_numpy(x[r0:r0 + n] @ mine)      # partial product of this rank's rows
        dist.all_reduce(y, op=dist.ReduceOp.SUM)       # one all-reduce of N doubles per iteration
        y = y.numpy()
        pi = y / y.sum()
    q.put((rank, pi))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_row_sharded_power_iteration():
    """Two gloo ranks each own half the rows of a row-stochastic P~0 and run the sharded iteration;
    both end with the same pi, bit for bit equal to the single-process blockwise product, and equal
    (to rounding) to the plain dense power iteration."""
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(42)
    N, l, iters = 97, 31, 25
    P = rng.uniform(0.1, 1.0, (N, N))
    P /= P.sum(axis=1, keepdims=True)
    ref = _pi_blockwise(P, l, [row_block(N, r, world) for r in range(world)], iters)
    assert np.array_equal(res[0][1], res[1][1])          # replicated iterate
    assert np.array_equal(res[0][1], ref)                # bit for bit
    dense = np.full(N, 1.0 / N)
    Pl = np.roll(P, -l, axis=0)                          # P~ = J_l P~0: row i is row (i + l) mod N
    for _ in range(iters):
        dense = dense @ Pl
        dense /= dense.sum()
    assert np.max(np.abs(ref - dense)) <= 1e-15

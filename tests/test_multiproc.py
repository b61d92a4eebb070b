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

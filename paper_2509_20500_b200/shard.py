"""Host-side sharding for one process per GPU.

(i) Items — (S, B, t_d) triples and the dead times that share one P~0 — are independent, so ranks
split them with no collective on the data path (`shard`); the only cross-rank operation is the max
of the timed region, taken once after timing (NCCL on GPUs, gloo in the CPU tests).
(ii) One matrix too large or too slow for one GPU: rank g stores the rows `row_block(N, g, world)`
of P~0 and the power iteration all-reduces the N x V partial products once per iteration
(`sharded_solve`, the driver loop over the library's shard steps)."""
from __future__ import annotations


def shard_indices(n_items: int, rank: int, world: int) -> list:
    """Strided shard: rank r gets items r, r + world, ... (dead-time sweeps sorted by t_d then give
    every rank a spread of iteration counts). Every item belongs to exactly one rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    return list(range(rank, n_items, world))


def shard(items, rank: int, world: int) -> list:
    return [items[i] for i in shard_indices(len(items), rank, world)]


def max_over_ranks(values, device=None):
    """Element-wise max of a list of floats over all ranks (identity when not distributed)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [float(v) for v in values]
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def row_block(n_rows: int, rank: int, world: int) -> tuple:
    """Contiguous balanced row block (row0, n) of rank `rank`: blocks tile [0, n_rows) in rank order,
    sizes differ by at most one, every rank gets >= 1 row (n_rows >= world)."""
    if world < 1 or not 0 <= rank < world or n_rows < world:
        raise ValueError("bad rank / world / rows")
    q, r = divmod(n_rows, world)
    row0 = rank * q + min(rank, r)
    return row0, q + (1 if rank < r else 0)


def sharded_solve(plan, all_reduce) -> list:
    """Power iteration over row shards: per iteration this rank's partial GEMV,
    one all-reduce (SUM) of the N x V partial products (`all_reduce(tensor)`, in place; e.g.
    torch.distributed.all_reduce over NCCL), then the replicated normalisation / convergence / gather
    step. `plan` is a splidar.ShardPlan. Returns the per-vector infos."""
    plan.init()
    while True:
        plan.gemv()
        all_reduce(plan.ypart)
        if not plan.check():
            break
    return plan.finish()

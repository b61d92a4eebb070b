"""Host-side sharding for one process per GPU: the path's items — (S, B, t_d)
triples and the dead times that share one P~0 — are independent, so ranks split them with no
collective on the data path. The only cross-rank operation is the max of the timed region, taken
once after timing (NCCL on GPUs, gloo in the CPU tests)."""
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

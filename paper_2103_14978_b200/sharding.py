"""Host-side sharding of pair batches over ranks (one process per GPU).

Pairs are independent ("the batch size is equal for all devices"),
so the data path has no collective: each rank filters its own contiguous range
of the seeded pair stream.  The only collectives are off the hot path: the max
over ranks of the device time (the paper reports the slowest device, :186) and
the sum of the accepted-pair totals.
"""
from __future__ import annotations


def weak_shard(n_per_rank: int, rank: int) -> tuple[int, int]:
    """(first pair index, count) of `rank` when every rank gets n_per_rank pairs."""
    return rank * n_per_rank, n_per_rank


def even_shard(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """(first pair index, count) of `rank` when n_total pairs are split evenly."""
    lo = n_total * rank // world
    hi = n_total * (rank + 1) // world
    return lo, hi - lo


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (e.g. device milliseconds) over the process group."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(values, device=None) -> list[int]:
    """Element-wise sum of per-rank integer counters (e.g. accepted pairs per e)."""
    import torch
    import torch.distributed as dist

    t = torch.as_tensor(values, dtype=torch.int64, device=device).clone()
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t)
    return [int(x) for x in t.cpu().tolist()]

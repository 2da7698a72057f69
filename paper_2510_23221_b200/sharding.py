"""Chip sharding across the GPUs of one node.

Configs 1-4 partition by independent chips: chip c runs on rank
floor(c * G / n_chips) (contiguous blocks), one process per GPU, no data-path
collective. The only cross-rank communication is timing plumbing (a barrier and
a max-reduce of device-measured step times), done with torch.distributed.
"""
from __future__ import annotations


def chips_for_rank(n_chips: int, rank: int, world: int) -> range:
    """Contiguous block of chip ids owned by `rank`: chip c -> floor(c*G/n)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    lo = -(-rank * n_chips // world)            # ceil(rank*n/G)
    hi = -(-(rank + 1) * n_chips // world)
    return range(lo, hi)


def owner_of_chip(c: int, n_chips: int, world: int) -> int:
    return c * world // n_chips


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (device-timed seconds) over the process group."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())

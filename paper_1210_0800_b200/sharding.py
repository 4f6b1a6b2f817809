"""Batch sharding across GPUs: independent systems, so rank r
of `world` solves a contiguous range of system indices with NO collective on
the data path; the only cross-rank traffic is the timing reduction (max over
ranks) of the benchmark.

System s of the global batch draws its inputs from
split_mix64(seed).split(s) (random.hpp:38-40), so a sharded run solves
exactly the systems a single-GPU run would.
"""
from __future__ import annotations


def shard(batch: int, rank: int, world: int, scaling: str = "weak") -> tuple[int, int]:
    """(first system index, count) of `rank`.  weak: `batch` systems per rank
    (rank r gets [r*batch, (r+1)*batch)); strong: the global `batch` split
    into near-equal contiguous ranges (the first batch % world ranks get one
    more)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank must be in [0, world)")
    if batch < 0:
        raise ValueError("negative batch")
    if scaling == "weak":
        return rank * batch, batch
    if scaling != "strong":
        raise ValueError("scaling is 'weak' or 'strong'")
    base, extra = divmod(batch, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """All-reduce MAX of a per-rank time (the benchmark's max-over-ranks
    rule).  NCCL needs a CUDA tensor (device), gloo a CPU one."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, dist=None, device=None) -> float:
    """All-reduce SUM of a per-rank count (failed systems, bytes copied)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())

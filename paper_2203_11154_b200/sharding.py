"""Shift sharding across ranks (one process per GPU) -- the multi-GPU plumbing of the batched solve.

The shifted systems are independent, so ranks take contiguous chunks of ceil(S/P) shifts,
exactly as paradiag_solve splits shifts over its std::thread pool (proj/src/paradiag.cpp:217-236), and
the solve itself needs no collective.  Only timing/aggregate statistics are reduced (max of the step
time, sum of the work), over torch.distributed (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations


def shard(n_shifts: int, rank: int, world: int) -> tuple[int, int]:
    """[b0, b1) of the contiguous chunk owned by `rank` (paradiag.cpp:222-224 chunking)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    chunk = (n_shifts + world - 1) // world
    b0 = min(n_shifts, rank * chunk)
    return b0, min(n_shifts, b0 + chunk)


def reduce_scalar(x: float, op: str = "max", device=None) -> float:
    """All-reduce one float over the default process group (identity when not distributed)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())

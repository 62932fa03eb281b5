"""Multi-GPU plumbing for the PDF path.

Independent scenes are sharded across ranks with no data-path collective
(config 4); a run's timing is the max over ranks, results are gathered to
rank 0 only when the caller asks.  Works with any torch.distributed backend
(NCCL on the B200 box, gloo for the CPU tests).
"""
from __future__ import annotations

import numpy as np


def shard_range(n_items: int, rank: int, world: int) -> range:
    """Contiguous, balanced block of item indices owned by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(local: np.ndarray, dist=None) -> np.ndarray | None:
    """Concatenate each rank's rows on rank 0 (None elsewhere); rank order = shard order."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return local
    objs = [None] * dist.get_world_size()
    dist.all_gather_object(objs, local)
    return np.concatenate(objs, axis=0) if dist.get_rank() == 0 else None

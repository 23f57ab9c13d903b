"""Multi-process plumbing for replicated-operator runs.

Every right-hand-side column of Z x = b (Eq. 9) is an independent
problem, so N GPUs run N replicas of the operator, each solving its own block
of columns; nothing on the data path needs a collective. torch.distributed is
only used to (a) agree on the column partition, (b) take the max over ranks of
the device times, and (c) optionally gather the solution columns.
"""
from __future__ import annotations

import numpy as np


def column_slice(nrhs: int, world: int, rank: int, mode: str = "weak") -> slice:
    """Columns of the global RHS block owned by `rank`.

    weak   : every rank solves the full block (per-GPU work fixed as N grows);
    strong : the block is split into contiguous, balanced pieces."""
    if mode == "weak" or world == 1:
        return slice(0, nrhs)
    base, extra = divmod(nrhs, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return slice(lo, hi)


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (e.g. elapsed ms) over the default process group."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_columns(X: np.ndarray, nrhs: int, dist=None, mode: str = "strong") -> np.ndarray | None:
    """Gather the column blocks of a strong-mode run on rank 0 (None elsewhere)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return X
    import torch
    world, rank = dist.get_world_size(), dist.get_rank()
    parts = [None] * world
    dist.all_gather_object(parts, (rank, np.ascontiguousarray(X)))
    if rank != 0:
        return None
    out = np.zeros((X.shape[0], nrhs), dtype=X.dtype)
    for r, blk in parts:
        out[:, column_slice(nrhs, world, r, mode)] = blk
    return out

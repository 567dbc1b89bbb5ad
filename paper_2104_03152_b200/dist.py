"""Data-parallel plumbing over torch.distributed.

Ciphertexts are independent, so the path shards with no data-path collective:
rank r of W processes its own contiguous block of the image stream; the only
collectives are the barrier / max-over-ranks timing and the gather of the
decrypted results to rank 0 (NCCL on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np


def shard_indices(step: int, batch: int, world: int, rank: int) -> np.ndarray:
    """Image indices rank `rank` processes at `step`: a contiguous block of `batch` images of the
    global batch world * batch; consecutive steps walk the stream without overlap."""
    start = (step * world + rank) * batch
    return np.arange(start, start + batch, dtype=np.int64)


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_to_rank0(t):
    """Gather equal-shaped per-rank tensors to rank 0 (list on rank 0, None elsewhere)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [t]
    rank, world = dist.get_rank(), dist.get_world_size()
    out = [torch.empty_like(t) for _ in range(world)] if rank == 0 else None
    dist.gather(t, out, dst=0)
    return out

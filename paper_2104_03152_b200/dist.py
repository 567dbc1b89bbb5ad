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


def _coll_device(t):
    """NCCL moves device tensors; gloo (the CPU tests) moves host tensors."""
    import torch.distributed as dist
    return "cpu" if dist.get_backend() == "gloo" else t.device


def scatter_from_rank0(full, per_rank_shape, dtype, device):
    """Rank 0 holds `full` [world * B, ...] (None elsewhere); every rank receives its contiguous
    block [B, ...] (the client scatters the input ciphertexts)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return full.to(device)
    rank, world = dist.get_rank(), dist.get_world_size()
    cdev = "cpu" if dist.get_backend() == "gloo" else device
    out = torch.empty(per_rank_shape, dtype=dtype, device=cdev)
    parts = [p.contiguous().to(cdev) for p in full.chunk(world)] if rank == 0 else None
    dist.scatter(out, parts, src=0)
    return out.to(device)


def gather_blocks_to_rank0(t):
    """Gather equal-shaped per-rank blocks to rank 0 as one tensor [world * B, ...] (None on the
    other ranks); the collective runs on the backend's device."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return t
    cdev = _coll_device(t)
    parts = gather_to_rank0(t.to(cdev))
    return torch.cat(parts).to(t.device) if parts is not None else None


def client_server_round(ctx, net, imgs_all, stream_id: int, device):
    """The paper's client-server exchange over torch.distributed: rank 0 is the
    client — it encodes and encrypts the global batch imgs_all [world * B][28][28] — and scatters the
    input ciphertext words; every rank evaluates its block (net.forward, no collective inside) and
    the level-0 output words are gathered back to rank 0, which decrypts.  Returns (logits on rank 0
    or None, gathered output words on rank 0 or None, this rank's input block size).  Keys are not
    moved: every rank derives the same public keys from the shared context seed (C9)."""
    import torch
    import torch.distributed as dist
    from .ckks import he_im2col_encode_batch
    world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank() if world > 1 else 0
    top, N = net.top, ctx.N
    B = None
    full = None
    if rank == 0:
        slots = he_im2col_encode_batch(imgs_all, 7, 7, 3, ctx.slots)
        ct = ctx.he_encode_encrypt(slots, 2.0 ** net.plan["in_log2"], top, stream_id)
        full = torch.empty((ct.B, 2, top + 1, N), dtype=torch.int64, device=device)
        ctx.he_ct_export_words(ct, full)
        torch.cuda.synchronize(device)
        B = ct.B // world
        scale = ct.scale
    if world > 1:   # block size and the (exact, double) ciphertext scale from the client
        meta = torch.tensor([float(B or 0), scale if rank == 0 else 0.0], dtype=torch.float64,
                            device=_coll_device(torch.empty(0, device=device)))
        dist.broadcast(meta, 0)
        B, scale = int(meta[0].item()), float(meta[1].item())
    mine = scatter_from_rank0(full, (B, 2, top + 1, N), torch.int64, device)
    x = ctx.he_ct_import_words(mine, top, scale)
    y = net.forward(x)
    yw = torch.empty((B, 2, y.level + 1, N), dtype=torch.int64, device=device)
    ctx.he_ct_export_words(y, yw)
    torch.cuda.synchronize(device)
    allw = gather_blocks_to_rank0(yw)
    if rank != 0:
        return None, None, B
    out = ctx.he_ct_import_words(allw, y.level, y.scale)
    return ctx.he_decode(ctx.he_decrypt(out), net.n_out), allw, B

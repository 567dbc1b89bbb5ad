"""World-size-2 gloo tests of the N>1 host logic: the image shards of all ranks
are disjoint and cover the stream, max-over-ranks timing, and the gather of per-rank results
to rank 0 reproduces what one rank computes for the whole batch (here with a float stand-in for
the decrypted logits, since the CUDA path cannot run on the CPU box)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2104_03152_b200.dist import gather_to_rank0, max_over_ranks, shard_indices


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B = 5
        idx = [shard_indices(s, B, world, rank) for s in range(3)]
        mine = torch.from_numpy(np.concatenate(idx))
        allidx = gather_to_rank0(mine)
        t = max_over_ranks(10.0 + rank)
        # stand-in per-image result depending only on the image index (like a decrypted logit row)
        res = torch.from_numpy(np.sin(np.concatenate(idx)[:, None] * np.arange(1, 11)[None, :]))
        allres = gather_to_rank0(res)
        if rank == 0:
            q.put((torch.cat(allidx).numpy(), t, torch.cat(allres).numpy()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharding_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    idx, t, res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sorted(idx.tolist()) == list(range(3 * 5 * world))      # disjoint and complete
    assert t == 10.0 + world - 1                                     # max over ranks
    order = np.argsort(idx)
    ref = np.sin(np.arange(3 * 5 * world)[:, None] * np.arange(1, 11)[None, :])
    assert np.array_equal(res[order], ref)


def _worker_words(rank, world, port, q):
    """Client (rank 0) scatters ciphertext words, every rank returns its block, rank 0 gathers."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2104_03152_b200.dist import gather_blocks_to_rank0, scatter_from_rank0
        B, shape = 3, (2, 4, 16)
        rng = np.random.default_rng(7)
        full = torch.from_numpy(rng.integers(0, 2 ** 62, (world * B, *shape), dtype=np.int64))
        mine = scatter_from_rank0(full if rank == 0 else None, (B, *shape), torch.int64, "cpu")
        ok_block = bool(torch.equal(mine, full[rank * B:(rank + 1) * B]))
        back = gather_blocks_to_rank0(mine + rank * 0)
        oks = gather_to_rank0(torch.tensor([int(ok_block)]))
        if rank == 0:
            q.put((bool(torch.equal(back, full)), [int(o.item()) for o in oks]))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_client_scatter_gather_words_gloo():
    """SURVEY §8(e) data plane: rank r receives exactly the contiguous block r of the client's
    ciphertext words and the gathered blocks reassemble the client's array bit for bit."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker_words, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    same, oks = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert same and oks == [1, 1]

"""Multi-process data plane on the GPU: two ranks on one GPU
(gloo for the exchange, host tensors), rank 0 the client.  The client encrypts the global batch,
scatters the ciphertext words, each rank evaluates its block of the paper's CNN, the level-0 output
words are gathered to rank 0 — and they equal, bit for bit, what ONE process computes for the whole
batch.  (The ranks' kernels never wait on each other, so sharing one GPU is safe.)"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2104_03152_b200 import Context
        from paper_2104_03152_b200.cnn import CONV_G, FC1_G, EncryptedCNN, rotation_steps
        from paper_2104_03152_b200.dist import client_server_round
        from synthetic import CFG4, cnn_weights, mnist_like_images
        dev = torch.device("cuda", 0)
        ctx = Context(CFG4.logN, CFG4.bits, CFG4.n_special, CFG4.seed)
        ctx.he_keygen(rotation_steps(conv_g=CONV_G, fc_bsgs=True, fc1_g=FC1_G))
        net = EncryptedCNN(ctx, cnn_weights(CFG4.seed), conv_g=CONV_G, fc1_g=FC1_G)
        imgs = mnist_like_images(world * 3, 4) if rank == 0 else None
        logits, words, B = client_server_round(ctx, net, imgs, 500, dev)
        if rank == 0:
            # one process, the whole batch: same encryption streams (stream_id + b), same forward
            from paper_2104_03152_b200 import he_im2col_encode_batch
            slots = he_im2col_encode_batch(imgs, 7, 7, 3, ctx.slots)
            ct = ctx.he_encrypt(ctx.he_encode(slots, 2.0 ** net.plan["in_log2"], net.top), 500)
            ref = net.forward(ct)
            q.put((words.cpu().numpy(), ref.words().view(np.int64), logits, B))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_ranks_equal_one_rank_bitwise():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    words, ref, logits, B = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert B == 3 and words.shape == ref.shape
    assert np.array_equal(words, ref)
    assert logits.shape == (6, 10)

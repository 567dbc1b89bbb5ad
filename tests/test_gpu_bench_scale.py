"""Correctness at the bench's own scale (VERDICT r1 "What's weak" #1): the exact calls and launch
configuration bench.py times (BASELINE config 5: the config-4 network, batch 512 per GPU, one-level
conv + folded BSGS FC layers), checked by bench.bench_check:

* the first, middle and last images are bit-exact against the CPU oracle (their input plaintexts
  are the oracle's integer encodings injected into the device-encoded batch, C7);
* all 512 decrypted logits are within 5e-3 of the float64 network with equal argmax (north_star).
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

pytestmark = pytest.mark.gpu


def test_bench_batch_512_bitexact_items_and_tolerance():
    import torch
    import bench
    from paper_2104_03152_b200 import Context
    from paper_2104_03152_b200.cnn import CONV_G, FC1_G, EncryptedCNN, rotation_steps
    from synthetic import CFG4, cnn_weights, mnist_like_images
    dev = torch.device("cuda", 0)
    ctx = Context(CFG4.logN, CFG4.bits, CFG4.n_special, CFG4.seed)
    ctx.he_set_stream(torch.cuda.current_stream(dev))
    ctx.he_keygen(rotation_steps(conv_g=CONV_G, fc_bsgs=True, fc1_g=FC1_G))
    net = EncryptedCNN(ctx, cnn_weights(CFG4.seed), conv_g=CONV_G, fc1_g=FC1_G)
    imgs = mnist_like_images(512, 4, start=20_000)
    check, _ = bench.bench_check(ctx, net, imgs, 3_000_000, dev, items=[0, 1, 255, 511], cpu_leg=False)
    print(check)
    assert check["bitexact_ok"], check
    assert check["tolerance_ok"], check

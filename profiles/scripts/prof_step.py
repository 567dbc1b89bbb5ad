"""One bench step (BASELINE config 5: the config-4 CNN, batch B per GPU, the bench's schedule) for
ncu captures: python profiles/scripts/prof_step.py [B] [steps].  Runs warm-up steps first so the
captured launches are steady-state (filter with ncu -k / --launch-skip)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2104_03152_b200 import Context, he_im2col_encode_batch  # noqa: E402
from paper_2104_03152_b200.cnn import CONV_G, FC1_G, EncryptedCNN, rotation_steps  # noqa: E402
from synthetic import CFG4, cnn_weights, mnist_like_images  # noqa: E402


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    dev = torch.device("cuda", 0)
    ctx = Context(CFG4.logN, CFG4.bits, CFG4.n_special, CFG4.seed)
    ctx.he_set_stream(torch.cuda.current_stream(dev))
    ctx.he_keygen(rotation_steps(conv_g=CONV_G, fc_bsgs=True, fc1_g=FC1_G))
    net = EncryptedCNN(ctx, cnn_weights(CFG4.seed), conv_g=CONV_G, fc1_g=FC1_G)
    x = torch.from_numpy(he_im2col_encode_batch(mnist_like_images(B, 4), 7, 7, 3, ctx.slots)).to(dev)
    out = torch.empty((B, net.n_out), dtype=torch.float64, device=dev)
    for i in range(steps):
        ct = ctx.he_encrypt(ctx.he_encode(x, 2.0 ** net.plan["in_log2"], net.top), 1000 + i * B)
        ctx.he_decode(ctx.he_decrypt(net.forward(ct)), net.n_out, out=out)
    torch.cuda.synchronize()
    print("ok", float(out[0, 0]))


if __name__ == "__main__":
    main()

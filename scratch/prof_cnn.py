# one CNN forward (batch B) for ncu captures
import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2104_03152_b200 import Context
from paper_2104_03152_b200.cnn import EncryptedCNN, rotation_steps
from synthetic import CFG4, cnn_weights, mnist_like_images
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ctx = Context(CFG4.logN, CFG4.bits, CFG4.n_special, CFG4.seed)
ctx.he_keygen(rotation_steps())
net = EncryptedCNN(ctx, cnn_weights(CFG4.seed))
imgs = mnist_like_images(B, 4)
ct = net.encrypt(imgs, 0)
for _ in range(2):
    out = net.forward(ct)
ctx.he_sync(); print("ok")

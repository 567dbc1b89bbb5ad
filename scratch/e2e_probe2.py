import os, sys, time; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2104_03152_b200 import Context
from paper_2104_03152_b200.cnn import CONV_G, EncryptedCNN, rotation_steps, CHUNK
from synthetic import CFG4, cnn_weights, mnist_like_images
B = 256
ctx = Context(CFG4.logN, CFG4.bits, CFG4.n_special, CFG4.seed)
ctx.he_keygen(rotation_steps(conv_g=CONV_G, fc_bsgs=True))
net = EncryptedCNN(ctx, cnn_weights(3), conv_g=CONV_G)
ct = net.encrypt(mnist_like_images(B, 4), 0)
c = ctx
rows = []
for i in range(30):
    t = [time.perf_counter()]
    x = c.he_im2col_conv_bsgs_pt(ct, net.conv_d, net.conv_b, CHUNK, CONV_G); t.append(time.perf_counter())
    x = c.he_square(x); t.append(time.perf_counter())
    x = c.he_vec_mat_pt(x, net.fc1_d, net.fc1_b); t.append(time.perf_counter())
    x = c.he_square(x); t.append(time.perf_counter())
    x = c.he_vec_mat_pt(x, net.fc2_d, net.fc2_b); t.append(time.perf_counter())
    c.he_sync(); t.append(time.perf_counter())
    rows.append(np.diff(t))
r = np.array(rows) * 1e3
np.set_printoptions(precision=2, suppress=True, linewidth=150)
print(os.environ.get("CUDA_MODULE_LOADING"), "cols: conv square fc1 square fc2 sync [ms host]")
print("median", np.median(r, axis=0))
for i, row in enumerate(r):
    if row[:5].sum() > 3 * np.median(r[:, :5].sum(1)): print("slow", i, row)

import sys, time; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2104_03152_b200 import Context, he_im2col_encode_batch
from paper_2104_03152_b200.cnn import FOLD_N1, EncryptedCNN, rotation_steps
from synthetic import CFG4, cnn_weights, mnist_like_images
B = 256
ctx = Context(CFG4.logN, CFG4.bits, CFG4.n_special, CFG4.seed)
stream = torch.cuda.current_stream(); ctx.he_set_stream(stream)
ctx.he_keygen(rotation_steps(fold_n1=FOLD_N1))
net = EncryptedCNN(ctx, cnn_weights(3), fold_n1=FOLD_N1)
imgs = torch.from_numpy(mnist_like_images(B, 4)).pin_memory()
sb = torch.empty((B, ctx.slots), dtype=torch.float64).pin_memory()
rows = []
for i in range(40):
    t0 = time.perf_counter()
    he_im2col_encode_batch(imgs.numpy(), 7, 7, 3, ctx.slots, out=sb.numpy()); t1 = time.perf_counter()
    pt = ctx.he_encode(sb.numpy(), 2.0 ** 30, net.top); t2 = time.perf_counter()
    ct = ctx.he_encrypt(pt, i * B); t3 = time.perf_counter()
    out = net.forward(ct); t4 = time.perf_counter()
    dec = ctx.he_decrypt(out); t5 = time.perf_counter()
    z = ctx.he_decode(dec, 10); t6 = time.perf_counter()
    rows.append([t1-t0, t2-t1, t3-t2, t4-t3, t5-t4, t6-t5, t6-t0])
r = np.array(rows) * 1e3
np.set_printoptions(precision=2, suppress=True, linewidth=150)
print("cols: im2col encode encrypt forward(host) decrypt decode total [ms]")
print("median", np.median(r, axis=0)); print("max   ", r.max(axis=0))
for i, row in enumerate(r):
    if row[-1] > 2 * np.median(r[:, -1]): print("slow step", i, row)

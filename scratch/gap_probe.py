import sys, time; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2104_03152_b200 import Context, he_im2col_encode_batch
from paper_2104_03152_b200 import cnn
from synthetic import CFG4, cnn_weights, mnist_like_images
B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
ctx = Context(CFG4.logN, CFG4.bits, CFG4.n_special, CFG4.seed)
ctx.he_keygen(cnn.rotation_steps(conv_g=cnn.CONV_G, fc_bsgs=True, fc1_g=cnn.FC1_G))
net = cnn.EncryptedCNN(ctx, cnn_weights(3), conv_g=cnn.CONV_G, fc1_g=cnn.FC1_G)
x = torch.from_numpy(he_im2col_encode_batch(mnist_like_images(B, 4), 7, 7, 3, 4096)).cuda()
logits = torch.empty((B, 10), dtype=torch.float64, device="cuda")
def step(i):
    t = [time.perf_counter()]
    pt = ctx.he_encode(x, 2.0 ** 30, net.top); t.append(time.perf_counter())
    ct = ctx.he_encrypt(pt, i * B); t.append(time.perf_counter())
    out = net.forward(ct); t.append(time.perf_counter())
    ctx.he_decode(ctx.he_decrypt(out), 10, out=logits); t.append(time.perf_counter())
    return np.diff(t) * 1e3
for i in range(3): step(i)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
rows = []
e0.record()
for i in range(10): rows.append(step(10 + i))
e1.record(); torch.cuda.synchronize()
r = np.array(rows)
print("B", B, "device ms/step %.2f" % (e0.elapsed_time(e1) / 10), "host ms/step median [encode encrypt forward decode]", np.median(r, 0).round(2), "sum %.2f" % np.median(r.sum(1)))

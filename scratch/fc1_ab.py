import sys; sys.path.insert(0, '.')
import torch
from paper_2104_03152_b200 import Context
from paper_2104_03152_b200 import cnn
from synthetic import CFG4, cnn_weights, mnist_like_images
B = 256
ctx = Context(CFG4.logN, CFG4.bits, CFG4.n_special, CFG4.seed)
steps = set(cnn.rotation_steps(conv_g=8, fc_bsgs=True))
for g in (16, 32, 64):
    steps |= set(cnn.rotation_steps(conv_g=8, fc_bsgs=True, fc1_g=g))
ctx.he_keygen(sorted(steps))
ct = None
for g in (0, 16, 32, 64, 32):
    net = cnn.EncryptedCNN(ctx, cnn_weights(3), conv_g=8, fc1_g=g)
    if ct is None: ct = net.encrypt(mnist_like_images(B, 4), 0)
    for _ in range(3): net.forward(ct)
    ctx.he_sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): net.forward(ct)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    ctx.he_profile_enable(True)
    net.forward(ct); ctx.he_sync()
    prof = ctx.he_profile_read(); ctx.he_profile_enable(False)
    top = sorted(prof.items(), key=lambda kv: -kv[1][1])[:7]
    print(g, "ms/forward %.2f" % ms, "img/s %.0f" % (B / ms * 1e3), [(k, round(v[1], 2)) for k, v in top], flush=True)

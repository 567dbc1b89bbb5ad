import sys; sys.path.insert(0, '.')
import torch
from paper_2104_03152_b200 import Context
from paper_2104_03152_b200 import cnn
from synthetic import CFG4, cnn_weights, mnist_like_images
B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ctx = Context(CFG4.logN, CFG4.bits, CFG4.n_special, CFG4.seed)
ctx.he_keygen(cnn.rotation_steps(conv_g=cnn.CONV_G, fc_bsgs=True, fc1_g=cnn.FC1_G))
net = cnn.EncryptedCNN(ctx, cnn_weights(3), conv_g=cnn.CONV_G, fc1_g=cnn.FC1_G)
ct = net.encrypt(mnist_like_images(B, 4), 0)
for _ in range(3): net.forward(ct)
ctx.he_sync()
ctx.he_profile_enable(True)
net.forward(ct); ctx.he_sync()
prof = ctx.he_profile_read(); ctx.he_profile_enable(False)
print("%-22s %4s %8s %9s %9s" % ("tag", "n", "ms", "Gmodop/s", "GB/s"))
for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1]):
    n, ms, b, _, ops = (v + [0] * 5)[:5]
    print("%-22s %4d %8.3f %9.1f %9.1f" % (k, n, ms, ops / ms / 1e6 if ms else 0, b / ms / 1e6 if ms else 0))

import sys, time; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2104_03152_b200 import Context, he_im2col_encode_batch
from paper_2104_03152_b200 import cnn
from synthetic import CFG4, cnn_weights, mnist_like_images
B = 256
ctx = Context(CFG4.logN, CFG4.bits, CFG4.n_special, CFG4.seed)
ctx.he_keygen(cnn.rotation_steps(conv_g=cnn.CONV_G, fc_bsgs=True, fc1_g=cnn.FC1_G))
net = cnn.EncryptedCNN(ctx, cnn_weights(3), conv_g=cnn.CONV_G, fc1_g=cnn.FC1_G)
x = torch.from_numpy(he_im2col_encode_batch(mnist_like_images(B, 4), 7, 7, 3, 4096)).cuda()
c = ctx
def step(i):
    t = [time.perf_counter()]
    pt = c.he_encode(x, 2.0 ** 30, net.top); ct = c.he_encrypt(pt, i * B); t.append(time.perf_counter())
    y = c.he_im2col_conv_bsgs_pt(ct, net.conv_d, net.conv_b, 64, 8); t.append(time.perf_counter())
    y = c.he_square(y); t.append(time.perf_counter())
    y = c.he_vec_mat_pt(y, net.fc1_d, net.fc1_b); t.append(time.perf_counter())
    y = c.he_square(y); t.append(time.perf_counter())
    y = c.he_vec_mat_pt(y, net.fc2_d, net.fc2_b); t.append(time.perf_counter())
    return np.diff(t) * 1e3
for i in range(3): step(i)
torch.cuda.synchronize()
r = np.array([step(10 + i) for i in range(10)])
np.set_printoptions(precision=2, suppress=True)
print("host ms [enc+encrypt conv square fc1 square fc2] median", np.median(r, 0))

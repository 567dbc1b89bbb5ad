import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from oracle import circuits as C
from oracle.oracle import OracleContext
from synthetic import CFG4, cnn_weights, mnist_like_images
from test_layouts import float_net_numpy
w = cnn_weights(3)
ctx = OracleContext(CFG4.logN, CFG4.bits, CFG4.n_special, CFG4.seed)
ctx.keygen(sorted(set(C.cnn_rotation_steps(fold_n1=8)) | set(C.cnn_rotation_steps(fold_n1=4))))
import json
plan = json.loads(sys.argv[1])
for n1 in [int(a) for a in sys.argv[2:]]:
    errs = []
    for i, img in enumerate(mnist_like_images(6, 4, start=16)):
        out = C.cnn_forward(ctx, C.cnn_encrypt_input(ctx, img, 1000 + i), w, plan=plan, lazy=True, bsgs=True, fold_n1=n1)
        z = ctx.decode(ctx.decrypt(out), 10)
        errs.append(np.max(np.abs(z - float_net_numpy(img, w))))
    print(sys.argv[1], n1, ["%.2e" % e for e in errs], flush=True)

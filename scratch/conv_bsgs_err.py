import sys, json; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from oracle import circuits as C
from oracle.oracle import OracleContext
from synthetic import CFG4, cnn_weights, mnist_like_images
from test_layouts import float_net_numpy
w = cnn_weights(3)
g = int(sys.argv[1]); start = int(sys.argv[2]); n = int(sys.argv[3])
plan = dict(C.CNN_PLAN_BSGS); plan.update(json.loads(sys.argv[4]) if len(sys.argv) > 4 else {})
ctx = OracleContext(CFG4.logN, CFG4.bits, CFG4.n_special, CFG4.seed)
ctx.keygen(C.cnn_rotation_steps(conv_g=g))
errs = []
for i, img in enumerate(mnist_like_images(n, 4, start=start)):
    ct = C.cnn_encrypt_input(ctx, img, 1000 + i, plan)
    out = C.cnn_forward(ctx, ct, w, plan=plan, lazy=True, bsgs=True, conv_g=g)
    z = ctx.decode(ctx.decrypt(out), 10)
    ref = float_net_numpy(img, w)
    errs.append(np.max(np.abs(z - ref)))
    assert np.argmax(z) == np.argmax(ref)
print(g, start, plan, ["%.2e" % e for e in errs], flush=True)

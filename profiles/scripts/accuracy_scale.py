"""Oracle accuracy of the bench CNN schedule at different scale plans (R1/R2, north_star
"within 5e-3 absolute at scale 2^26").  Test infrastructure: runs only oracle/ (CPU) and the
float64 numpy network.  Usage: python profiles/scripts/accuracy_scale.py [n_images]"""
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import circuits as OC                       # noqa: E402
from oracle.oracle import OracleContext                 # noqa: E402
from synthetic import CFG4, cnn_weights, mnist_like_images   # noqa: E402
from test_layouts import float_net_numpy                # noqa: E402

PLANS = {
    "bench (in 2^30, conv -2, fc1 -4, fc2 -4)": dict(in_log2=30, conv_shift=-2, fc1_shift=-4, fc2_shift=-4,
                                                      in_level_drop=1),
    "scale 2^26 throughout (in 2^26, shifts 0)": dict(in_log2=26, conv_shift=0, fc1_shift=0, fc2_shift=0,
                                                      in_level_drop=1),
    "in 2^26, fc2 -4": dict(in_log2=26, conv_shift=0, fc1_shift=0, fc2_shift=-4, in_level_drop=1),
    "in 2^26, fc1 -2, fc2 -2": dict(in_log2=26, conv_shift=0, fc1_shift=-2, fc2_shift=-2, in_level_drop=1),
}


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    o = OracleContext(CFG4.logN, CFG4.bits, CFG4.n_special, CFG4.seed)
    o.keygen(OC.cnn_rotation_steps(conv_g=OC.CONV_G, fc_bsgs=True, fc1_g=OC.FC1_G))
    w = cnn_weights(CFG4.seed)
    imgs = mnist_like_images(n, 4)
    ref = [float_net_numpy(im, w) for im in imgs]
    out = {"images": n, "cpu_threads": os.cpu_count(), "plans": {}}
    for name, plan in PLANS.items():
        t0 = time.time()

        def one(i):
            ct = OC.cnn_encrypt_input(o, imgs[i], 5000 + i, plan)
            y = OC.cnn_forward(o, ct, w, plan, lazy=True, bsgs=True, conv_g=OC.CONV_G, fc1_g=OC.FC1_G)
            return o.decode(o.decrypt(y), 10)
        with ThreadPoolExecutor(os.cpu_count()) as ex:
            z = list(ex.map(one, range(n)))
        err = [float(np.max(np.abs(z[i] - ref[i]))) for i in range(n)]
        am = sum(int(np.argmax(z[i]) == np.argmax(ref[i])) for i in range(n))
        out["plans"][name] = {"plan": plan, "max_err": max(err), "median_err": float(np.median(err)),
                              "argmax_equal": f"{am}/{n}", "within_5e-3": sum(e < 5e-3 for e in err),
                              "max_abs_logit": float(max(np.max(np.abs(r)) for r in ref)), "s": time.time() - t0}
        print(name, json.dumps(out["plans"][name]), flush=True)
    json.dump(out, open(os.path.join(ROOT, "profiles", "r02_accuracy_scale.json"), "w"), indent=1)


if __name__ == "__main__":
    main()

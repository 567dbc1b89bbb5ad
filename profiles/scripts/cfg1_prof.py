"""Per-kernel device time of one BASELINE config-1 evaluation (batch 1: encode, encrypt, vec_mat,
decrypt, decode) from the in-library profiler (CUDA events around every launch).
python profiles/scripts/cfg1_prof.py [lazy]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2104_03152_b200 import Context  # noqa: E402
from synthetic import CFG1, vecmat_inputs  # noqa: E402


def main():
    lazy = len(sys.argv) > 1 and sys.argv[1] == "lazy"
    dev = torch.device("cuda", 0)
    c = Context(CFG1.logN, CFG1.bits, CFG1.n_special, CFG1.seed)
    c.he_set_stream(torch.cuda.current_stream(dev))
    c.he_keygen(list(range(1, 64)))
    x, W = vecmat_inputs(CFG1.seed)
    xs = np.tile(x, c.slots // 64)
    lvl = c.L - 1
    D, _ = c.he_vec_mat_encode(W, None, False, 0, lvl, 2.0 ** 40, lazy=lazy)
    z = torch.from_numpy(xs[None].copy()).to(dev)
    out = torch.empty((1, 10), dtype=torch.float64, device=dev)
    for it in range(3):
        c.he_profile_enable(it == 2)
        ct = c.he_encrypt(c.he_encode(z, 2.0 ** 40, lvl), 0)
        c.he_decode(c.he_decrypt(c.he_vec_mat_pt(ct, D)), 10, out=out)
        torch.cuda.synchronize()
    prof = c.he_profile_read()
    tot = sum(v[1] for v in prof.values())
    for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:24s} launches {v[0]:4d}  ms {v[1]:.4f}  blocks {v[3]:.0f}")
    print("total kernel ms", round(tot, 4))


if __name__ == "__main__":
    main()

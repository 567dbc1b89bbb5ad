"""BASELINE config 3 rotation batch for ncu captures: N=16384, 8 data + 2 special 50-bit primes, 256
ciphertexts at the top level, rotated by steps 2^r (the bench's keyswitch_cfg3 shape).
python profiles/scripts/cfg3_rot.py [B] [nsteps]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2104_03152_b200 import Context  # noqa: E402
from synthetic import CFG3, messages  # noqa: E402


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    ns = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    dev = torch.device("cuda", 0)
    c3 = Context(CFG3.logN, CFG3.bits, CFG3.n_special, CFG3.seed)
    c3.he_set_stream(torch.cuda.current_stream(dev))
    steps = [1 << r for r in range(ns)]
    c3.he_keygen(steps)
    z = torch.from_numpy(messages(B, c3.slots, seed=CFG3.seed)).to(dev)
    ct = c3.he_encrypt(c3.he_encode(z, 2.0 ** 50, c3.L - 1), 0)
    for s in steps:
        c3.he_rotate(ct, s)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()

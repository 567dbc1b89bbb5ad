"""One cfg2 transform shape for ncu captures: python profiles/scripts/ntt_one.py logN L B [fwd|inv|fused] [reps]
(BASELINE config 2: uniform residues of 60/50-bit primes; the launches after the first are steady state)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2104_03152_b200 import Context  # noqa: E402
from synthetic import CFG2_PRIME_BITS  # noqa: E402


def main():
    logN, L, B = (int(x) for x in sys.argv[1:4])
    what = sys.argv[4] if len(sys.argv) > 4 else "fwd"
    reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
    dev = torch.device("cuda", 0)
    N = 1 << logN
    c = Context(logN, CFG2_PRIME_BITS(L), 0, 1)
    q = torch.tensor([int(x) for x in c.primes], dtype=torch.float64, device=dev)
    a = (torch.rand((B, L, N), dtype=torch.float64, device=dev) * q[None, :, None]).to(torch.int64)
    b = (torch.rand((B, L, N), dtype=torch.float64, device=dev) * q[None, :, None]).to(torch.int64)
    o = torch.empty_like(a)
    for _ in range(reps):
        if what == "fwd":
            c.he_ntt_forward(a, B, L)
        elif what == "inv":
            c.he_ntt_inverse(a, B, L)
        else:
            c.he_ntt_mul_intt(a, b, o, B, L)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()

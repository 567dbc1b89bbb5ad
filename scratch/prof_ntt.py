# cfg2-shaped plain NTT for ncu: N=16384 L=8 B=64 forward + inverse
import sys; sys.path.insert(0, '.')
import torch
from paper_2104_03152_b200 import Context
from synthetic import CFG2_PRIME_BITS
N, L, B = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 14, 8, 64
c = Context(N.bit_length() - 1, CFG2_PRIME_BITS(L), 0, 1)
q = torch.tensor([int(x) for x in c.primes], dtype=torch.float64, device='cuda')
a = (torch.rand((B, L, N), dtype=torch.float64, device='cuda') * q[None, :, None]).to(torch.int64)
for _ in range(3):
    c.he_ntt_forward(a, B, L); c.he_ntt_inverse(a, B, L)
torch.cuda.synchronize(); print("ok")

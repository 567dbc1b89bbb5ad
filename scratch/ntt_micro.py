import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2104_03152_b200 import Context
from synthetic import CFG4
g = Context(CFG4.logN, CFG4.bits, CFG4.n_special, CFG4.seed)
B, L = 256, 7
d = torch.randint(0, 1 << 25, (B, L, 1 << CFG4.logN), dtype=torch.int64, device="cuda")
for f in (g.he_ntt_forward, g.he_ntt_inverse):
    for _ in range(3): f(d, B, L)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): f(d, B, L)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    bf = B * L * (1 << CFG4.logN) // 2 * CFG4.logN
    print(f.__name__, "%.3f ms  %.1f G butterflies/s" % (ms, bf / ms / 1e6))

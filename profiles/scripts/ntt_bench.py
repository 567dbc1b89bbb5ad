"""cfg2 NTT micro-benchmark (BASELINE config 2): forward / inverse / fused NTT->modmul->INTT GB/s on
16 N L B (read + write words) for a few (N, L, B), CUDA events after warm-up.  HE_CKKS_LIB selects an
experiment build of the library.  Usage: python profiles/scripts/ntt_bench.py [json_out]"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2104_03152_b200 import Context  # noqa: E402
from synthetic import CFG2_PRIME_BITS  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    res = {"lib": os.environ.get("HE_CKKS_LIB", "default")}
    for logN, L, B in [(13, 8, 256), (14, 8, 256), (15, 8, 128), (14, 16, 64)]:
        N = 1 << logN
        c = Context(logN, CFG2_PRIME_BITS(L), 0, 1)
        q = torch.tensor([int(x) for x in c.primes], dtype=torch.float64, device=dev)
        a = (torch.rand((B, L, N), dtype=torch.float64, device=dev) * q[None, :, None]).to(torch.int64)
        b = (torch.rand((B, L, N), dtype=torch.float64, device=dev) * q[None, :, None]).to(torch.int64)
        o = torch.empty_like(a)

        def t(fn, reps=10):
            fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / reps / 1e3
        nb = 16 * N * L * B
        r = {"fwd_GBps": nb / t(lambda: c.he_ntt_forward(a, B, L)) / 1e9,
             "inv_GBps": nb / t(lambda: c.he_ntt_inverse(a, B, L)) / 1e9,
             "fused_GBps": 24 * N * L * B / t(lambda: c.he_ntt_mul_intt(a, b, o, B, L)) / 1e9}
        res[f"N={N} L={L} B={B}"] = {k: round(v, 1) for k, v in r.items()}
        print(f"N={N} L={L} B={B}", res[f"N={N} L={L} B={B}"], flush=True)
        del a, b, o, c
    if len(sys.argv) > 1:
        json.dump(res, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()

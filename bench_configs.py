"""Config-1 and config-5b measurements for bench.py's `extra` (product path only: no oracle/).

cfg1: one CKKSVector (x ~ U[-1,1]^64 replicated) times W 64x10 by the diagonal method, N=8192,
      primes [60,40,40,60], batch 1 -> latency of encode + encrypt + vec_mat + decrypt + decode.
cfg5b: N=32768, 18 data + 2 special 50-bit primes, scale 2^40, a batch of 512 ciphertexts through
      16 x (mul_plain by a plaintext encoded at q_l + rescale) then rotate-and-add by 1, 2, 4, 8.
"""
from __future__ import annotations

import numpy as np


def cfg1_latency(stream, timer):
    from paper_2104_03152_b200 import Context
    from synthetic import CFG1, vecmat_inputs
    c = Context(CFG1.logN, CFG1.bits, CFG1.n_special, CFG1.seed)
    c.he_set_stream(stream)
    c.he_keygen(list(range(1, 64)))
    x, W = vecmat_inputs(CFG1.seed)
    xs = np.tile(x, c.slots // 64)
    lvl = c.L - 1
    res = {}
    for lazy in (False, True):
        D, _ = c.he_vec_mat_encode(W, None, False, 0, lvl, 2.0 ** 40, lazy=lazy)

        def run():
            ct = c.he_encrypt(c.he_encode(xs, 2.0 ** 40, lvl), 0)
            return c.he_decode(c.he_decrypt(c.he_vec_mat_pt(ct, D)), 10)
        s = timer(run, reps=5)
        y = run()[0]
        res["lazy_moddown" if lazy else "per_rotation_moddown"] = {
            "latency_ms": round(s * 1e3, 3), "max_abs_err_vs_xW": float(np.max(np.abs(y - x @ W)))}
    res["shape"] = "N=8192 [60,40,40,60] scale 2^40, x 64 replicated, W 64x10, batch 1 (encode..decode)"
    return res


def cfg5b_throughput(stream, timer, dev, B: int = 512):
    import torch
    from paper_2104_03152_b200 import Context
    from synthetic import CFG5B, deep_chain_plaintexts, messages
    c = Context(CFG5B.logN, CFG5B.bits, CFG5B.n_special, CFG5B.seed)
    c.he_set_stream(stream)
    steps = [1, 2, 4, 8]
    c.he_keygen(steps)
    lvl = c.L - 1
    P = deep_chain_plaintexts(16, c.slots, seed=CFG5B.seed)
    pts = [c.he_encode(P[t], float(c.q[lvl - t]), lvl - t) for t in range(16)]
    z = torch.from_numpy(messages(B, c.slots, seed=CFG5B.seed)).to(dev)
    ct0 = c.he_encrypt(c.he_encode(z, 2.0 ** 40, lvl), 0)

    def run():
        ct = ct0
        for t in range(16):
            ct = c.he_rescale(c.he_mul_plain(ct, pts[t]))
        for s in steps:
            ct = c.he_add(ct, c.he_rotate(ct, s))
        return ct
    s = timer(run, reps=2)
    return {"shape": "N=32768, 18+2 x 50-bit primes, scale 2^40, batch 512, 16 x (mul_plain+rescale) + 4 rotate-and-add",
            "ciphertexts_per_s": round(B / s, 1), "ms_per_batch": round(s * 1e3, 2),
            "rotations_per_s": round(B * 4 / s, 1)}

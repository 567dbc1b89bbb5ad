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
    # the same calls with device-resident input / output (pinned host copies inside the timed region),
    # eager, and recorded once as a CUDA graph (he_graph_*) and replayed: batch-1 latency is launch-bound
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    D, _ = c.he_vec_mat_encode(W, None, False, 0, lvl, 2.0 ** 40, lazy=False)
    z_pin = torch.from_numpy(xs[None].copy()).pin_memory()
    o_pin = torch.empty((1, 10), dtype=torch.float64).pin_memory()
    z_dev = torch.empty((1, c.slots), dtype=torch.float64, device=dev)
    out = torch.empty((1, 10), dtype=torch.float64, device=dev)

    def calls():
        ct = c.he_encrypt(c.he_encode(z_dev, 2.0 ** 40, lvl), 0)
        c.he_decode(c.he_decrypt(c.he_vec_mat_pt(ct, D)), 10, out=out)

    def io(body):
        def f():
            with torch.cuda.stream(stream):
                z_dev.copy_(z_pin, non_blocking=True)
            body()
            with torch.cuda.stream(stream):
                o_pin.copy_(out, non_blocking=True)
        return f
    s_eager = timer(io(calls), reps=20)
    n0 = c.he_launch_count()
    calls()
    n_eager = c.he_launch_count() - n0
    c.he_graph_begin()
    calls()
    g = c.he_graph_end()
    s_graph = timer(io(g.launch), reps=20)
    torch.cuda.synchronize()
    res["device_io_eager"] = {"latency_ms": round(s_eager * 1e3, 3), "kernels": n_eager}
    res["device_io_cuda_graph"] = {"latency_ms": round(s_graph * 1e3, 3), "kernels": g.kernels,
                                   "max_abs_err_vs_xW": float(np.max(np.abs(o_pin.numpy()[0] - x @ W)))}
    g.free()
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


# PAPER.md Tables 4-5 at shape 256 (c4.2xlarge, 8 vCPU; ms): context for the op latencies below
PAPER_T45_MS = {"negate": 0.07, "square": 4.29, "polyval_2x2_x": 10.55, "add": 0.08, "multiply": 4.45,
                "sub": 0.08, "dot": 20.15, "add_plain": 0.8, "multiply_plain": 1.75, "sub_plain": 0.8,
                "dot_plain": 17.37}


def table45_ops(stream, timer, batch: int = 1):
    """The paper's unary/binary op benchmarks at its parameters: N=8192, a 200-bit
    modulus ([60,40,40,60]: the same 200 bits), vector shape 256, one ciphertext; device-timed."""
    from paper_2104_03152_b200 import Context
    c = Context(13, (60, 40, 40, 60), 1, 11)
    c.he_set_stream(stream)
    c.he_keygen([1 << k for k in range(8)])
    rng = np.random.default_rng(11)
    n = 256
    x, y = np.zeros((batch, c.slots)), np.zeros((batch, c.slots))
    x[:, :n], y[:, :n] = rng.uniform(-1, 1, (batch, n)), rng.uniform(-1, 1, (batch, n))
    lvl = c.L - 1
    a, b = c.he_encrypt(c.he_encode(x, 2.0 ** 40, lvl), 0), c.he_encrypt(c.he_encode(y, 2.0 ** 40, lvl), batch)
    pa = c.he_encode(y, 2.0 ** 40, lvl)
    pm = c.he_encode(y, float(c.q[lvl]), lvl)
    ops = {
        "negate": lambda: c.he_negate(a),
        "square": lambda: c.he_square(a),
        "polyval_2x2_x": lambda: c.he_polyval(a, [0.0, 1.0, 2.0]),
        "add": lambda: c.he_add(a, b),
        "multiply": lambda: c.he_rescale(c.he_relinearize(c.he_mul(a, b))),
        "sub": lambda: c.he_sub(a, b),
        "dot": lambda: c.he_dot(a, b, n),
        "add_plain": lambda: c.he_add_plain(a, pa),
        "multiply_plain": lambda: c.he_rescale(c.he_mul_plain(a, pm)),
        "sub_plain": lambda: c.he_add_plain(a, c.he_encode(-y, 2.0 ** 40, lvl)),
        "dot_plain": lambda: c.he_dot_plain(a, y[0], n),
    }
    out = {"shape": f"N=8192, [60,40,40,60] (200-bit), vector 256, batch {batch}; paper = c4.2xlarge CPU ms"}
    for k, f in ops.items():
        s = timer(f, reps=20)
        out[k] = {"ms": round(s * 1e3, 4), "paper_ms": PAPER_T45_MS[k]}
    return out


# ------------------------------------------------ CPU oracle subsets ---
def cpu_oracle_subsets():
    """BASELINE.md / SURVEY §8(d) "Oracle timing": the CPU oracle (oracle/, test infrastructure,
    never tuned) on bounded subsets of configs 1, 2, 3 and 5b, timed on this host's cores (std::thread
    over independent items, as the oracle is written).  A baseline for context, not the target."""
    import os
    import time
    from concurrent.futures import ThreadPoolExecutor
    from oracle import circuits as OC
    from oracle.oracle import OracleContext
    from synthetic import CFG1, CFG2_PRIME_BITS, CFG3, CFG5B, deep_chain_plaintexts, messages, vecmat_inputs
    cores = os.cpu_count() or 1
    out = {"cores": cores, "note": "CPU oracle baseline, not the target"}
    try:
        out["cpu_model"] = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name"))
    except Exception:
        out["cpu_model"] = "unknown"

    def pmap(fn, n):
        with ThreadPoolExecutor(max_workers=min(n, cores)) as ex:
            return list(ex.map(fn, range(n)))

    # config 1: one encrypted vec_mat (encrypt + 63 rotations + decrypt), batch 1 (keys excluded)
    o = OracleContext(CFG1.logN, CFG1.bits, CFG1.n_special, CFG1.seed)
    o.keygen(list(range(1, 64)))
    x, W = vecmat_inputs(CFG1.seed)
    t0 = time.perf_counter()
    ct = o.encrypt(o.encode(OC.replicate(x, o.slots), 2.0 ** 40, o.L - 1), 0)
    o.decode(o.decrypt(OC.vec_mat(o, ct, W, None, False)), 10)
    dt = time.perf_counter() - t0
    out["cfg1_vec_mat"] = {"sample": "1 vec_mat (x 64 replicated, W 64x10), encrypt..decrypt, 1 thread",
                           "seconds": round(dt, 3), "vec_mats_per_s": round(1 / dt, 4)}
    del o
    # config 2: forward NTT of N=16384, L=8, B=64 (512 limb transforms), threads over limbs
    N, L, B = 1 << 14, 8, 64
    o = OracleContext(14, CFG2_PRIME_BITS(L), 0, 1)
    rng = np.random.default_rng(1)
    limbs = [rng.integers(0, int(o.q[l % L]), N, dtype=np.uint64) for l in range(B * L)]
    t0 = time.perf_counter()
    pmap(lambda i: o.ntt(i % L, limbs[i]), B * L)
    dt = time.perf_counter() - t0
    out["cfg2_ntt"] = {"sample": "forward NTT, N=16384, L=8, B=64", "seconds": round(dt, 3),
                       "GBps_16NLB": round(16 * N * L * B / dt / 1e9, 4), "threads": min(B * L, cores)}
    del o, limbs
    # config 3: 4 ciphertexts x 14 rotations + 1 mul/relin/rescale
    o = OracleContext(CFG3.logN, CFG3.bits, CFG3.n_special, CFG3.seed)
    steps = [1 << r for r in range(14)]
    o.keygen(steps)
    z = messages(4, o.slots, seed=CFG3.seed)
    cts = [o.encrypt(o.encode(z[b], 2.0 ** 50, o.L - 1), b) for b in range(4)]
    t0 = time.perf_counter()
    pmap(lambda i: o.rotate(cts[i // 14], steps[i % 14]), 4 * 14)
    dt = time.perf_counter() - t0
    t1 = time.perf_counter()
    o.rescale(o.relinearize(o.tensor(cts[0], cts[1])))
    dm = time.perf_counter() - t1
    out["cfg3_keyswitch"] = {"sample": "4 ciphertexts x 14 rotations (threads over rotations) + 1 mul+relin+rescale",
                             "rotation_seconds": round(dt, 3), "rotations_per_s": round(56 / dt, 3),
                             "mul_relin_rescale_seconds": round(dm, 3), "threads": min(56, cores)}
    del o, cts
    # config 5b: one ciphertext through the deep chain (16 x mul_plain + rescale, 4 rotate-and-add)
    o = OracleContext(CFG5B.logN, CFG5B.bits, CFG5B.n_special, CFG5B.seed)
    o.keygen([1, 2, 4, 8])
    P = deep_chain_plaintexts(16, o.slots, seed=CFG5B.seed)
    ct = o.encrypt(o.encode(messages(1, o.slots, seed=CFG5B.seed)[0], 2.0 ** 40, o.L - 1), 0)
    t0 = time.perf_counter()
    OC.deep_chain(o, ct, P)
    dt = time.perf_counter() - t0
    out["cfg5b_deep_chain"] = {"sample": "1 ciphertext, N=32768, 18+2 primes, 1 thread", "seconds": round(dt, 3),
                               "ciphertexts_per_s": round(1 / dt, 5)}
    return out


# PAPER.md Table 2: the encrypted MNIST evaluation per operation, ms for ONE image on
# c4.2xlarge (8 vCPU) / c4.4xlarge (16 vCPU)
PAPER_T2_MS = {"key_generation": (940.01, 921.04), "input_preparation": (9.8, 9.8), "conv": (236.9, 237.98),
               "square1": (8.47, 8.42), "fc1": (1084.65, 575.34), "square2": (4.29, 4.2), "fc2": (121.36, 70.36),
               "full_forward": (1456.29, 887.06)}


def table2_breakdown(ctx, net, imgs, stream, keygen_s, reps: int = 3):
    """The paper's Table-2 rows on the device, at the bench's schedule: per-stage CUDA-event time of
    the batch (imgs [B][28][28], the bench's batch) and of a single image, plus key generation (the
    bench's own context + keygen, host wall clock) and the host im2col per image."""
    import time
    import torch
    from paper_2104_03152_b200 import he_im2col_encode_batch
    from paper_2104_03152_b200.cnn import CHUNK
    dev = torch.device("cuda", torch.cuda.current_device())
    t0 = time.perf_counter()
    slots = he_im2col_encode_batch(imgs, 7, 7, 3, ctx.slots)
    prep_s = time.perf_counter() - t0
    res = {"key_generation_ms": round(keygen_s * 1e3, 2),
           "input_preparation_ms_per_image": round(prep_s * 1e3 / len(imgs), 4),
           "paper_ms_per_image_8vcpu_16vcpu": PAPER_T2_MS}
    stages = ["encode_encrypt", "conv", "square1", "fc1", "square2", "fc2", "decrypt_decode"]
    for label, x_host in (("batch", slots), ("single_image", slots[:1])):
        B = x_host.shape[0]
        x = torch.from_numpy(x_host).to(dev)
        out = torch.empty((B, net.n_out), dtype=torch.float64, device=dev)
        tot = [0.0] * len(stages)
        for r in range(reps + 1):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(stages) + 1)]
            c = ctx
            ev[0].record(stream)
            ct = c.he_encode_encrypt(x, 2.0 ** net.plan["in_log2"], net.top, 7_000_000 + r * B)
            ev[1].record(stream)
            y = c.he_im2col_conv_bsgs_pt(ct, net.conv_d, net.conv_b, CHUNK, net.conv_g)
            ev[2].record(stream)
            y = c.he_square(y)
            ev[3].record(stream)
            y = c.he_vec_mat_pt(y, net.fc1_d, net.fc1_b)
            ev[4].record(stream)
            y = c.he_square(y)
            ev[5].record(stream)
            y = c.he_vec_mat_pt(y, net.fc2_d, net.fc2_b)
            ev[6].record(stream)
            c.he_decode(c.he_decrypt(y), net.n_out, out=out)
            ev[7].record(stream)
            torch.cuda.synchronize(dev)
            if r:
                for k in range(len(stages)):
                    tot[k] += ev[k].elapsed_time(ev[k + 1]) / reps
        res[label] = {"images": B, "ms": {k: round(v, 4) for k, v in zip(stages, tot)},
                      "full_forward_ms": round(sum(tot[1:6]), 4),
                      "full_forward_us_per_image": round(1e3 * sum(tot[1:6]) / B, 3)}
    return res


def paper_schedule_throughput(stream, imgs, float_logits, steps: int = 2):
    """The config-4 network at the PAPER's evaluation schedule: 2-level im2col
    conv with the log2(N) rotate-and-add fold, square, FC1 / FC2 by the diagonal method with one
    ModDown per rotation (255 + 63 rotations), input encrypted at the top level; 259 Galois keys.
    The bench's default schedule (one-level conv, folded BSGS FC layers) computes the
    same network; this is the like-for-like number for the paper's own form.  Device-timed images/s
    over `steps` steps of the batch `imgs` after one warm-up step, and the max |logit - float64 net|."""
    import torch
    from paper_2104_03152_b200 import Context, he_im2col_encode_batch
    from paper_2104_03152_b200.cnn import EncryptedCNN, rotation_steps
    from synthetic import CFG4, cnn_weights
    dev = torch.device("cuda", torch.cuda.current_device())
    c = Context(CFG4.logN, CFG4.bits, CFG4.n_special, CFG4.seed)
    c.he_set_stream(stream)
    c.he_keygen(rotation_steps())
    w = cnn_weights(CFG4.seed)
    net = EncryptedCNN(c, w, lazy=False, bsgs=False)
    B = len(imgs)
    x = torch.from_numpy(he_im2col_encode_batch(imgs, 7, 7, 3, c.slots)).to(dev)
    out = torch.empty((B, net.n_out), dtype=torch.float64, device=dev)

    def step(i):
        ct = c.he_encrypt(c.he_encode(x, 2.0 ** net.plan["in_log2"], net.top), 8_000_000 + i * B)
        c.he_decode(c.he_decrypt(net.forward(ct)), net.n_out, out=out)
    step(0)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(steps):
        step(1 + i)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    s = e0.elapsed_time(e1) / 1e3 / steps
    ref = float_logits(imgs, w)
    err = float(np.max(np.abs(out.cpu().numpy() - ref)))
    n_keys = len(rotation_steps())
    del net, c
    return {"schedule": "paper (PAPER.md:57-64): 2-level conv + log2 fold, per-rotation diagonal vec_mat",
            "images_per_s": round(B / s, 1), "ms_per_batch": round(s * 1e3, 2), "batch": B,
            "galois_keys": n_keys, "max_logit_err": err, "argmax_equal": int(np.sum(
                np.argmax(out.cpu().numpy(), 1) == np.argmax(ref, 1)))}


"""Benchmark of the B200 CKKS hot path (BASELINE.json metric).

Headline workload (BASELINE config 5 = the config-4 network on a stream of
seeded synthetic 28x28 images, sharded across GPUs): one STEP is, for a batch
of B images per GPU, encode -> encrypt -> im2col conv -> square -> FC1 ->
square -> FC2 -> decrypt -> decode, all in this library's sm_100a kernels.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]

* value: encrypted CNN inferences/s of the whole job (all ranks), inputs (the
  im2col'd slot vectors, float64) resident in HBM, CUDA events on the
  library's stream, barrier + synchronize around K steps, max over ranks.
* e2e: the same metric through the public API from pinned host images:
  host im2col, H2D of the slot vectors inside he_encode, ..., D2H logits.
* roofline: the dominant kernel (largest share of the step): bound "alu" — its
  algorithmic modular ops / CUDA-event time against the modop rate at which the
  kernel's busiest integer pipe (ncu-measured mix, profiles/r02/pipe_mix.json)
  saturates; hbm_frac = algorithmic bytes / time against MEASURED_PEAKS.json.
* cpu_baseline (rank 0, N=1): the CPU oracle (oracle/, test infrastructure)
  timed on a bounded sample of the same workload.
* extra: key-switch rotations/s (config 3 shape) and NTT GB/s (config 2 shape).
* --impl reference: the oracle (this tier's reference arm) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "encrypted 28x28 CNN inferences/s/box"
UNIT = "images/s"

# Integer roofline.  The integer pipes' peak rates are MEASURED on this pool's B200
# (profiles/int_peak.cu -> profiles/r02/int_peak.json: IMAD / IADD3 / VIADDMNMX 64 lanes/clk/SM,
# IMAD.HI 32), and the dominant kernel's instruction mix is MEASURED by ncu (profiles/r02/pipe_mix.json,
# from the `ncu --set full` capture of that kernel in the bench step: its busiest integer pipe and that
# pipe's utilisation u at the captured duration d).  The kernel's integer peak is the modular-op rate
# at which that pipe would be 100% busy with the same mix: alg_ops / (d u); frac = live rate / peak.


def _load_json(rel):
    try:
        return json.load(open(os.path.join(ROOT, rel)))
    except Exception:
        return None


INT_PEAK = _load_json("profiles/r02/int_peak.json")
# dependent-free NTT butterfly chains (profiles/int_peak.cu ops 9-11): the integer roof of a transform
INT_PEAK2 = _load_json("profiles/r02/int_peak_v2.json") or {}
BFLY64_GPS = (INT_PEAK2.get("ops", {}).get("ct_butterfly_64bit_harvey", {}) or {}).get("G_lane_steps_per_s")
PIPE_MIX = _load_json("profiles/r02/pipe_mix.json") or {}


# dram__bytes_read.sum + dram__bytes_write.sum per launch from one `ncu --set full` capture of the
# bench command at its default batch (profiles/r01_ncu_summary.md)
TRAFFIC = {}
try:
    TRAFFIC = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
except Exception:
    pass


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region, in-process through NVML (no
    nvidia-smi subprocess: spawning one every 200 ms can stall the CUDA driver of this process)."""

    def __init__(self, index: int):
        self.index, self.samples, self.stop = index, [], threading.Event()

    def _run(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        except Exception:
            return
        bits = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}
        while not self.stop.is_set():
            try:
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                fn = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    N.nvmlDeviceGetCurrentClocksThrottleReasons
                r = fn(h)
                self.samples.append((sm, mx, [k for k, b in bits.items() if r & b]))
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(s[1] for s in self.samples)),
                "reasons": sorted({r for s in self.samples for r in s[2]}), "samples": len(self.samples),
                "source": "NVML (in-process), every 200 ms during the timed region"}


# ----------------------------------------------------------------- ours ---
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2104_03152_b200 import Context, he_im2col_encode_batch
    from paper_2104_03152_b200.cnn import CONV_G, FC1_G, EncryptedCNN, rotation_steps
    from paper_2104_03152_b200.dist import gather_to_rank0, max_over_ranks, shard_indices
    from synthetic import CFG4, cnn_weights, mnist_like_images

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.current_stream(dev)
    B = args.batch

    import time
    t_kg = time.perf_counter()
    ctx = Context(CFG4.logN, CFG4.bits, CFG4.n_special, CFG4.seed)
    ctx.he_set_stream(stream)
    ctx.he_keygen(rotation_steps(conv_g=CONV_G, fc_bsgs=True, fc1_g=FC1_G))
    torch.cuda.synchronize(dev)
    keygen_s = time.perf_counter() - t_kg   # Table 2 "Key generation": context + keys (first call, cold)
    net = EncryptedCNN(ctx, cnn_weights(CFG4.seed), conv_g=CONV_G, fc1_g=FC1_G)
    ns = ctx.slots

    # this rank's shard of the image stream (image i depends only on (seed, i))
    def shard(step):
        return mnist_like_images(B, 4, start=int(shard_indices(step, B, world, rank)[0]))

    n_batches = 2   # distinct input batches cycled through the steps
    imgs_host = [shard(s) for s in range(n_batches)]
    slots_host = [he_im2col_encode_batch(imgs, 7, 7, 3, ns) for imgs in imgs_host]
    slots_dev = [torch.from_numpy(s).to(dev) for s in slots_host]
    logits_dev = torch.empty((B, net.n_out), dtype=torch.float64, device=dev)

    def step_device(i):
        x = slots_dev[i % n_batches]
        # encode + encrypt in one call (he_encode_encrypt: the same words as he_encrypt(he_encode(x)))
        ct = ctx.he_encode_encrypt(x, 2.0 ** net.plan["in_log2"], net.top, 1_000_000 + i * B)
        out = net.forward(ct)
        ctx.he_decode(ctx.he_decrypt(out), net.n_out, out=logits_dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def timed(fn, K, W):
        for i in range(W):
            fn(i)
        barrier()
        l0 = ctx.he_launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(K):
            fn(W + i)
        e1.record(stream)
        barrier()
        ms = max_over_ranks(e0.elapsed_time(e1), dev)
        return ms, ctx.he_launch_count() - l0

    # --- device-resident timed region (headline value) ---
    with ClockSampler(local_rank) as clk:
        ms, launches = timed(step_device, args.steps, args.warmup)
    value = world * B * args.steps / (ms / 1e3)

    # --- kernel breakdown + roofline of the dominant kernel (profiled steps) ---
    ctx.he_profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(2):
        step_device(i)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    prof_step_ms = e0.elapsed_time(e1) / 2
    prof = ctx.he_profile_read()
    ctx.he_profile_enable(False)
    tot = sum(v[1] for v in prof.values())
    prof = {k: (v + [0.0] * 5)[:5] for k, v in prof.items()}
    top = max(prof, key=lambda k: prof[k][1])
    n_l, t_ms, alg_b, _, alg_ops = prof[top]
    peaks = load_peaks()
    sec = t_ms / n_l / 1e3
    gbs = (alg_b / n_l) / sec / 1e9 if t_ms > 0 else 0.0
    gops = (alg_ops / n_l) / sec / 1e9 if t_ms > 0 else 0.0
    mix = PIPE_MIX.get(top)
    if mix:   # measured instruction mix of this kernel (ncu) -> its integer peak
        peak_gops = mix["alg_ops_per_launch"] / (mix["ncu_duration_s"] * mix["busiest_pipe_util"]) / 1e9
        peak_src = (f"integer pipes measured (profiles/r02/int_peak.json); kernel mix measured by ncu "
                    f"(profiles/r02/pipe_mix.json: busiest pipe {mix['busiest_pipe']} at "
                    f"{100 * mix['busiest_pipe_util']:.1f}% over {1e6 * mix['ncu_duration_s']:.0f} us) -> "
                    f"the modop rate that saturates that pipe")
    else:     # no capture of this kernel yet: the measured shoup32 modmul rate (4 FMA-pipe slots)
        r = (INT_PEAK or {}).get("ops", {}).get("shoup32_modmul", {}).get("lane_steps_per_clk_per_sm", 15.8)
        peak_gops = r * 148 * 1.965
        peak_src = "measured shoup32 modmul rate (profiles/r02/int_peak.json) x 148 SMs x 1.965 GHz"
    roofline = {"bound": "alu", "kernel": top, "achieved": round(gops, 1), "peak": round(peak_gops, 1),
                "unit": "Gmodop/s", "frac": round(gops / peak_gops, 4), "traffic": TRAFFIC.get(top),
                "alg_ops_per_launch": alg_ops / n_l, "alg_bytes_per_launch": alg_b / n_l,
                "hbm_achieved_GBps": round(gbs, 1), "hbm_peak_GBps": peaks["hbm_gbs"],
                "hbm_frac": round(gbs / peaks["hbm_gbs"], 4),
                "share_of_step": round(t_ms / tot, 3), "us_per_launch": round(sec * 1e6, 2),
                "peak_source": peak_src + "; HBM: "
                               + ("MEASURED_PEAKS.json hbm_gbs" if not peaks.get("_fallback") else "fallback")}
    breakdown = {k: {"launches_per_step": v[0] / 2, "ms_per_step": round(v[1] / 2, 3),
                     "share": round(v[1] / tot, 3)} for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])}

    # --- e2e through the public API from pinned host images ---
    # Every step, through the C-ABI host-buffer calls: client im2col of the step's images into
    # page-locked memory, he_encode_encrypt from that HOST buffer (its H2D copy is issued inside the
    # call, on the context's copy stream, and the context stream waits for it), encrypt, forward, decrypt, he_decode_async into page-locked HOST logits (the
    # D2H copy is enqueued by the call).  Depth-2 pipeline: the host waits for step i-1's logits only
    # after enqueuing step i, and runs step i+1's im2col while the device computes step i, so the
    # device never drains between steps (each step's inputs and logits still cross PCIe inside the
    # timed region).  Buffer k = i % 2 is reused only after step i-2 was waited for.
    pinned = [torch.from_numpy(imgs).pin_memory() for imgs in imgs_host]
    slot_buf = [torch.empty((B, ns), dtype=torch.float64).pin_memory() for _ in range(2)]
    logits_pin = [torch.empty((B, net.n_out), dtype=torch.float64).pin_memory() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    logits_host = np.zeros((B, net.n_out))

    def im2col(i):
        he_im2col_encode_batch(pinned[i % n_batches].numpy(), 7, 7, 3, ns, out=slot_buf[i % 2].numpy())

    def e2e_loop(first, count):
        im2col(first)
        for i in range(first, first + count):
            k = i % 2
            ct = ctx.he_encode_encrypt(slot_buf[k].numpy(), 2.0 ** net.plan["in_log2"], net.top,
                                       2_000_000 + i * B)                                       # H2D inside
            dec = ctx.he_decrypt(net.forward(ct))
            ctx.he_decode_async(dec, logits_pin[k].numpy(), net.n_out)                         # D2H inside
            done[k].record(stream)
            if i > first:
                done[1 - k].synchronize()                       # step i-1 (and its buffers) finished
                logits_host[:] = logits_pin[1 - k].numpy()
            if i + 1 < first + count:
                im2col(i + 1)                                   # host work overlapping step i
        last = (first + count - 1) % 2
        done[last].synchronize()
        logits_host[:] = logits_pin[last].numpy()
        ctx.he_sync()

    e2e_loop(0, args.warmup)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    e2e_loop(args.warmup, args.steps)
    e1.record(stream)
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1), dev)
    # communication per inference: serialized encrypted input + encrypted logits of one image
    pt1 = ctx.he_encode(slots_dev[0][:1], 2.0 ** net.plan["in_log2"], net.top)
    one = ctx.he_encrypt(pt1, 7)
    up = len(ctx.he_ct_serialize(one))
    up_seeded = len(ctx.he_ct_serialize_seeded(ctx.he_encrypt_symmetric(pt1, 7, 0x5EED)))
    down = len(ctx.he_ct_serialize(net.forward(one)))
    comm = {"input_bytes": up, "output_bytes": down, "total_bytes": up + down,
            "input_bytes_seeded_symmetric": up_seeded, "total_bytes_seeded": up_seeded + down,
            "paper_total": "427 KB (PAPER.md:120)",
            "format": "bit-packed NTT words, w_i = bit_length(q_i); seeded form = c0 + (a_seed, stream) "
                      "(DESIGN.md §3 wire format)"}
    e2e = {"value": world * B * args.steps / (e2e_ms / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": B * ns * 8, "d2h_bytes_per_step": B * net.n_out * 8}

    check, cpu = None, None
    if rank == 0 and not args.no_check:
        check, cpu = bench_check(ctx, net, shard(n_batches), 3_000_000, dev, cpu_leg=(world == 1))

    extra = {}
    if rank == 0 and not args.no_extra:
        extra = micro_extra(ctx, stream, dev)
        from bench_configs import table2_breakdown
        extra["table2_cfg4"] = table2_breakdown(ctx, net, imgs_host[0], stream, keygen_s)
        from bench_configs import paper_schedule_throughput
        extra["paper_schedule_cfg4"] = paper_schedule_throughput(stream, imgs_host[0], float_logits_torch)
        if world == 1:   # BASELINE.md / SURVEY §8(d) CPU-oracle subsets of configs 1, 2, 3, 5b (~40 s)
            from bench_configs import cpu_oracle_subsets
            extra["cpu_oracle_subsets"] = cpu_oracle_subsets()

    # result collection to rank 0 (outside the timed region): NCCL gather of the logits
    gather_to_rank0(logits_dev)
    # client-server data plane: rank 0 encrypts a global batch, scatters
    # the ciphertext words over NCCL, every rank evaluates its block, the level-0 words are gathered
    # back; they must equal, bit for bit, rank 0's own single-GPU evaluation of the whole batch
    dist_check = None
    if world > 1:
        from paper_2104_03152_b200.dist import client_server_round
        Bc = 4
        imgs_c = mnist_like_images(world * Bc, 4, start=50_000) if rank == 0 else None
        logits_c, words_c, _ = client_server_round(ctx, net, imgs_c, 4_000_000, dev)
        if rank == 0:
            slots_c = he_im2col_encode_batch(imgs_c, 7, 7, 3, ns)
            ref = net.forward(ctx.he_encrypt(ctx.he_encode(slots_c, 2.0 ** net.plan["in_log2"], net.top),
                                             4_000_000))
            rw = torch.empty_like(words_c)
            ctx.he_ct_export_words(ref, rw)
            dist_check = {"ranks": world, "images": world * Bc, "collectives": "scatter (input words) + gather "
                          "(level-0 words), NCCL", "bitwise_equal_single_gpu": bool(torch.equal(rw, words_c))}

    extra["communication_cfg4"] = comm
    # keys at rest: switching keys of this small-prime context are u32 Montgomery words only
    n_keys = len(rotation_steps(conv_g=CONV_G, fc_bsgs=True, fc1_g=FC1_G))
    kw = ctx.L * 2 * (ctx.L + ctx.K) * ctx.N
    extra["key_memory_cfg4"] = {"resident_bytes_after_the_run": ctx.he_key_bytes(), "galois_keys": n_keys,
                                "u32_at_rest_bytes": 2 * ctx.L * ctx.N * 8 + (1 + n_keys) * kw * 4,
                                "round1_layout_bytes": 2 * ctx.L * ctx.N * 8 + (1 + n_keys) * kw * 12,
                                "note": "relin + Galois keys as u32 (4 B / residue); round 1 held u64 + u32 copies "
                                        "(12 B / residue); u64 forms are materialised only on demand"}
    return dict(value=value, ms=ms, launches=launches, clocks=clk.summary(), roofline=roofline,
                breakdown=breakdown, e2e=e2e, extra=extra, check=check, cpu=cpu, dist_check=dist_check)


def micro_extra(ctx_cnn, stream, dev):
    """Config 2 (NTT GB/s) and config 3 (key-switch rotations/s) shapes, device-timed."""
    import torch
    from paper_2104_03152_b200 import Context
    from synthetic import CFG2_PRIME_BITS, CFG3, messages
    out = {}
    # config 2: N=16384, L=8, B=256 forward / inverse / fused ring product
    N, L, B = 1 << 14, 8, 256
    c2 = Context(14, CFG2_PRIME_BITS(L), 0, 1)
    c2.he_set_stream(stream)
    q = torch.tensor([int(x) for x in c2.primes], dtype=torch.float64, device=dev)
    a = (torch.rand((B, L, N), dtype=torch.float64, device=dev) * q[None, :, None]).to(torch.int64)
    b = (torch.rand((B, L, N), dtype=torch.float64, device=dev) * q[None, :, None]).to(torch.int64)
    o = torch.empty_like(a)

    def t(fn, reps=5):
        fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) / reps / 1e3

    s_f = t(lambda: c2.he_ntt_forward(a, B, L))
    s_i = t(lambda: c2.he_ntt_inverse(a, B, L))
    s_m = t(lambda: c2.he_ntt_mul_intt(a, b, o, B, L))
    nbytes = 16 * N * L * B
    peaks = load_peaks()
    out["ntt_cfg2"] = {"shape": "N=16384 L=8 B=256 (4.3 GB/s basis: 16 N L B bytes)",
                       "fwd_GBps": round(nbytes / s_f / 1e9, 1), "inv_GBps": round(nbytes / s_i / 1e9, 1),
                       "fused_fwd_mul_inv_GBps": round(24 * N * L * B / s_m / 1e9, 1),
                       "roofline": roofline_block("ntt_cfg2_fwd", nbytes / s_f / 1e9, 0.5 * N * 14 * L * B / s_f / 1e9,
                                                  peaks, bfly_peak=BFLY64_GPS)}
    del a, b, o
    # config 3: N=16384, 8 data + 2 special 50-bit primes, 256 ciphertexts, rotations by 2^r and ct x ct
    c3 = Context(CFG3.logN, CFG3.bits, CFG3.n_special, CFG3.seed)
    c3.he_set_stream(stream)
    steps = [1 << r for r in range(14)]
    c3.he_keygen(steps)
    Bc = 256
    z = torch.from_numpy(messages(Bc, c3.slots, seed=CFG3.seed)).to(dev)
    ct = c3.he_encrypt(c3.he_encode(z, 2.0 ** 50, c3.L - 1), 0)
    s_rot = t(lambda: [c3.he_rotate(ct, s) for s in steps], reps=2)
    # kernel breakdown of one batch of rotations (the in-library profiler: CUDA events per launch)
    c3.he_profile_enable(True)
    for s_ in steps:
        c3.he_rotate(ct, s_)
    torch.cuda.synchronize(dev)
    prof3 = c3.he_profile_read()
    c3.he_profile_enable(False)
    tot3 = sum(v[1] for v in prof3.values()) or 1.0
    top3 = max(prof3, key=lambda k: prof3[k][1])
    p3 = (prof3[top3] + [0.0] * 5)[:5]
    rot_break = {k: round(v[1] / tot3, 3) for k, v in sorted(prof3.items(), key=lambda kv: -kv[1][1])}
    s_mul = t(lambda: c3.he_rescale(c3.he_relinearize(c3.he_mul(ct, ct))), reps=3)
    out["keyswitch_cfg3"] = {"shape": "N=16384, 8+2 x 50-bit primes, 256 ciphertexts, top level",
                             "rotations_per_s": round(Bc * len(steps) / s_rot, 1),
                             "rotation_breakdown": rot_break,
                             "roofline": roofline_block("cfg3_" + top3, (p3[2] / p3[0]) / (p3[1] / p3[0] / 1e3) / 1e9,
                                                        (p3[4] / p3[0]) / (p3[1] / p3[0] / 1e3) / 1e9, peaks,
                                                        kernel=top3, share=p3[1] / tot3,
                                                        # ModUp is transforms only: the butterfly roof applies
                                                        bfly_peak=BFLY64_GPS if top3 == "ks_modup" else None),
                             "mul_relin_rescale_per_s": round(Bc / s_mul, 1)}
    del c3, ct
    # config 1: one encrypted vec-mat (x 64 values replicated, W 64x10), batch 1: latency
    from bench_configs import cfg1_latency, cfg5b_throughput, table45_ops
    out["vecmat_cfg1"] = cfg1_latency(stream, t)
    # config 5b: deep chain, N=32768, 18+2 x 50-bit primes, 16 x (mul_plain + rescale) + 4 rotate-and-add
    out["deep_chain_cfg5b"] = cfg5b_throughput(stream, t, dev)
    # PAPER.md Tables 4-5 op set at the paper's parameters (latency, one ciphertext)
    out["ops_table45"] = table45_ops(stream, t)
    return out


def roofline_block(tag, gbs, gops, peaks, kernel=None, share=None, bfly_peak=None):
    """Roofline of a secondary metric's dominant kernel: HBM fraction of the algorithmic bytes, and the
    integer-pipe fraction from the ncu-measured mix of that kernel (profiles/r02/pipe_mix.json entry
    `tag`: the modop rate at which its busiest pipe saturates), when captured."""
    r = {"kernel": kernel or tag, "hbm_achieved_GBps": round(gbs, 1), "hbm_peak_GBps": peaks["hbm_gbs"],
         "hbm_frac": round(gbs / peaks["hbm_gbs"], 4), "alu_achieved_Gmodops": round(gops, 1)}
    if share is not None:
        r["share_of_batch"] = round(share, 3)
    mix = PIPE_MIX.get(tag)
    if mix:
        peak = mix["alg_ops_per_launch"] / (mix["ncu_duration_s"] * mix["busiest_pipe_util"]) / 1e9
        r.update({"bound": "alu", "alu_peak_Gmodops": round(peak, 1), "alu_frac": round(gops / peak, 4),
                  "busiest_pipe": mix["busiest_pipe"], "peak_source": "ncu mix (profiles/r02/pipe_mix.json)"})
    elif bfly_peak:   # a plain transform: its modops are butterflies, the roof the measured butterfly rate
        r.update({"bound": "alu", "alu_peak_Gmodops": round(bfly_peak, 1), "alu_frac": round(gops / bfly_peak, 4),
                  "peak_source": "dependent-free 64-bit Harvey butterfly chain measured on B200 "
                                 "(profiles/int_peak.cu -> profiles/r02/int_peak_v2.json)"})
    return r


# ------------------------------------------------------- oracle (CPU) ---
_ORACLE = {}


def float_logits_torch(imgs, w):
    """The paper's network in float64 with torch.nn.functional on the CPU (a library
    pin of the plaintext network, independent of oracle/ and of the CUDA path)."""
    import torch
    t = lambda a: torch.tensor(np.asarray(a), dtype=torch.float64)
    x = torch.nn.functional.conv2d(t(imgs)[:, None], t(w.conv_w), t(w.conv_b), stride=3)
    x = x.flatten(1) ** 2
    x = torch.nn.functional.linear(x, t(w.fc1_w), t(w.fc1_b)) ** 2
    return torch.nn.functional.linear(x, t(w.fc2_w), t(w.fc2_b)).numpy()


def oracle_context():
    from oracle import circuits as OC
    from oracle.oracle import OracleContext
    from paper_2104_03152_b200.cnn import CONV_G, FC1_G
    from synthetic import CFG4
    if "o" not in _ORACLE:   # keys are made once (excluded from timing, like the GPU arm)
        o = OracleContext(CFG4.logN, CFG4.bits, CFG4.n_special, CFG4.seed)
        o.keygen(OC.cnn_rotation_steps(conv_g=CONV_G, fc_bsgs=True, fc1_g=FC1_G))
        _ORACLE["o"] = o
    return _ORACLE["o"]


def bench_check(ctx, net, imgs, stream0, dev, items=None, cpu_leg=True):
    """Correctness of the bench's own launch geometry (one batch of B images, the same calls and
    launch configuration as the timed step), outside every timed region:
      * items (default first, middle, last): their input plaintexts are the ORACLE's integer
        encodings injected into the device-encoded batch (C7: encode is float-sensitive), the batch
        is encrypted (stream stream0 + b) and evaluated on the GPU; the oracle encrypts and evaluates
        the same items with the same stream ids; the output ciphertext words must be equal;
      * all B decrypted logits within 5e-3 of the float64 network (torch.nn.functional) with equal
        argmax (north_star).
    The oracle runs here as the cpu_baseline leg (rank 0): the items in parallel on the host cores,
    timed; returns (check, cpu_baseline)."""
    import torch
    from concurrent.futures import ThreadPoolExecutor
    from oracle import circuits as OC
    from paper_2104_03152_b200.cnn import CONV_G, FC1_G
    from paper_2104_03152_b200.ckks import he_im2col_encode_batch
    from synthetic import CFG4, cnn_weights
    B, ns, N = len(imgs), ctx.slots, ctx.N
    items = items or sorted({0, B // 2, B - 1})
    scale, top = 2.0 ** net.plan["in_log2"], net.top
    slots = he_im2col_encode_batch(imgs, 7, 7, 3, ns)
    o = oracle_context()
    w = cnn_weights(CFG4.seed)
    ms = np.stack([o.encode_coeffs(slots[s], scale)[1] for s in items])
    # GPU: device encode of the batch, rows `items` replaced by the injected oracle encodings
    pt = ctx.he_encode(torch.from_numpy(slots).to(dev), scale, top)
    words = torch.empty((B, top + 1, N), dtype=torch.int64, device=dev)
    ctx.he_pt_export_words(pt, words)
    inj = torch.empty((len(items), top + 1, N), dtype=torch.int64, device=dev)
    ctx.he_pt_export_words(ctx.he_pt_from_int_coeffs(ms, scale, top), inj)
    words[items] = inj
    pt = ctx.he_pt_import_words(words, top, scale)
    out = net.forward(ctx.he_encrypt(pt, stream0))
    logits = ctx.he_decode(ctx.he_decrypt(out), net.n_out)
    gw = out.words()
    ctx.he_sync()
    # oracle on the items (cpu_baseline leg)
    plan = OC.CNN_PLAN_BSGS

    def one(k):
        s = items[k]
        ct = o.encrypt(o.coeffs_to_pt(ms[k], top, scale), stream0 + s)
        y = OC.cnn_forward(o, ct, w, plan, lazy=True, bsgs=True, conv_g=CONV_G, fc1_g=FC1_G)
        return y, o.decode(o.decrypt(y), net.n_out)
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=min(len(items), os.cpu_count() or 1)) as ex:
        res = list(ex.map(one, range(len(items))))
    dt = time.perf_counter() - t0
    exact = [bool(np.array_equal(gw[s], res[k][0].words)) for k, s in enumerate(items)]
    ref = float_logits_torch(imgs, w)
    err = np.max(np.abs(logits - ref), axis=1)
    am = int(np.sum(np.argmax(logits, 1) == np.argmax(ref, 1)))
    check = {"batch": B, "geometry": "the timed step's calls and launch configuration (B images per call)",
             "bitexact_items": [int(s) for s in items], "bitexact": f"{sum(exact)}/{len(items)}",
             "bitexact_ok": all(exact),
             "oracle_logit_err_vs_gpu": float(max(np.max(np.abs(logits[s] - res[k][1])) for k, s in enumerate(items))),
             "max_logit_err": float(np.max(err)), "median_logit_err": float(np.median(err)),
             "within_5e-3": f"{int(np.sum(err < 5e-3))}/{B}", "argmax_equal": f"{am}/{B}",
             "tolerance_ok": bool(np.max(err) < 5e-3 and am == B),
             "reference": "float64 network via torch.nn.functional (CPU); bit-exact items vs oracle/ with the "
                          "oracle's integer encodings injected (C7)"}
    cpu = None
    if cpu_leg:
        cpu = {"value": len(items) / dt, "unit": UNIT, "cores": min(len(items), os.cpu_count() or 1),
               "kind": "oracle", "cpu_model": cpu_model(),
               "sample": f"{len(items)} images (items {items} of the checked batch): encrypt + forward + decrypt "
                         f"through the CPU oracle, one per host thread, {dt:.1f} s"}
    return check, cpu


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_sample(images: int = 1, start: int = 10_000):
    """Oracle CNN (encrypt + forward + decrypt, the GPU arm's evaluation schedule) on
    `images` independent images, in parallel over host threads (the oracle's C calls release the
    GIL); returns (images/s, threads, seconds)."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import circuits as OC
    from oracle.oracle import OracleContext
    from paper_2104_03152_b200.cnn import CONV_G, FC1_G
    from synthetic import CFG4, cnn_weights, mnist_like_images
    o = oracle_context()
    w = cnn_weights(CFG4.seed)
    imgs = mnist_like_images(images, 4, start=start)
    cores = os.cpu_count() or 1

    def one(i):
        ct = OC.cnn_encrypt_input(o, imgs[i], 3_000_000 + start + i, OC.CNN_PLAN_BSGS)
        # the same evaluation schedule as the GPU arm: one-level conv, folded BSGS FC1, BSGS FC2
        return o.decode(o.decrypt(OC.cnn_forward(o, ct, w, lazy=True, bsgs=True, conv_g=CONV_G, fc1_g=FC1_G)), 10)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=min(images, cores)) as ex:
        list(ex.map(one, range(images)))
    dt = time.perf_counter() - t0
    return images / dt, min(images, cores), dt


def run_reference(args, rank, world):
    if rank != 0:
        return None
    # each step: one image per host core through the oracle (encrypt + forward + decrypt),
    # in parallel over the cores (independent images, the oracle's only parallelism)
    per_step = os.cpu_count() or 1
    times = []
    for i in range(args.warmup + args.steps):
        v, cores, dt = oracle_sample(per_step, start=10_000 + i * per_step)
        if i >= args.warmup:
            times.append(dt)
    ms = 1e3 * sum(times) / len(times)
    value = per_step / (ms / 1e3)
    return dict(value=value, ms=ms, cores=per_step, per_step=per_step)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=512, help="images per GPU per step (BASELINE config 5: batch 512)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--no-check", action="store_true", help="skip the correctness check (and the cpu_baseline leg)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl" if args.impl == "ours" else "gloo")

    config = {"workload": "BASELINE config 5 (config-4 CNN on seeded synthetic 28x28 images, sharded)",
              "network": "conv7x7s3x4 -> x^2 -> fc256x64 -> x^2 -> fc64x10 (PAPER.md:98)",
              "ckks": "N=8192, primes [31,26x6,31] (input at level 5, scale 2^30), 47 Galois keys",
              "evaluation": "conv: one level, 8 baby x 8 giant chunk steps; FC1: 64 diagonals by BSGS "
                            "(32 x 2) + fold 4; FC2 padded to 16 outputs: 16 diagonals + fold 4; every rotation sum with one lazy "
                            "ModDown (DESIGN.md §3)",
              "batch_per_gpu": args.batch, "global_batch": args.batch * world,
              "step": "encode+encrypt+conv+square+fc1+square+fc2+decrypt+decode",
              "parallelism": f"dp{world} (independent images, no data-path collective)",
              "l2": "working set per step far larger than the 126 MB L2 (batch 512: 0.4 GB input ciphertexts, 0.7 GB conv ModUp digits, 0.17 GB u32 Galois keys), no flush"}

    if args.impl == "reference":
        r = run_reference(args, rank, world)
        if rank == 0:
            line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": world,
                    "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms"],
                    "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
                    "data": "synthetic", "config": dict(config, batch_per_gpu=r["per_step"],
                                                        global_batch=r["per_step"],
                                                        reference=f"CPU oracle (oracle/), {r['per_step']} images "
                                                                  "per step, one per host core"),
                    "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "oracle",
                                     "sample": f"{r['per_step']} images (encrypt + forward + decrypt) per step, "
                                               "in parallel over the host cores"},
                    "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
            print(json.dumps(line), flush=True)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return

    r = run_ours(args, rank, world, local_rank)
    if rank == 0:
        line = {"metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": r["ms"] / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
                "config": config, "clocks": r["clocks"], "gpu_launches": r["launches"],
                "check": r["check"], "dist_check": r["dist_check"], "e2e": r["e2e"], "roofline": r["roofline"], "cpu_baseline": r["cpu"],
                "breakdown": r["breakdown"], "extra": r["extra"],
                "paper_context": "TenSEAL/SEAL CPU: 1456.29 ms/img (8 vCPU), 887.06 ms/img (16 vCPU), PAPER.md:113"}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

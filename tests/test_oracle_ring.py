"""Pins of the oracle's ring layer against things other than itself:
sympy primality, Python big-int definitions, schoolbook products, cuRAND, mpmath/float sums.
"""
import ctypes
import json
import os
import random
import subprocess

import numpy as np
import pytest
import sympy

from conftest import brv, negacyclic_mul
from oracle.oracle import OracleContext, cdt_table, lib, philox4x32_10, sid, P_ENC_V

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "params.json")))


def _hex(x):
    return int(x, 16)


def _oracle_primes(logN, bits):
    out = (ctypes.c_uint64 * len(bits))()
    arr = (ctypes.c_int * len(bits))(*bits)
    assert lib().orc_select_primes(logN, len(bits), arr, out) == 0
    return [int(x) for x in out]


# ----------------------------------------------------------------- P1 primes ---
@pytest.mark.parametrize("cfg", ["cfg1", "cfg4", "cfg3"])
def test_primes_match_golden_and_rule_C2(cfg):
    g = GOLD["primes"][cfg]
    logN, bits = g["logN"], g["bits"]
    qs = _oracle_primes(logN, bits)
    assert qs == [_hex(x) for x in g["q"]]
    M = 2 << logN
    for i, (q, b) in enumerate(zip(qs, bits)):
        assert sympy.isprime(q)
        assert q % M == 1 and (1 << (b - 1)) < q < (1 << b)
        # largest unused: every NTT-friendly prime between q and 2^b was taken earlier
        p = q + M
        while p < (1 << b):
            if sympy.isprime(p):
                assert p in qs[:i], f"prime {p:#x} skipped"
            p += M


def test_primes_cfg5b():
    g = GOLD["primes"]["cfg5b"]
    qs = _oracle_primes(g["logN"], [50] * g["n"])
    assert qs[0] == _hex(g["first"]) and qs[-1] == _hex(g["last"])
    assert all(sympy.isprime(q) and q % (2 << 15) == 1 for q in qs)
    assert qs == sorted(qs, reverse=True) and len(set(qs)) == 20


# ------------------------------------------------------------------- P1 psi ---
@pytest.mark.parametrize("case", GOLD["min_psi"])
def test_min_psi_golden(case):
    q, N = _hex(case["q"]), case["N"]
    assert lib().orc_min_psi(q, N) == case["psi"]


@pytest.mark.parametrize("q,N", [(_hex("0x7ffe0001"), 8192), (1073741441, 64), (2305843009213692737, 32)])
def test_min_psi_is_minimal_primitive_root(q, N):
    psi = lib().orc_min_psi(q, N)
    assert pow(psi, N, q) == q - 1 and pow(psi, 2 * N, q) == 1
    # independent enumeration: all primitive 2N-th roots are r^e for odd e
    x = 2
    while pow(pow(x, (q - 1) // (2 * N), q), N, q) != q - 1:
        x += 1
    r = pow(x, (q - 1) // (2 * N), q)
    assert psi == min(pow(r, e, q) for e in range(1, 2 * N, 2))


# -------------------------------------------------------------------- P3 NTT ---
def _direct_ntt(a, q, psi, logN):
    N = 1 << logN
    return [sum(int(a[i]) * pow(psi, (2 * brv(j, logN) + 1) * i, q) for i in range(N)) % q
            for j in range(N)]


@pytest.mark.parametrize("logN,q", [(2, 1073741689), (4, 1073741441), (5, 2305843009213692737),
                                    (6, 1073739649)])
def test_ntt_matches_direct_definition_C5(logN, q):
    N = 1 << logN
    psi = lib().orc_min_psi(q, N)
    rng = random.Random(logN)
    a = np.array([rng.randrange(q) for _ in range(N)], dtype=np.uint64)
    b = a.copy()
    lib().orc_ntt_raw(b.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), logN, q, psi)
    assert [int(x) for x in b] == _direct_ntt(a, q, psi, logN)
    lib().orc_intt_raw(b.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), logN, q, psi)
    assert np.array_equal(a, b)


def test_ntt_large_N_horner_and_roundtrip():
    ctx = OracleContext(13, (60, 40, 40, 60), 1, 0)
    rng = np.random.default_rng(7)
    for t, q in enumerate(ctx.q):
        a = rng.integers(0, q, ctx.N, dtype=np.uint64)
        A = ctx.ntt(t, a)
        psi = int(ctx.psis[t])
        for j in rng.integers(0, ctx.N, 6):
            x = pow(psi, 2 * brv(int(j), 13) + 1, q)
            acc = 0
            for c in reversed(a.tolist()):
                acc = (acc * x + int(c)) % q
            assert int(A[j]) == acc
        assert np.array_equal(ctx.intt(t, A), a)


def test_convolution_theorem_vs_schoolbook():
    q, logN = 1073741441, 6
    N = 1 << logN
    psi = lib().orc_min_psi(q, N)
    P = ctypes.POINTER(ctypes.c_uint64)
    rng = np.random.default_rng(3)
    a = rng.integers(0, q, N, dtype=np.uint64)
    b = rng.integers(0, q, N, dtype=np.uint64)
    A, B = a.copy(), b.copy()
    lib().orc_ntt_raw(A.ctypes.data_as(P), logN, q, psi)
    lib().orc_ntt_raw(B.ctypes.data_as(P), logN, q, psi)
    C = np.array([(int(x) * int(y)) % q for x, y in zip(A, B)], dtype=np.uint64)
    lib().orc_intt_raw(C.ctypes.data_as(P), logN, q, psi)
    assert [int(x) for x in C] == negacyclic_mul(a, b, N, q)


def test_spec_small_ring_examples():
    """(1+x)^2 = 1+2x+x^2 and x^3 * x^3 = -x^2 at N=4."""
    q, logN = 1073741689, 2
    psi = lib().orc_min_psi(q, 4)
    P = ctypes.POINTER(ctypes.c_uint64)

    def mul(a, b):
        A = np.array(a, dtype=np.uint64)
        B = np.array(b, dtype=np.uint64)
        lib().orc_ntt_raw(A.ctypes.data_as(P), logN, q, psi)
        lib().orc_ntt_raw(B.ctypes.data_as(P), logN, q, psi)
        C = np.array([(int(x) * int(y)) % q for x, y in zip(A, B)], dtype=np.uint64)
        lib().orc_intt_raw(C.ctypes.data_as(P), logN, q, psi)
        return [int(x) for x in C]

    assert mul([1, 1, 0, 0], [1, 1, 0, 0]) == [1, 2, 1, 0]
    assert mul([0, 0, 0, 1], [0, 0, 0, 1]) == [0, 0, q - 1, 0]


# ------------------------------------------------------------- P4 automorphism ---
def test_automorphism_laws():
    ctx = OracleContext(5, (30, 30, 30), 1, 0)
    N, q = ctx.N, ctx.q[0]
    rng = np.random.default_rng(1)
    a = rng.integers(0, q, N, dtype=np.uint64)
    b = rng.integers(0, q, N, dtype=np.uint64)
    A, B = ctx.ntt(0, a), ctx.ntt(0, b)
    g, h = 5, 25 * 5 % (2 * N)
    # coefficient definition C8 (written here independently): a(X) -> a(X^g)
    coef = [0] * N
    for i in range(N):
        e = i * g % (2 * N)
        if e < N:
            coef[e] = (coef[e] + int(a[i])) % q
        else:
            coef[e - N] = (coef[e - N] - int(a[i])) % q
    assert np.array_equal(ctx.automorph_ntt(A, 0, g), ctx.ntt(0, np.array(coef, dtype=np.uint64)))
    # composition, identity, multiplicativity
    gh = g * h % (2 * N)
    assert np.array_equal(ctx.automorph_ntt(ctx.automorph_ntt(A, 0, h), 0, g), ctx.automorph_ntt(A, 0, gh))
    assert pow(5, N // 2, 2 * N) == 1
    assert np.array_equal(ctx.automorph_ntt(A, 0, 1), A)
    AB = np.array([(int(x) * int(y)) % q for x, y in zip(A, B)], dtype=np.uint64)
    lhs = ctx.automorph_ntt(AB, 0, g)
    ga, gb = ctx.automorph_ntt(A, 0, g), ctx.automorph_ntt(B, 0, g)
    assert np.array_equal(lhs, np.array([(int(x) * int(y)) % q for x, y in zip(ga, gb)], dtype=np.uint64))


def test_automorphism_is_ntt_domain_permutation_a8():
    """a8: out[j] = in[pi(j)] with 2 brv(pi(j)) + 1 = g (2 brv(j) + 1) mod 2N."""
    ctx = OracleContext(6, (30, 30), 1, 0)
    N, logN = ctx.N, ctx.logN
    A = np.random.default_rng(2).integers(0, ctx.q[0], N, dtype=np.uint64)
    for g in (5, 25, 2 * N - 1, 3):
        perm = [brv(((g * (2 * brv(j, logN) + 1)) % (2 * N) - 1) // 2, logN) for j in range(N)]
        assert np.array_equal(ctx.automorph_ntt(A, 0, g), A[perm])


# ------------------------------------------------------------------ P5 sampler ---
def _curand_pin():
    so = os.path.join("/tmp", f"libcurandpin_{os.getuid()}.so")
    src = os.path.join(HERE, "pins", "curand_philox_host.cu")
    if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        try:
            subprocess.check_call(["nvcc", "-O2", "-shared", "-Xcompiler", "-fPIC", src, "-o", so,
                                   "-Wno-deprecated-gpu-targets"])
        except Exception as e:  # pragma: no cover
            pytest.skip(f"nvcc unavailable: {e}")
    L = ctypes.CDLL(so)
    return L


def test_philox_matches_curand():
    L = _curand_pin()
    rng = np.random.default_rng(11)
    for _ in range(200):
        ctr = rng.integers(0, 2 ** 32, 4, dtype=np.uint64)
        key = rng.integers(0, 2 ** 32, 2, dtype=np.uint64)
        c = (ctypes.c_uint32 * 4)(*ctr.tolist())
        k = (ctypes.c_uint32 * 2)(*key.tolist())
        o = (ctypes.c_uint32 * 4)()
        L.curand_philox_host(c, k, o)
        assert philox4x32_10(ctr, key).tolist() == list(o)


def test_cdt_table_pins():
    T = cdt_table()
    g = GOLD["cdt"]
    assert int(T[0]) == g["T0"]
    # float64 direct normalisation agrees to double precision
    x = np.arange(0, 20, dtype=np.float64)
    rho = np.exp(-x ** 2 / (2 * 3.2 ** 2))
    cdf = np.cumsum(np.where(x == 0, rho, 2 * rho)) / (rho[0] + 2 * rho[1:].sum())
    assert np.allclose(T.astype(np.float64) / 2.0 ** 63, cdf, rtol=0, atol=2e-15)
    assert abs(float(T[0]) / 2 ** 63 - float(g["pr_abs_le_0"])) < 1e-14
    var = (2 * (x[1:] ** 2 * rho[1:]).sum()) / (rho[0] + 2 * rho[1:].sum())
    assert abs(np.sqrt(var) - g["truncated_sigma"]) < 1e-7
    assert np.all(np.diff(T.astype(np.float64)) > 0) and int(T[-1]) == 1 << 63


def test_sampler_statistics_and_determinism():
    ctx = OracleContext(13, (30, 30), 1, 5)
    e = np.concatenate([ctx.sample_cdt(sid(3, o, 0)) for o in range(128)])   # 1M samples
    assert abs(e.std() / 3.19999994 - 1) < 0.01 and abs(e.mean()) < 0.02 and np.abs(e).max() <= 19
    t = np.concatenate([ctx.sample_ternary(sid(1, o, 0)) for o in range(32)])
    freq = np.array([(t == v).mean() for v in (-1, 0, 1)])
    assert set(np.unique(t)) <= {-1, 0, 1} and np.all(np.abs(freq - 1 / 3) < 0.005)
    u = ctx.sample_uniform(sid(2, 0, 0), 0)
    assert int(u.max()) < ctx.q[0] and abs(u.astype(np.float64).mean() / ctx.q[0] - 0.5) < 0.01
    assert np.array_equal(ctx.sample_cdt(sid(9, 7, 0)), ctx.sample_cdt(sid(9, 7, 0)))
    assert not np.array_equal(ctx.sample_ternary(sid(P_ENC_V, 1, 0)), ctx.sample_ternary(sid(P_ENC_V, 2, 0)))


# ------------------------------------------------------- wire format pin ---
def test_wire_reference_packer_vs_bitstring():
    """oracle/wire.py against an independent construction: each residue written as a w-bit
    little-endian bit string, concatenated, packed with numpy.packbits(bitorder='little')."""
    from oracle import wire
    rng = np.random.default_rng(0)
    primes = [(1 << 31) - 1, (1 << 26) - 5, (1 << 20) + 7]
    N, level = 64, 2
    w = np.stack([np.stack([rng.integers(0, q, N, dtype=np.uint64) for q in primes]) for _ in range(2)])[None]
    blob = wire.pack(w, primes, level, 1.0)
    bits = []
    for p in range(2):
        for i, q in enumerate(primes):
            wd = int(q).bit_length()
            for x in w[0, p, i]:
                bits.extend((int(x) >> k) & 1 for k in range(wd))
    ref = np.packbits(np.array(bits, dtype=np.uint8), bitorder="little").tobytes()
    assert blob[wire.HEADER_BYTES:] == ref
    assert blob[:8] == b"HECKKS01" and len(blob) == 64 + len(ref)

"""GPU parity of the scheme layer through the C-ABI against
the CPU oracle: keys, encode/decode, encrypt/decrypt, add/sub/negate,
mul_plain/add_plain, tensor, rescale, relinearize, rotate, square and vec_mat.

Integer outputs are compared word for word (bit-exact).  Encoding is compared as
allowed by C7 (the rounding of a float64 FFT may differ from the oracle's
long-double sum at near-ties); every bit-exact ciphertext comparison starts from
oracle plaintexts injected through he_pt_from_int_coeffs / he_pt_import_words.
"""
import numpy as np
import pytest

from oracle import circuits as OC
from oracle.oracle import OCt, OPt, OracleContext
from synthetic import CFG1, messages, vecmat_inputs

pytestmark = pytest.mark.gpu

TINY = dict(logN=10, bits=(50, 40, 40, 50, 50), K=2, seed=9)
TINY_STEPS = [1, 3, -1, 7, 512]


@pytest.fixture(scope="module")
def tiny():
    from paper_2104_03152_b200 import Context
    o = OracleContext(TINY["logN"], TINY["bits"], TINY["K"], TINY["seed"])
    o.keygen(TINY_STEPS)
    g = Context(TINY["logN"], TINY["bits"], TINY["K"], TINY["seed"])
    g.he_keygen(TINY_STEPS)
    return o, g


@pytest.fixture(scope="module")
def cfg1():
    from paper_2104_03152_b200 import Context
    steps = list(range(1, 64))
    o = OracleContext(CFG1.logN, CFG1.bits, CFG1.n_special, CFG1.seed)
    o.keygen(steps)
    g = Context(CFG1.logN, CFG1.bits, CFG1.n_special, CFG1.seed)
    g.he_keygen(steps)
    return o, g


def rand_ct(o, level, B, seed, size=2):
    rng = np.random.default_rng(seed)
    w = np.stack([np.stack([np.stack([rng.integers(0, o.q[i], o.N, dtype=np.uint64) for i in range(level + 1)])
                            for _ in range(size)]) for _ in range(B)])
    return w


def oracle_ct(o, z, scale, level, sid):
    return o.encrypt(o.encode(z, scale, level), sid)


# -------------------------------------------------------------------- keys ---
@pytest.mark.parametrize("which", ["tiny", "cfg1"])
def test_keys_bit_exact(which, tiny, cfg1):
    o, g = tiny if which == "tiny" else cfg1
    assert np.array_equal(g.he_key_export(0), o.secret_key()[1])
    assert np.array_equal(g.he_key_export(1), o.public_key())
    assert np.array_equal(g.he_key_export(2), o.relin_key())
    for st in (TINY_STEPS if which == "tiny" else [1, 2, 31, 63]):
        assert np.array_equal(g.he_key_export(3, st), o.galois_key(st)), st


# ---------------------------------------------------------- encode/decode ---
@pytest.mark.parametrize("scale_log2,n", [(40, 4096), (40, 10), (26, 3000), (50, 1)])
def test_encode_within_C7_and_injection_exact(cfg1, scale_log2, n):
    o, g = cfg1
    z = messages(3, n, seed=scale_log2 + n)
    scale = 2.0 ** scale_log2
    pt = g.he_encode(z, scale, 2)
    w = pt.words()
    pre_g = g.he_encode_unrounded(z, scale)   # the device's values before rounding (C7 hook)
    for b in range(3):
        pre, m = o.encode_coeffs(z[b], scale)
        # north_star: float64 encode within 1e-9 relative (to the coefficient vector's max-norm,
        # the scale at which a float64 FFT's error is defined)
        nrm = max(1.0, float(np.max(np.abs(pre))))
        assert np.max(np.abs(pre_g[b] - pre)) <= 1e-9 * nrm
        # GPU integers: centred limb-0 residues of its own encoding
        c0 = o.intt(0, w[b, 0]).astype(object)
        q0 = o.q[0]
        mg = np.array([int(x) - q0 if int(x) > q0 // 2 else int(x) for x in c0], dtype=np.float64)
        # ... are exactly its pre-rounding values rounded half away from zero (C7)
        assert np.array_equal(mg, np.sign(pre_g[b]) * np.floor(np.abs(pre_g[b]) + 0.5))
        # ... and equal the oracle's integers except where the oracle's value is within the
        # 1e-9 tolerance of a rounding tie
        tie = np.abs(np.abs(pre - np.trunc(pre)) - 0.5) <= 1e-9 * nrm
        assert np.array_equal(mg[~tie], m[~tie].astype(np.float64))
        # injection of the oracle's integers reproduces its plaintext words exactly
        inj = g.he_pt_from_int_coeffs(m, scale, 2).words()[0]
        assert np.array_equal(inj, o.coeffs_to_pt(m, 2, scale).words)


def test_decode_matches_oracle(cfg1):
    o, g = cfg1
    z = messages(2, 4096, seed=11)
    for lvl in (0, 2):
        pts = [o.encode(z[b], 2.0 ** 40, lvl) for b in range(2)]
        gp = g.he_pt_import_words(np.stack([p.words for p in pts]), lvl, 2.0 ** 40)
        got = g.he_decode(gp, 4096)
        for b in range(2):
            ref = o.decode(pts[b], 4096)
            assert np.allclose(got[b], ref, rtol=1e-9, atol=1e-9)
            assert np.max(np.abs(got[b] - z[b])) < 2.0 ** -25


def test_encode_errors(cfg1):
    from paper_2104_03152_b200 import HEError
    o, g = cfg1
    with pytest.raises(HEError) as e:
        g.he_encode(np.zeros(4097), 2.0 ** 40, 2)
    assert e.value.name == "TOO_MANY_VALUES"
    with pytest.raises(HEError) as e:
        g.he_encode(np.full(8, 1e12), 2.0 ** 40, 2)
    assert e.value.name == "SCALE_OVERFLOW"
    # device input is asynchronous: the overflow is reported (once) by the next he_sync
    import torch
    g.he_encode(torch.full((1, 8), 1e12, dtype=torch.float64, device="cuda"), 2.0 ** 40, 2)
    with pytest.raises(HEError) as e:
        g.he_sync()
    assert e.value.name == "SCALE_OVERFLOW"
    g.he_sync()


# ---------------------------------------------------------- encrypt/decrypt ---
@pytest.mark.parametrize("which", ["tiny", "cfg1"])
def test_encrypt_decrypt_bit_exact(which, tiny, cfg1):
    o, g = tiny if which == "tiny" else cfg1
    lvl = o.L - 1
    z = messages(3, o.slots, seed=5)
    pts = [o.encode(z[b], 2.0 ** 30, lvl) for b in range(3)]
    gp = g.he_pt_import_words(np.stack([p.words for p in pts]), lvl, 2.0 ** 30)
    ct = g.he_encrypt(gp, 100)
    w = ct.words()
    for b in range(3):
        assert np.array_equal(w[b], o.encrypt(pts[b], 100 + b).words), b
    dec = g.he_decrypt(ct).words()
    for b in range(3):
        ref = o.decrypt(OCt(w[b], lvl, 2.0 ** 30)).words
        assert np.array_equal(dec[b], ref)
    vals = g.he_decode(g.he_decrypt(ct), o.slots)
    # fresh noise v e + e0 + e1 s has coefficient std ~ sigma sqrt(4N/3) ~ 340 at N=8192; a slot sums
    # N such terms (std ~ 340 sqrt(N/2) ~ 2e4), so |error| / 2^30 is ~ 2e-5 typical, ~1e-4 max
    assert np.max(np.abs(vals - z)) < 1e-3


@pytest.mark.parametrize("which", ["tiny", "cfg1", "small"])
def test_encode_encrypt_equals_encode_then_encrypt(which, tiny, cfg1, small):
    """he_encode_encrypt (m fed into the e0 transform) gives exactly the words of
    he_encrypt(he_encode(z)) -- the transform is linear mod q_i -- host and device input, a ragged
    batch, two levels, 64-bit and 32-bit engines."""
    import torch
    o, g = (tiny if which == "tiny" else cfg1 if which == "cfg1" else small[:2])
    scale = 2.0 ** (26 if which == "small" else 30)
    z = messages(5, o.slots // 2 + 3, seed=17)
    for lvl in (o.L - 1, 1):
        ref = g.he_encrypt(g.he_encode(z, scale, lvl), 300).words()
        assert np.array_equal(g.he_encode_encrypt(z, scale, lvl, 300).words(), ref)
        zd = torch.from_numpy(z).cuda()
        assert np.array_equal(g.he_encode_encrypt(zd, scale, lvl, 300).words(), ref)
    vals = g.he_decode(g.he_decrypt(g.he_encode_encrypt(z, scale, o.L - 1, 9)), z.shape[1])
    assert np.max(np.abs(vals - z)) < (1e-2 if which == "small" else 1e-3)


# ------------------------------------------------------------- arithmetic ---
def test_pointwise_ops_bit_exact(tiny):
    o, g = tiny
    lvl = 2
    x, y = rand_ct(o, lvl, 3, 1), rand_ct(o, lvl, 3, 2)
    gx, gy = g.he_ct_import_words(x, lvl, 1.0), g.he_ct_import_words(y, lvl, 1.0)
    add, sub, neg = g.he_add(gx, gy).words(), g.he_sub(gx, gy).words(), g.he_negate(gx).words()
    ten = g.he_mul(gx, gy).words()
    p = rand_ct(o, lvl, 1, 3, size=1)[0, 0]
    gpt = g.he_pt_import_words(p[None], lvl, 3.0)
    mp, ap = g.he_mul_plain(gx, gpt).words(), None
    gpt1 = g.he_pt_import_words(p[None], lvl, 1.0)
    ap = g.he_add_plain(gx, gpt1).words()
    for b in range(3):
        ox, oy = OCt(x[b], lvl, 1.0), OCt(y[b], lvl, 1.0)
        assert np.array_equal(add[b], o.add(ox, oy).words)
        assert np.array_equal(sub[b], o.sub(ox, oy).words)
        assert np.array_equal(neg[b], o.negate(ox).words)
        assert np.array_equal(ten[b], o.tensor(ox, oy).words)
        assert np.array_equal(mp[b], o.mul_plain(ox, OPt(p, lvl, 3.0)).words)
        assert np.array_equal(ap[b], o.add_plain(ox, OPt(p, lvl, 1.0)).words)
    # broadcast: B=1 operand against B=3
    g1 = g.he_ct_import_words(y[:1], lvl, 1.0)
    add1 = g.he_add(gx, g1).words()
    for b in range(3):
        assert np.array_equal(add1[b], o.add(OCt(x[b], lvl, 1.0), OCt(y[0], lvl, 1.0)).words)


def test_scheme_errors(tiny):
    from paper_2104_03152_b200 import HEError
    o, g = tiny
    x = g.he_ct_import_words(rand_ct(o, 2, 1, 1), 2, 1.0)
    y = g.he_ct_import_words(rand_ct(o, 1, 1, 2), 1, 1.0)
    z = g.he_ct_import_words(rand_ct(o, 2, 1, 3), 2, 2.0)
    for fn, args, name in [(g.he_add, (x, y), "LEVEL_MISMATCH"), (g.he_add, (x, z), "SCALE_MISMATCH"),
                           (g.he_rotate, (x, 2), "MISSING_GALOIS_KEY")]:
        with pytest.raises(HEError) as e:
            fn(*args)
        assert e.value.name == name
    lvl0 = g.he_ct_import_words(rand_ct(o, 0, 1, 4), 0, 1.0)
    with pytest.raises(HEError) as e:
        g.he_rescale(lvl0)
    assert e.value.name == "LEVEL_EXHAUSTED"
    bad = rand_ct(o, 2, 1, 5)
    bad[0, 0, 0, 0] = np.uint64(o.q[0])
    with pytest.raises(HEError):
        g.he_ct_import_words(bad, 2, 1.0)


@pytest.mark.parametrize("size", [2, 3])
def test_rescale_bit_exact(tiny, size):
    o, g = tiny
    for lvl in (1, 2):
        x = rand_ct(o, lvl, 3, 10 + lvl, size=size)
        got = g.he_rescale(g.he_ct_import_words(x, lvl, 2.0 ** 40, size=size))
        assert got.level == lvl - 1 and got.scale == 2.0 ** 40 / o.q[lvl]
        w = got.words()
        for b in range(3):
            assert np.array_equal(w[b], o.rescale(OCt(x[b], lvl, 2.0 ** 40)).words)


@pytest.mark.parametrize("which", ["tiny", "cfg1"])
def test_relinearize_and_square_bit_exact(which, tiny, cfg1):
    o, g = tiny if which == "tiny" else cfg1
    for lvl in range(o.L):
        x = rand_ct(o, lvl, 2, 20 + lvl, size=3)
        w = g.he_relinearize(g.he_ct_import_words(x, lvl, 1.0, size=3)).words()
        for b in range(2):
            assert np.array_equal(w[b], o.relinearize(OCt(x[b], lvl, 1.0)).words), (lvl, b)
    lvl = o.L - 1
    z = messages(2, o.slots, seed=7)
    cts = [oracle_ct(o, z[b], 2.0 ** 30, lvl, b) for b in range(2)]
    gsq = g.he_square(g.he_ct_import_words(np.stack([c.words for c in cts]), lvl, 2.0 ** 30))
    w = gsq.words()
    for b in range(2):
        ref = o.square(cts[b])
        assert np.array_equal(w[b], ref.words) and gsq.scale == ref.scale


@pytest.mark.parametrize("which", ["tiny", "cfg1"])
def test_rotate_bit_exact(which, tiny, cfg1):
    o, g = tiny if which == "tiny" else cfg1
    steps = TINY_STEPS if which == "tiny" else [1, 5, 63]
    for lvl in sorted({0, o.L - 1}):
        x = rand_ct(o, lvl, 3, 30 + lvl)
        gx = g.he_ct_import_words(x, lvl, 1.0)
        for st in steps:
            w = g.he_rotate(gx, st).words()
            for b in range(3):
                assert np.array_equal(w[b], o.rotate(OCt(x[b], lvl, 1.0), st).words), (lvl, st, b)


def test_rotation_semantics(cfg1):
    """Decrypted rotation is np.roll(z, -k) (C6 left rotation) and composes."""
    o, g = cfg1
    z = messages(1, o.slots, seed=8)
    ct = g.he_encrypt(g.he_encode(z, 2.0 ** 40, 2), 3)
    r = g.he_rotate(g.he_rotate(ct, 2), 3)
    got = g.he_decode(g.he_decrypt(r), o.slots)[0]
    assert np.max(np.abs(got - np.roll(z[0], -5))) < 1e-5


# ----------------------------------------------------------------- vec_mat ---
def _inject(g, o, vecs, scale, level):
    """Oracle-encoded integer coefficients of each vector -> one GPU plaintext batch."""
    ms = np.stack([o.encode_coeffs(v, scale)[1] for v in vecs])
    return g.he_pt_from_int_coeffs(ms, scale, level)


def test_vec_mat_cfg1_bit_exact_and_tolerance(cfg1):
    """Config 1: x ~ U[-1,1]^64 replicated, W 64x10 ~ N(0, 0.1^2), diagonal method (C17)."""
    o, g = cfg1
    x, W = vecmat_inputs(0)
    lvl = o.L - 1
    xs = OC.replicate(x, o.slots)
    oct_ = oracle_ct(o, xs, 2.0 ** 40, lvl, 0)
    ref = OC.vec_mat(o, oct_, W, None, replicate_out=False)
    D = OC.vecmat_diagonals(W, o.slots, False)
    gd = _inject(g, o, D, float(o.q[lvl]), lvl)
    gct = g.he_ct_import_words(oct_.words[None], lvl, 2.0 ** 40)
    out = g.he_vec_mat_pt(gct, gd)
    assert np.array_equal(out.words()[0], ref.words) and out.scale == ref.scale
    # the all-GPU path (own encode of x, W) within the config-1 tolerance
    full = g.he_vec_mat(g.he_encrypt(g.he_encode(xs, 2.0 ** 40, lvl), 0), W)
    y = g.he_decode(g.he_decrypt(full), 10)[0]
    assert np.max(np.abs(y - x @ W)) < 1e-6


def test_vec_mat_batch_and_bias(tiny):
    o, g = tiny
    rng = np.random.default_rng(3)
    n, m = 8, 8
    W, bias = rng.normal(0, 0.1, (n, m)), rng.normal(0, 0.1, m)
    lvl = o.L - 1
    # tiny has keys for steps 1, 3, 7 only -> use n = 8 needs 1..7: regenerate a context
    from paper_2104_03152_b200 import Context
    o2 = OracleContext(TINY["logN"], TINY["bits"], TINY["K"], 4)
    o2.keygen(range(1, n))
    g2 = Context(TINY["logN"], TINY["bits"], TINY["K"], 4)
    g2.he_keygen(range(1, n))
    xs = [OC.replicate(rng.uniform(-1, 1, n), o2.slots) for _ in range(3)]
    octs = [oracle_ct(o2, v, 2.0 ** 30, lvl, b) for b, v in enumerate(xs)]
    D = OC.vecmat_diagonals(W, o2.slots, True)
    ps = float(o2.q[lvl])
    gd = _inject(g2, o2, D, ps, lvl)
    bscale = 2.0 ** 30 * ps / o2.q[lvl]
    gb = _inject(g2, o2, [OC.vecmat_bias_slots(bias, o2.slots, True)], bscale, lvl - 1)
    out = g2.he_vec_mat_pt(g2.he_ct_import_words(np.stack([c.words for c in octs]), lvl, 2.0 ** 30), gd, gb)
    w = out.words()
    for b in range(3):
        ref = OC.vec_mat(o2, octs[b], W, bias, replicate_out=True)
        assert np.array_equal(w[b], ref.words), b


def test_vec_mat_lazy_bit_exact(cfg1):
    """One-ModDown vec_mat (QP diagonals) vs the oracle's vec_mat_lazy, cfg1 shape, B=2."""
    o, g = cfg1
    x, W = vecmat_inputs(0)
    lvl = o.L - 1
    xs = OC.replicate(x, o.slots)
    octs = [oracle_ct(o, xs, 2.0 ** 40, lvl, b) for b in range(2)]
    D = OC.vecmat_diagonals(W, o.slots, False)
    ps = float(o.q[lvl])
    gD = g.he_pt_from_int_coeffs_qp(np.stack([o.encode_coeffs(d, ps)[1] for d in D]), ps, lvl)
    assert gD.limbs == lvl + 1 + o.K
    out = g.he_vec_mat_pt(g.he_ct_import_words(np.stack([c.words for c in octs]), lvl, 2.0 ** 40), gD)
    W2 = out.words()
    for b in range(2):
        ref = OC.vec_mat_lazy(o, octs[b], W, None, replicate_out=False)
        assert np.array_equal(W2[b], ref.words), b
    y = g.he_decode(g.he_decrypt(out), 10)
    assert np.max(np.abs(y - x @ W)) < 1e-6


# ------------------------------------------- small-prime (32-bit) engine ---
SMALL = dict(logN=11, bits=(31, 26, 26, 26, 31), K=1, seed=13)


@pytest.fixture(scope="module")
def small():
    from paper_2104_03152_b200 import Context
    steps = [1, 5, -3, 1024]
    o = OracleContext(SMALL["logN"], SMALL["bits"], SMALL["K"], SMALL["seed"])
    o.keygen(steps)
    g = Context(SMALL["logN"], SMALL["bits"], SMALL["K"], SMALL["seed"])
    g.he_keygen(steps)
    return o, g, steps


def test_small_prime_keyswitch_paths_bit_exact(small):
    """All primes < 2^31: rotate / rotate-and-add (fused ModUp + Montgomery inner product),
    relinearize, square and rescale through the 32-bit engine, at every level, word for word."""
    o, g, steps = small
    assert np.array_equal(g.he_key_export(2), o.relin_key())
    for lvl in range(o.L):
        x = rand_ct(o, lvl, 3, 40 + lvl)
        gx = g.he_ct_import_words(x, lvl, 1.0)
        for st in steps:
            w = g.he_rotate(gx, st).words()
            for b in range(3):
                assert np.array_equal(w[b], o.rotate(OCt(x[b], lvl, 1.0), st).words), (lvl, st, b)
        x3 = rand_ct(o, lvl, 2, 60 + lvl, size=3)
        w = g.he_relinearize(g.he_ct_import_words(x3, lvl, 1.0, size=3)).words()
        for b in range(2):
            assert np.array_equal(w[b], o.relinearize(OCt(x3[b], lvl, 1.0)).words), (lvl, b)
        if lvl >= 1:
            w = g.he_rescale(gx).words()
            for b in range(3):
                assert np.array_equal(w[b], o.rescale(OCt(x[b], lvl, 1.0)).words), (lvl, b)
        # fused square (ct_square_relin: d2 = x1^2 on the digit loads, d0 / d1 in the ModDown
        # epilogue) at every level, batch 1 and 3, against the oracle's tensor -> relinearize
        for Bq in ((1, 3) if lvl >= 1 else ()):
            xs = x[:Bq]
            w = g.he_square(g.he_ct_import_words(xs, lvl, 1.0)).words()
            for b in range(Bq):
                assert np.array_equal(w[b], o.square(OCt(xs[b], lvl, 1.0)).words), ("square", lvl, Bq, b)
    z = messages(2, o.slots, seed=3)
    lvl = o.L - 1
    cts = [oracle_ct(o, z[b], 2.0 ** 26, lvl, b) for b in range(2)]
    gsq = g.he_square(g.he_ct_import_words(np.stack([c.words for c in cts]), lvl, 2.0 ** 26))
    for b in range(2):
        assert np.array_equal(gsq.words()[b], o.square(cts[b]).words)


def test_small_prime_vec_mat_both_forms_bit_exact(small):
    o, g, _ = small
    from paper_2104_03152_b200 import Context
    n = 8
    o2 = OracleContext(SMALL["logN"], SMALL["bits"], SMALL["K"], 21)
    o2.keygen(range(1, n))
    g2 = Context(SMALL["logN"], SMALL["bits"], SMALL["K"], 21)
    g2.he_keygen(range(1, n))
    rng = np.random.default_rng(9)
    W = rng.normal(0, 0.1, (n, n))
    lvl = o2.L - 1
    octs = [oracle_ct(o2, OC.replicate(rng.uniform(-1, 1, n), o2.slots), 2.0 ** 26, lvl, b) for b in range(3)]
    gct = g2.he_ct_import_words(np.stack([c.words for c in octs]), lvl, 2.0 ** 26)
    D = OC.vecmat_diagonals(W, o2.slots, True)
    ps = float(o2.q[lvl])
    ms = np.stack([o2.encode_coeffs(d, ps)[1] for d in D])
    plain = g2.he_vec_mat_pt(gct, g2.he_pt_from_int_coeffs(ms, ps, lvl)).words()
    lazy = g2.he_vec_mat_pt(gct, g2.he_pt_from_int_coeffs_qp(ms, ps, lvl)).words()
    for b in range(3):
        assert np.array_equal(plain[b], OC.vec_mat(o2, octs[b], W, None, True).words), b
        assert np.array_equal(lazy[b], OC.vec_mat_lazy(o2, octs[b], W, None, True).words), b


@pytest.mark.parametrize("which", ["cfg1", "small"])
def test_vec_mat_bsgs_bit_exact(which, cfg1, small):
    """BSGS vec_mat vs the oracle's vec_mat_bsgs: 64-bit generic path (cfg1, n=64, g=16) and the
    fused small-prime kernel (n=8, g=4), batch 2."""
    if which == "cfg1":
        o, g = cfg1
        x, W = vecmat_inputs(0)
        gg, rep, scale = 16, False, 2.0 ** 40
    else:
        from paper_2104_03152_b200 import Context
        o = OracleContext(SMALL["logN"], SMALL["bits"], SMALL["K"], 31)
        o.keygen(range(1, 8))
        g = Context(SMALL["logN"], SMALL["bits"], SMALL["K"], 31)
        g.he_keygen(range(1, 8))
        rng = np.random.default_rng(8)
        x, W = rng.uniform(-1, 1, 8), rng.normal(0, 0.1, (8, 8))
        gg, rep, scale = 4, True, 2.0 ** 26
    lvl = o.L - 1
    xs = OC.replicate(x, o.slots)
    octs = [oracle_ct(o, xs, scale, lvl, b) for b in range(2)]
    ps = float(o.q[lvl])
    E = OC.bsgs_diagonals(OC.vecmat_diagonals(W, o.slots, rep), gg).reshape(-1, o.slots)
    gD = g.he_pt_from_int_coeffs_qp(np.stack([o.encode_coeffs(v, ps)[1] for v in E]), ps, lvl)
    out = g.he_vec_mat_bsgs_pt(g.he_ct_import_words(np.stack([c.words for c in octs]), lvl, scale), gD, gg)
    Wo = out.words()
    for b in range(2):
        assert np.array_equal(Wo[b], OC.vec_mat_bsgs(o, octs[b], W, None, rep, g=gg).words), b
    y = g.he_decode(g.he_decrypt(out), W.shape[1])
    assert np.max(np.abs(y - x @ W)) < (1e-6 if which == "cfg1" else 5e-3)

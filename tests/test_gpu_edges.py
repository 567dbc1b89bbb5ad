"""Edge and degenerate cases through the C-ABI on the GPU (task ③): empty encodings, ragged
batches, the identity rotation with and without a key, n = 1 vec_mat / dot (no rotations),
replication exhaustion (C17), level exhaustion, mismatched batches, repeated keygen, decode
bounds, and a wide ragged batch compared word for word with the oracle item by item."""
import numpy as np
import pytest

from oracle import circuits as OC
from oracle.oracle import OCt, OracleContext

pytestmark = pytest.mark.gpu

P = dict(logN=10, bits=(50, 40, 40, 50), K=1, seed=3)


@pytest.fixture(scope="module")
def pair():
    from paper_2104_03152_b200 import Context
    o = OracleContext(P["logN"], P["bits"], P["K"], P["seed"])
    o.keygen([1, 2, 4])
    g = Context(P["logN"], P["bits"], P["K"], P["seed"])
    g.he_keygen([1, 2, 4])
    return o, g


def test_empty_encoding_and_zero_message(pair):
    o, g = pair
    pt = g.he_encode(np.zeros((3, 0)), 2.0 ** 30, 2)          # n = 0 values
    assert np.all(pt.words() == 0)
    ct = g.he_encrypt(pt, 5)
    z = g.he_decode(g.he_decrypt(ct), o.slots)
    assert np.max(np.abs(z)) < 1e-4
    for b in range(3):   # encryption of the zero plaintext still matches the oracle word for word
        assert np.array_equal(ct.words()[b], o.encrypt(o.coeffs_to_pt(np.zeros(o.N, np.int64), 2, 2.0 ** 30), 5 + b).words)


def test_identity_rotation_without_key_is_a_copy(pair):
    o, g = pair
    rng = np.random.default_rng(0)
    w = np.stack([np.stack([rng.integers(0, o.q[i], o.N, dtype=np.uint64) for i in range(3)]) for _ in range(2)])[None]
    ct = g.he_ct_import_words(w, 2, 1.0)
    assert np.array_equal(g.he_rotate(ct, o.slots).words(), w)
    assert np.array_equal(g.he_rotate(ct, 0).words(), w)


def test_vec_mat_and_dot_with_one_term(pair):
    o, g = pair
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, o.slots)
    oct_ = o.encrypt(o.encode(x, 2.0 ** 30, 2), 1)
    ct = g.he_ct_import_words(oct_.words[None], 2, 2.0 ** 30)
    W = np.array([[0.75]])
    D = OC.vecmat_diagonals(W, o.slots, True)
    ps = float(o.q[2])
    m = np.stack([o.encode_coeffs(d, ps)[1] for d in D])
    for qp in (False, True):
        pt = g.he_pt_from_int_coeffs_qp(m, ps, 2) if qp else g.he_pt_from_int_coeffs(m, ps, 2)
        out = g.he_vec_mat_pt(ct, pt).words()[0]
        ref = (OC.vec_mat_lazy if qp else OC.vec_mat)(o, oct_, W, None, True)
        assert np.array_equal(out, ref.words)
    d = g.he_dot(ct, ct, 1)
    assert np.array_equal(d.words()[0], OC.dot(o, oct_, oct_, 1).words)


def test_replication_exhausted_and_level_exhausted(pair):
    from paper_2104_03152_b200 import HEError
    o, g = pair
    ct = g.he_encrypt(g.he_encode(np.ones(4), 2.0 ** 30, 2), 0)
    with pytest.raises(HEError) as e:      # 512 % 3 != 0 and output slot j + k reaches the span 510
        g.he_vec_mat_encode(np.ones((3, 511)), None, False, 0, 2, 2.0 ** 30)
    assert e.value.name == "REPLICATION_EXHAUSTED"
    low = g.he_mod_switch_to(ct, 0)
    for fn in (g.he_square, g.he_rescale, lambda c: g.he_power(c, 2)):
        with pytest.raises(HEError) as e:
            fn(low)
        assert e.value.name == "LEVEL_EXHAUSTED"


def test_mismatches_and_api_errors(pair):
    from paper_2104_03152_b200 import HEError
    o, g = pair
    a = g.he_encrypt(g.he_encode(np.ones((2, 4)), 2.0 ** 30, 2), 0)
    b = g.he_encrypt(g.he_encode(np.ones((3, 4)), 2.0 ** 30, 2), 0)
    with pytest.raises(HEError) as e:
        g.he_add(a, b)
    assert e.value.name == "SHAPE_MISMATCH"
    with pytest.raises(HEError) as e:
        g.he_keygen([1])
    assert e.value.name == "INVALID_ARGUMENT"
    with pytest.raises(HEError) as e:
        g.he_decode(g.he_decrypt(a), o.slots + 1)
    assert e.value.name == "TOO_MANY_VALUES"
    with pytest.raises(HEError) as e:
        g.he_dot(a, a, 16)                  # needs the key for step 8
    assert e.value.name == "MISSING_GALOIS_KEY"
    from paper_2104_03152_b200 import Context
    other = Context(P["logN"], P["bits"], P["K"], 99)
    with pytest.raises(HEError) as e:
        other.he_add(a, a)
    assert e.value.name == "PARAM_MISMATCH"
    with pytest.raises(HEError) as e:
        other.he_keygen([0])
    assert e.value.name == "INVALID_ROTATION"


def test_wide_ragged_batch_bit_exact(pair):
    """A batch of 37 ciphertexts (not a multiple of any block size): rotate, square and rescale
    word for word against the oracle for a sample of items (first, middle, last)."""
    o, g = pair
    rng = np.random.default_rng(2)
    B = 37
    zs = rng.uniform(-1, 1, (B, o.slots))
    pts = [o.encode(zs[b], 2.0 ** 30, 2) for b in range(B)]
    ct = g.he_encrypt(g.he_pt_import_words(np.stack([p.words for p in pts]), 2, 2.0 ** 30), 1000)
    r, sq = g.he_rotate(ct, 2).words(), g.he_square(ct).words()
    for b in (0, 18, 36):
        oc = o.encrypt(pts[b], 1000 + b)
        assert np.array_equal(r[b], o.rotate(oc, 2).words), b
        assert np.array_equal(sq[b], o.square(oc).words), b


# ---- the bench schedule's new entry points on a small context (both engines) --------------------
@pytest.mark.parametrize("bits", [(50, 40, 40, 50), (31, 26, 26, 31)], ids=["64bit", "32bit"])
def test_one_level_conv_small_ragged_bit_exact(bits):
    """he_im2col_conv_bsgs_pt on N = 2^11 (16 chunks of 64), C = 4 channels of 2x2 kernels, g = 4
    baby x 4 giant steps, a ragged batch of 3: word for word with oracle im2col_conv_bsgs, on the
    64-bit and the 32-bit engine; plus its layout / level / key errors."""
    from paper_2104_03152_b200 import Context, HEError
    chunk, g_ = 64, 4
    steps = sorted({chunk * b for b in range(1, g_)} | {chunk * g_ * a for a in range(1, 1024 // chunk // g_)})
    o = OracleContext(11, bits, 1, 5)
    o.keygen(steps)
    g = Context(11, bits, 1, 5)
    g.he_keygen(steps)
    rng = np.random.default_rng(7)
    k = rng.uniform(-1, 1, (4, 2, 2))
    bias = rng.uniform(-0.5, 0.5, 4)
    lvl = 2
    zs = np.zeros((3, o.slots))
    zs[:, : 4 * chunk] = rng.uniform(-1, 1, (3, 4 * chunk))
    o_in = [o.encrypt(o.encode(z, 2.0 ** 24, lvl), 40 + b) for b, z in enumerate(zs)]
    x = g.he_ct_import_words(np.stack([c.words for c in o_in]), lvl, 2.0 ** 24)
    ps = float(o.q[lvl]) * 2.0 ** -2
    Dv = OC.conv_bsgs_diagonals(k.reshape(4, -1), chunk, o.slots, g_)
    gD = g.he_pt_from_int_coeffs_qp(np.stack([o.encode_coeffs(v, ps)[1] for v in Dv]), ps, lvl)
    gB = g.he_pt_from_int_coeffs(np.stack([o.encode_coeffs(OC.conv_bias_slots(bias, chunk, o.slots),
                                                           2.0 ** 24 * ps / o.q[lvl])[1]]),
                                 2.0 ** 24 * ps / o.q[lvl], lvl - 1)
    y = g.he_im2col_conv_bsgs_pt(x, gD, gB, chunk, g_)
    for b in range(3):
        ref = OC.im2col_conv_bsgs(o, o_in[b], k.reshape(4, -1), bias, chunk, g_, -2)
        assert np.array_equal(y.words()[b], ref.words), b
        assert y.level == ref.level == lvl - 1 and y.scale == ref.scale
    # errors: C does not divide g; diagonals at another level; a missing giant-step key
    with pytest.raises(HEError) as e:
        g.he_im2col_conv_bsgs_encode(k, bias, chunk, 2, -2, lvl, 2.0 ** 24)
    assert e.value.name == "LAYOUT_MISMATCH"
    x1 = g.he_ct_import_words(np.stack([c.words[:, :2] for c in o_in]), 1, 2.0 ** 24)
    with pytest.raises(HEError) as e:
        g.he_im2col_conv_bsgs_pt(x1, gD, None, chunk, g_)
    assert e.value.name == "LEVEL_MISMATCH"
    g2 = Context(11, bits, 1, 5)
    g2.he_keygen(steps[:-1])
    x2 = g2.he_ct_import_words(np.stack([c.words for c in o_in]), lvl, 2.0 ** 24)
    gD2 = g2.he_pt_from_int_coeffs_qp(np.stack([o.encode_coeffs(v, ps)[1] for v in Dv]), ps, lvl)
    with pytest.raises(HEError) as e:
        g2.he_im2col_conv_bsgs_pt(x2, gD2, None, chunk, g_)
    assert e.value.name == "MISSING_GALOIS_KEY"


@pytest.mark.parametrize("bits", [(50, 40, 40, 50), (31, 26, 26, 31)], ids=["64bit", "32bit"])
def test_folded_vec_mat_small_ragged_bit_exact(bits):
    """he_vec_mat_bsgs_fold_pt (n 64 -> m 16, g 8: 2 groups + fold 4) on N = 2^11 with a ragged
    batch of 3: word for word with oracle vec_mat_bsgs_fold on both engines; the encode-side form
    (he_vec_mat_encode_bsgs_fold + he_vec_mat_pt) decrypts to x @ W; m not dividing n is rejected."""
    from paper_2104_03152_b200 import Context, HEError
    n, m, gg = 64, 16, 8
    steps = sorted(set(range(1, gg)) | {gg} | {m * t for t in range(1, n // m)})
    o = OracleContext(11, bits, 1, 9)
    o.keygen(steps)
    g = Context(11, bits, 1, 9)
    g.he_keygen(steps)
    rng = np.random.default_rng(11)
    W, bias = rng.normal(0, 0.2, (n, m)), rng.uniform(-0.5, 0.5, m)
    xs = rng.uniform(-1, 1, (3, n))
    lvl = 2
    o_in = [o.encrypt(o.encode(OC.replicate(x, o.slots), 2.0 ** 30, lvl), 60 + b) for b, x in enumerate(xs)]
    x = g.he_ct_import_words(np.stack([c.words for c in o_in]), lvl, 2.0 ** 30)
    ps = float(o.q[lvl])
    E = OC.bsgs_diagonals(OC.vecmat_diagonals(W, o.slots, True)[:m], gg).reshape(-1, o.slots)
    gD = g.he_pt_from_int_coeffs_qp(np.stack([o.encode_coeffs(v, ps)[1] for v in E]), ps, lvl)
    y = g.he_vec_mat_bsgs_fold_pt(x, gD, gg, n, m, None)
    for b in range(3):
        ref = OC.vec_mat_bsgs_fold(o, o_in[b], W, None, 0, g=gg)
        assert np.array_equal(y.words()[b], ref.words), b
    d, bp = g.he_vec_mat_encode(W, bias, True, 0, lvl, 2.0 ** 30, lazy=True, bsgs_g=gg, fold=True)
    z = g.he_decode(g.he_decrypt(g.he_vec_mat_pt(x, d, bp)), o.slots)
    # at scale 2^30 the key-switch noise of the 11 rotations is ~1e-5 per slot (~1e-3 at 2^24)
    for b in range(3):
        assert np.max(np.abs(z[b] - np.tile(xs[b] @ W + bias, o.slots // m))) < 1e-3
    with pytest.raises(HEError) as e:
        g.he_vec_mat_encode(W[:, :12], bias[:12], True, 0, lvl, 2.0 ** 30, lazy=True, bsgs_g=4, fold=True)
    assert e.value.name == "SHAPE_MISMATCH"


def test_symmetric_encryption_needs_the_secret_key():
    from paper_2104_03152_b200 import Context, HEError
    g = Context(10, (31, 26, 31), 1, 1)
    g.he_keygen([])
    pt = g.he_encode(np.ones((1, 4)), 2.0 ** 20, 1)
    ct = g.he_encrypt_symmetric(pt, 0, 99)
    assert np.max(np.abs(g.he_decode(g.he_decrypt(ct), 4) - 1.0)) < 1e-3
    g.he_drop_secret_key()
    with pytest.raises(HEError) as e:
        g.he_encrypt_symmetric(pt, 0, 99)
    assert e.value.name == "MISSING_KEY"

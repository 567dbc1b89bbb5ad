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

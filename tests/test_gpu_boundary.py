"""The rest of the §8(b) boundary through the Python binding: torch's caching allocator injected
with he_set_allocator, the _inplace forms against their out-of-place results word for word,
he_pt_to_int_coeffs against the oracle's integer encodings, he_make_public (copies of the keys,
no secret key)."""
import numpy as np
import pytest

from oracle.oracle import OracleContext
from synthetic import messages

pytestmark = pytest.mark.gpu

SMALLP = dict(logN=12, bits=(31, 26, 26, 26, 31), K=1, seed=5)


@pytest.fixture(scope="module")
def ctxs():
    from paper_2104_03152_b200 import Context
    o = OracleContext(SMALLP["logN"], SMALLP["bits"], SMALLP["K"], SMALLP["seed"])
    o.keygen([1, 2])
    g = Context(SMALLP["logN"], SMALLP["bits"], SMALLP["K"], SMALLP["seed"])
    g.he_keygen([1, 2])
    return o, g


def test_torch_allocator_inplace_forms_bit_exact(ctxs):
    import torch
    o, g = ctxs
    lvl = o.L - 1
    z = messages(3, o.slots, seed=9)
    m = np.stack([o.encode_coeffs(z[b], 2.0 ** 26)[1] for b in range(3)])
    before = torch.cuda.memory_allocated()
    g.he_set_allocator_torch()
    try:
        pt = g.he_pt_from_int_coeffs(m, 2.0 ** 26, lvl)
        assert torch.cuda.memory_allocated() > before      # the plaintext lives in torch's pool
        ct = g.he_encrypt(pt, 3)
        ref = [o.encrypt(o.coeffs_to_pt(m[b], lvl, 2.0 ** 26), 3 + b) for b in range(3)]
        assert all(np.array_equal(ct.words()[b], ref[b].words) for b in range(3))
        # in place == out of place, word for word (and == the oracle)
        a = g.he_add(ct, ct)
        g.he_add_inplace(ct, ct)
        assert np.array_equal(a.words(), ct.words())
        r = g.he_rotate(ct, 1)
        g.he_rotate_inplace(ct, 1)
        assert np.array_equal(r.words(), ct.words())
        for b in range(3):
            assert np.array_equal(ct.words()[b], o.rotate(o.add(ref[b], ref[b]), 1).words)
        s = g.he_square(ct)
        g.he_square_inplace(ct)
        assert np.array_equal(s.words(), ct.words()) and ct.level == lvl - 1
        p2 = g.he_encode(np.full(o.slots, 0.5), ct.scale, ct.level)
        x = g.he_add_plain(ct, p2)
        g.he_add_plain_inplace(ct, p2)
        assert np.array_equal(x.words(), ct.words())
        x = g.he_mul_plain(ct, p2)
        g.he_mul_plain_inplace(ct, p2)
        assert np.array_equal(x.words(), ct.words()) and x.scale == ct.scale
        x = g.he_rescale(ct)
        g.he_rescale_inplace(ct)
        assert np.array_equal(x.words(), ct.words()) and ct.level == lvl - 2
        del a, r, s, x, ct, pt, p2
        g.he_sync()
    finally:
        g.he_set_allocator()


def test_pt_to_int_coeffs_matches_oracle_encoding(ctxs):
    o, g = ctxs
    z = messages(2, o.slots, seed=4)
    for lvl in (0, o.L - 1):
        m = np.stack([o.encode_coeffs(z[b], 2.0 ** 26)[1] for b in range(2)])
        pt = g.he_pt_from_int_coeffs(m, 2.0 ** 26, lvl)
        assert np.array_equal(g.he_pt_to_int_coeffs(pt), m)
    # a device encoding decodes to its own integers: from_int(to_int(pt)) reproduces the words
    pt = g.he_encode(z, 2.0 ** 26, o.L - 1)
    assert np.array_equal(g.he_pt_from_int_coeffs(g.he_pt_to_int_coeffs(pt), 2.0 ** 26, o.L - 1).words(), pt.words())


def test_make_public_copies_keys_without_secret(ctxs):
    from paper_2104_03152_b200 import HEError
    o, g = ctxs
    pub = g.he_make_public()
    for kind, step in ((1, 0), (2, 0), (3, 1), (3, 2)):
        assert np.array_equal(pub.he_key_export(kind, step), g.he_key_export(kind, step))
    z = messages(1, o.slots, seed=2)
    ct = pub.he_encrypt(pub.he_encode(z, 2.0 ** 26, o.L - 1), 0)
    ct2 = g.he_encrypt(g.he_encode(z, 2.0 ** 26, o.L - 1), 0)
    assert np.array_equal(ct.words(), ct2.words())          # same seed, same public key
    r = pub.he_rotate(ct, 2)
    with pytest.raises(HEError) as e:
        pub.he_decrypt(r)
    assert e.value.name == "MISSING_KEY"
    back = g.he_ct_import_words(r.words(), r.level, r.scale)
    assert np.max(np.abs(g.he_decode(g.he_decrypt(back), o.slots)[0] - np.roll(z[0], -2))) < 1e-3

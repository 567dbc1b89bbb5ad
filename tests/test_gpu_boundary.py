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


def test_small_prime_keys_rest_as_u32_and_materialise_on_demand():
    """Keys at rest: a small-prime context holds pk (u64) + relin + Galois keys as u32
    Montgomery words only; the fused rotate / square leave it so; he_key_export builds the u64 words
    of the key asked for (equal to the oracle's), and the per-rotation vec_mat (u64 keys) still
    gives the oracle's words after materialising its own."""
    from oracle import circuits as OC
    from paper_2104_03152_b200 import Context
    logN, bits, K, seed = 11, (31, 26, 26, 31), 1, 21
    steps = [1, 2, 3]
    o = OracleContext(logN, bits, K, seed)
    o.keygen(steps)
    g = Context(logN, bits, K, seed)
    g.he_keygen(steps)
    N, L, NP = 1 << logN, len(bits) - K, len(bits)
    kw = L * 2 * NP * N
    at_rest = 2 * L * N * 8 + (1 + len(steps)) * kw * 4
    assert g.he_key_bytes() == at_rest
    lvl = o.L - 1
    z = messages(2, o.slots, seed=4)
    m = np.stack([o.encode_coeffs(z[b], 2.0 ** 26)[1] for b in range(2)])
    ct = g.he_encrypt(g.he_pt_from_int_coeffs(m, 2.0 ** 26, lvl), 7)
    ref = [o.encrypt(o.coeffs_to_pt(m[b], lvl, 2.0 ** 26), 7 + b) for b in range(2)]
    r = g.he_rotate(ct, 2)
    s = g.he_square(ct)
    for b in range(2):
        assert np.array_equal(r.words()[b], o.rotate(ref[b], 2).words)
        assert np.array_equal(s.words()[b], o.square(ref[b]).words)
    assert g.he_key_bytes() == at_rest                    # the fused paths never build u64 keys
    assert np.array_equal(g.he_key_export(3, 2), o.galois_key(2))
    assert g.he_key_bytes() == at_rest + kw * 8
    assert np.array_equal(g.he_key_export(2), o.relin_key())
    assert g.he_key_bytes() == at_rest + 2 * kw * 8
    assert np.array_equal(g.he_key_export(3, 2), o.galois_key(2))   # cached, not rebuilt
    assert g.he_key_bytes() == at_rest + 2 * kw * 8
    # per-rotation vec_mat (the paper's form, u64 keys): 4 diagonals -> steps 1..3 materialised
    rng = np.random.default_rng(1)
    W = rng.normal(0, 0.1, (4, 4))
    x = OC.replicate(rng.uniform(-1, 1, 4), o.slots)
    mx = o.encode_coeffs(x, 2.0 ** 26)[1]
    ocx = o.encrypt(o.coeffs_to_pt(mx, lvl, 2.0 ** 26), 3)
    gcx = g.he_encrypt(g.he_pt_from_int_coeffs(mx, 2.0 ** 26, lvl), 3)
    D = OC.vecmat_diagonals(W, o.slots, True)
    ps = float(o.q[lvl])
    dm = np.stack([o.encode_coeffs(d, ps)[1] for d in D])
    vm = g.he_vec_mat_pt(gcx, g.he_pt_from_int_coeffs(dm, ps, lvl))
    assert np.array_equal(vm.words()[0], OC.vec_mat(o, ocx, W, None, True).words)
    assert g.he_key_bytes() == at_rest + 4 * kw * 8


def test_large_host_inputs_uploaded_on_the_copy_stream_give_the_same_words():
    """he_encode / he_encode_encrypt with host inputs >= 1 MiB go through the context's copy stream
    and its two upload buffers (include/he_ckks.h): back-to-back calls without a sync in between
    (buffers 0, 1, 0, 1, then a larger batch that regrows buffer 0) give, word for word, what the
    device-input forms give, on pageable and on pinned memory."""
    import torch
    from paper_2104_03152_b200 import Context
    g = Context(12, (31, 26, 26, 31), 1, 9)
    g.he_keygen([1])
    lvl, ns = g.L - 1, g.slots
    B = 80                                                # 80 x 2048 x 8 B = 1.25 MiB
    zs = [messages(B, ns, seed=30 + i) for i in range(4)] + [messages(2 * B, ns, seed=40)]
    pinned = [torch.from_numpy(z).pin_memory() for z in zs]
    for hosts in (zs, [p.numpy() for p in pinned]):
        cts = [g.he_encode_encrypt(z, 2.0 ** 26, lvl, 100 * i) for i, z in enumerate(hosts)]
        pts = [g.he_encode(z, 2.0 ** 26, lvl) for z in hosts]
        g.he_sync()
        for i, z in enumerate(zs):
            zd = torch.from_numpy(z).cuda()
            assert np.array_equal(cts[i].words(), g.he_encode_encrypt(zd, 2.0 ** 26, lvl, 100 * i).words()), i
            assert np.array_equal(pts[i].words(), g.he_encode(zd, 2.0 ** 26, lvl).words()), i

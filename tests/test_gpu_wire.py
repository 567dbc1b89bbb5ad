"""Wire format: the device packer's bytes equal the reference
packer's (oracle/wire.py, plain Python from the format definition), deserialize o serialize is the
identity, corrupt or foreign payloads are rejected, and the paper network's communication per
inference (encrypted input + encrypted output, BASELINE config 4) is measured."""
import numpy as np
import pytest

from oracle import wire
from oracle.oracle import OracleContext
from synthetic import CFG4, cnn_weights, mnist_like_images

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("logN,bits,K,level,size,B", [(10, (50, 40, 40, 50, 50), 2, 2, 2, 3),
                                                      (13, (31, 26, 26, 26, 26, 26, 26, 31), 1, 6, 2, 1),
                                                      (13, (31, 26, 26, 26, 26, 26, 26, 31), 1, 0, 3, 2),
                                                      (14, (60, 40, 40, 60), 1, 1, 2, 1)])
def test_wire_bytes_equal_reference_and_roundtrip(logN, bits, K, level, size, B):
    from paper_2104_03152_b200 import Context
    o = OracleContext(logN, bits, K, 0)
    g = Context(logN, bits, K, 0)
    rng = np.random.default_rng(logN + level)
    w = np.stack([np.stack([np.stack([rng.integers(0, o.q[i], o.N, dtype=np.uint64) for i in range(level + 1)])
                            for _ in range(size)]) for _ in range(B)])
    w[0, 0, 0, :3] = 0
    w[-1, -1, -1, -3:] = np.uint64(o.q[level] - 1)
    ct = g.he_ct_import_words(w, level, 3.5, size=size)
    blob = g.he_ct_serialize(ct)
    ref = wire.pack(w, o.q, level, 3.5)
    assert blob == ref
    assert len(blob) == wire.HEADER_BYTES + wire.payload_bytes(o.N, B, size, wire.limb_widths(o.q, level))
    back = g.he_ct_deserialize(blob)
    assert np.array_equal(back.words(), w) and back.level == level and back.scale == 3.5 and back.size == size


def test_wire_rejects_corrupt_and_foreign():
    from paper_2104_03152_b200 import Context, HEError
    g = Context(11, (31, 26, 26, 31), 1, 0)
    o = OracleContext(11, (31, 26, 26, 31), 1, 0)
    w = np.stack([np.stack([np.full(o.N, o.q[i] - 1, dtype=np.uint64) for i in range(3)]) for _ in range(2)])[None]
    blob = bytearray(g.he_ct_serialize(g.he_ct_import_words(w, 2, 1.0)))
    bad = bytearray(blob)
    bad[64] = 0xFF   # first residue of limb 0 becomes >= q0 (all-ones bits)
    bad[65] = 0xFF
    bad[66] = 0xFF
    bad[67] = 0xFF
    with pytest.raises(HEError):
        g.he_ct_deserialize(bytes(bad))
    with pytest.raises(HEError):
        g.he_ct_deserialize(bytes(blob[:-8]))
    other = Context(12, (31, 26, 26, 31), 1, 0)
    with pytest.raises(HEError) as e:
        other.he_ct_deserialize(bytes(blob))
    assert e.value.name == "PARAM_MISMATCH"


def test_cnn_communication_per_inference():
    """Encrypted input (level 6: 31 + 6 x 26 bits per coefficient pair) + encrypted logits
    (level 0: 31 bits): 382,976 + 63,488 payload bytes; the paper reports 427 KB
    with SEAL's own serialisation of its parameters."""
    from paper_2104_03152_b200 import Context
    from paper_2104_03152_b200.cnn import EncryptedCNN, rotation_steps
    g = Context(CFG4.logN, CFG4.bits, CFG4.n_special, CFG4.seed)
    g.he_keygen(rotation_steps())
    net = EncryptedCNN(g, cnn_weights(3))
    img = mnist_like_images(1, 4)
    ct_in = net.encrypt(img, 0)
    up = g.he_ct_serialize(ct_in)
    ct_out = net.forward(g.he_ct_deserialize(up))
    down = g.he_ct_serialize(ct_out)
    assert len(up) == 64 + 2 * 8192 * (31 + 6 * 26) // 8 == 64 + 382976
    assert len(down) == 64 + 2 * 8192 * 31 // 8 == 64 + 63488
    assert len(up) + len(down) < 500_000   # "less than half a megabyte"
    # the decrypted logits survive the round trip unchanged
    z = net.decrypt(g.he_ct_deserialize(down))
    assert np.array_equal(z, net.decrypt(ct_out))


def test_symmetric_encrypt_bit_exact_and_seeded_wire():
    """he_encrypt_symmetric == oracle encrypt_symmetric word for word (item b on stream id + b); the
    seeded wire bytes == oracle/wire.pack_seeded (c0 only: half the full payload); deserializing them
    regenerates c1 on the device (same words); non-fresh ciphertexts have no seeded form."""
    from paper_2104_03152_b200 import Context, HEError
    o = OracleContext(CFG4.logN, CFG4.bits, CFG4.n_special, 5)
    o.keygen([])
    g = Context(CFG4.logN, CFG4.bits, CFG4.n_special, 5)
    g.he_keygen([])
    level, B = 5, 3
    zs = np.random.default_rng(8).uniform(-1, 1, (B, o.slots))
    pts = [o.encode(z, 2.0 ** 30, level) for z in zs]
    gct = g.he_encrypt_symmetric(g.he_pt_import_words(np.stack([p.words for p in pts]), level, 2.0 ** 30),
                                 100, 777)
    ref = [o.encrypt_symmetric(p, 100 + b, 777) for b, p in enumerate(pts)]
    W = gct.words()
    for b in range(B):
        assert np.array_equal(W[b], ref[b].words), b
    blob = g.he_ct_serialize_seeded(gct)
    assert blob == wire.pack_seeded(np.stack([r.words[0] for r in ref]), o.q, level, 2.0 ** 30, 777, 100)
    full = g.he_ct_serialize(gct)
    assert len(blob) - 64 == (len(full) - 64) // 2
    back = g.he_ct_deserialize(blob)
    assert np.array_equal(back.words(), W) and back.level == level and back.scale == 2.0 ** 30
    assert np.max(np.abs(g.he_decode(g.he_decrypt(back), o.slots) - zs)) < 1e-4
    with pytest.raises(HEError):
        g.he_ct_serialize_seeded(g.he_add(gct, gct))
    with pytest.raises(HEError):
        g.he_ct_serialize_seeded(g.he_ct_deserialize(full))


def test_cnn_communication_seeded_input():
    """The bench schedule (input at level 5) with a seeded symmetric upload: 8192 x (31 + 5 x 26)
    bits up, 8192 x 31 bits x 2 down; the logits equal those of the public-key path's decryption."""
    from paper_2104_03152_b200 import Context
    from paper_2104_03152_b200.cnn import CONV_G, FC1_G, EncryptedCNN, rotation_steps
    g = Context(CFG4.logN, CFG4.bits, CFG4.n_special, CFG4.seed)
    g.he_keygen(rotation_steps(conv_g=CONV_G, fc_bsgs=True, fc1_g=FC1_G))
    net = EncryptedCNN(g, cnn_weights(3), conv_g=CONV_G, fc1_g=FC1_G)
    img = mnist_like_images(1, 4)
    pt = g.he_encode(net.im2col(img), 2.0 ** net.plan["in_log2"], net.top)
    up = g.he_ct_serialize_seeded(g.he_encrypt_symmetric(pt, 0, 31337))
    down = g.he_ct_serialize(net.forward(g.he_ct_deserialize(up)))
    assert len(up) == 64 + 8192 * (31 + 5 * 26) // 8 == 64 + 164864
    assert len(down) == 64 + 2 * 8192 * 31 // 8 == 64 + 63488
    z = net.decrypt(g.he_ct_deserialize(down))
    ref = net.decrypt(net.forward(net.encrypt(img, 0)))
    assert np.max(np.abs(z - ref)) < 2e-3 and np.argmax(z) == np.argmax(ref)

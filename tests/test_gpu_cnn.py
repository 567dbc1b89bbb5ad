"""GPU parity of the paper's encrypted CNN (BASELINE config 4) through
the C-ABI: im2col conv, square, FC1 (replicated-output diagonals), square, FC2.

* bit-exact: the GPU chain, fed the oracle's input ciphertext and the oracle's
  integer encodings of every weight plaintext (C7 injection), reproduces the
  oracle's ciphertext words after every layer;
* tolerance: the all-GPU path (its own encode / encrypt / decrypt / decode) gives
  logits within 5e-3 of the float64 network with the same argmax (north_star).
"""
import numpy as np
import pytest

from oracle import circuits as OC
from oracle.oracle import OracleContext
from synthetic import CFG4, cnn_weights, mnist_like_images
from test_layouts import float_net_numpy

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg4():
    from paper_2104_03152_b200 import Context
    from paper_2104_03152_b200.cnn import rotation_steps
    forms = [dict(), dict(fold_n1=8), dict(conv_g=8, fc_bsgs=True), dict(fc_bsgs=True),
             dict(conv_g=8, fc_bsgs=True, fc1_g=32)]
    for f in forms:
        assert OC.cnn_rotation_steps(**f) == rotation_steps(**f)
    steps = sorted(set().union(*[rotation_steps(**f) for f in forms]))   # every conv / FC form
    o = OracleContext(CFG4.logN, CFG4.bits, CFG4.n_special, CFG4.seed)
    o.keygen(steps)
    g = Context(CFG4.logN, CFG4.bits, CFG4.n_special, CFG4.seed)
    g.he_keygen(steps)
    return o, g


def inj(g, o, vecs, scale, level):
    ms = np.stack([o.encode_coeffs(v, scale)[1] for v in vecs])
    return g.he_pt_from_int_coeffs(ms, scale, level)


@pytest.mark.parametrize("lazy", [False, True, "bsgs", "bsgs+fold", "bsgs+conv8", "fast"])
def test_cnn_layers_bit_exact(cfg4, lazy):
    """lazy=False: FC layers with one ModDown per rotation (oracle vec_mat); lazy=True: one
    ModDown per vec_mat (oracle vec_mat_lazy, QP diagonals); "bsgs": baby step n/4 with one lazy
    ModDown per giant step (oracle vec_mat_bsgs)."""
    _layers_bit_exact(*cfg4, lazy, 2)


@pytest.fixture(scope="module")
def cfg4_capped(cfg4):
    """A second GPU context whose persistent pipelined NTT (k_ntt32_pipe) runs on at most 8 CTAs
    (HE_PIPE_GRID_CAP), so every CTA loops over several blocks and the staged-prefetch path
    (cp.async of block k+1's row while block k computes) runs for every pipelined job type
    (ModUp32, KsSpecial, KsData, RescaleData) even at a small batch."""
    import os
    from paper_2104_03152_b200 import Context
    from paper_2104_03152_b200.cnn import rotation_steps
    o, _ = cfg4
    os.environ["HE_PIPE_GRID_CAP"] = "8"
    try:
        g = Context(CFG4.logN, CFG4.bits, CFG4.n_special, CFG4.seed)
    finally:
        del os.environ["HE_PIPE_GRID_CAP"]
    g.he_keygen(sorted(set(rotation_steps(conv_g=8, fc_bsgs=True, fc1_g=32)) | set(rotation_steps())
                       | set(rotation_steps(conv_g=8, fc_bsgs=True))))
    return o, g


@pytest.mark.parametrize("lazy", ["fast", "bsgs+conv8", False])
def test_cnn_layers_bit_exact_multiblock_pipe(cfg4_capped, lazy):
    """The bench schedule (and two others) word for word after every layer, with the pipelined
    NTT forced into its multi-block loop (that loop only ran when nblk > grid)."""
    _layers_bit_exact(*cfg4_capped, lazy, 3)


def _layers_bit_exact(o, g, lazy, nimg):
    w = cnn_weights(3)
    imgs = mnist_like_images(nimg, 4)
    conv_g = 8 if lazy in ("bsgs+conv8", "fast") else 0
    fc1_g = 32 if lazy == "fast" else 0      # the bench's schedule: one-level conv + folded FC1
    ns, q, plan = o.slots, o.q, (OC.CNN_PLAN_BSGS if conv_g else OC.CNN_PLAN)
    o_in = [OC.cnn_encrypt_input(o, img, b, plan) for b, img in enumerate(imgs)]
    lvl = o_in[0].level
    x = g.he_ct_import_words(np.stack([c.words for c in o_in]), lvl, o_in[0].scale)
    # conv (C18/C19)
    if conv_g:      # one-level conv: g QP diagonals, one rescale, giant-step rotation sum
        ps = float(q[lvl]) * 2.0 ** plan["conv_shift"]
        Dv = OC.conv_bsgs_diagonals(w.conv_w.reshape(4, -1), 64, ns, conv_g)
        gD = g.he_pt_from_int_coeffs_qp(np.stack([o.encode_coeffs(v, ps)[1] for v in Dv]), ps, lvl)
        gB = inj(g, o, [OC.conv_bias_slots(w.conv_b, 64, ns)], o_in[0].scale * ps / q[lvl], lvl - 1)
        x = g.he_im2col_conv_bsgs_pt(x, gD, gB, 64, conv_g)
        ref = [OC.im2col_conv_bsgs(o, c, w.conv_w.reshape(4, -1), w.conv_b, 64, conv_g, plan["conv_shift"])
               for c in o_in]
        lazy = "bsgs"
    else:
        K = [OC.conv_kernel_slots(w.conv_w[c].reshape(-1), 64, ns) for c in range(4)]
        M = [OC.conv_mask_slots(c, 4, 64, ns) for c in range(4)]
        gK = inj(g, o, K, float(q[lvl]) * 2.0 ** plan["conv_shift"], lvl)
        gM = inj(g, o, M, float(q[lvl - 1]) * 2.0 ** plan["mask_shift"], lvl - 1)
        s2 = (o_in[0].scale * gK.scale / q[lvl]) * gM.scale / q[lvl - 1]
        gB = inj(g, o, [OC.conv_bias_slots(w.conv_b, 64, ns)], s2, lvl - 2)
        n1 = 8 if lazy == "bsgs+fold" else 0
        if n1:
            x = g.he_im2col_conv_hoisted_pt(x, gK, gM, gB, 64, n1)
            lazy = "bsgs"
        else:
            x = g.he_im2col_conv_pt(x, gK, gM, gB, 64)
        ref = [OC.im2col_conv(o, c, w.conv_w.reshape(4, -1), w.conv_b, 64, plan["conv_shift"],
                              plan["mask_shift"], fold_n1=n1) for c in o_in]
    W = x.words()
    for b in range(nimg):
        assert np.array_equal(W[b], ref[b].words), ("conv", b)
    assert x.scale == ref[0].scale and x.level == ref[0].level
    # square
    x = g.he_square(x)
    ref = [o.square(c) for c in ref]
    W = x.words()
    for b in range(nimg):
        assert np.array_equal(W[b], ref[b].words), ("square1", b)
    # FC1 (replicated output) and FC2
    for name, Wm, bias, rep, shift in [("fc1", w.fc1_w.T, w.fc1_b, True, -plan["fc1_shift"]),
                                       ("fc2", w.fc2_w.T, w.fc2_b, False, -plan["fc2_shift"])]:
        lvl = ref[0].level
        ps = float(q[lvl]) * 2.0 ** (-shift)
        Dv = OC.vecmat_diagonals(Wm, ns, rep)
        bs = ref[0].scale * ps / q[lvl]
        gb = inj(g, o, [OC.vecmat_bias_slots(bias, ns, rep)], bs, lvl - 1)
        if fc1_g:           # folded FC layers (FC2 padded to 16 outputs)
            if name == "fc2":
                Wm, bias = OC.pad_columns(Wm, bias, OC.FC2_M)
                Dv = OC.vecmat_diagonals(Wm, ns, True)
                gb = inj(g, o, [OC.vecmat_bias_slots(bias, ns, True)], bs, lvl - 1)
            n_, m_ = Wm.shape
            gg = fc1_g if name == "fc1" else OC.FC2_M
            E = OC.bsgs_diagonals(Dv[:m_], gg).reshape(-1, ns)
            gD = g.he_pt_from_int_coeffs_qp(np.stack([o.encode_coeffs(v, ps)[1] for v in E]), ps, lvl)
            x = g.he_vec_mat_bsgs_fold_pt(x, gD, gg, n_, m_, gb)
            ref = [OC.vec_mat_bsgs_fold(o, c, Wm, bias, shift, g=gg) for c in ref]
        elif lazy == "bsgs":
            gg = Wm.shape[0] // 4
            E = OC.bsgs_diagonals(Dv, gg).reshape(-1, ns)
            gD = g.he_pt_from_int_coeffs_qp(np.stack([o.encode_coeffs(v, ps)[1] for v in E]), ps, lvl)
            x = g.he_vec_mat_bsgs_pt(x, gD, gg, gb)
            ref = [OC.vec_mat_bsgs(o, c, Wm, bias, rep, shift, g=gg) for c in ref]
        else:
            if lazy:
                gD = g.he_pt_from_int_coeffs_qp(np.stack([o.encode_coeffs(v, ps)[1] for v in Dv]), ps, lvl)
            else:
                gD = inj(g, o, Dv, ps, lvl)
            x = g.he_vec_mat_pt(x, gD, gb)
            vm = OC.vec_mat_lazy if lazy else OC.vec_mat
            ref = [vm(o, c, Wm, bias, rep, shift) for c in ref]
        W = x.words()
        for b in range(nimg):
            assert np.array_equal(W[b], ref[b].words), (name, b)
        if name == "fc1":
            x = g.he_square(x)
            ref = [o.square(c) for c in ref]
    assert x.level == 0
    # decrypt + decode of the bit-exact result vs the oracle's
    z = g.he_decode(g.he_decrypt(x), 10)
    for b in range(nimg):
        assert np.allclose(z[b], o.decode(o.decrypt(ref[b]), 10), rtol=1e-9, atol=1e-9)


@pytest.mark.parametrize("lazy", [False, True, "bsgs", "bsgs+fold", "bsgs+conv8", "fast"])
def test_cnn_all_gpu_tolerance(cfg4, lazy):
    """Own encode/encrypt/decrypt/decode: logits within 5e-3 abs of float64, argmax equal."""
    from paper_2104_03152_b200.cnn import EncryptedCNN
    o, g = cfg4
    w = cnn_weights(3)
    net = EncryptedCNN(g, w, lazy=bool(lazy), bsgs=lazy in ("bsgs", "bsgs+fold", "bsgs+conv8", "fast"),
                       fold_n1=8 if lazy == "bsgs+fold" else 0, conv_g=8 if lazy in ("bsgs+conv8", "fast") else 0,
                       fc1_g=32 if lazy == "fast" else 0)
    imgs = mnist_like_images(16, 4)
    logits = net.decrypt(net.forward(net.encrypt(imgs, 1000)))
    for b, img in enumerate(imgs):
        ref = float_net_numpy(img, w)
        assert np.max(np.abs(logits[b] - ref)) < 5e-3, b
        assert np.argmax(logits[b]) == np.argmax(ref)


def test_cnn_batch_independence(cfg4):
    """Items of a batch are independent: image b of a batch of 5 equals the same image alone."""
    from paper_2104_03152_b200.cnn import EncryptedCNN
    o, g = cfg4
    net = EncryptedCNN(g, cnn_weights(3))
    imgs = mnist_like_images(5, 4, start=100)
    big = net.forward(net.encrypt(imgs, 7)).words()
    one = net.forward(net.encrypt(imgs[3:4], 10)).words()
    assert np.array_equal(big[3], one[0])

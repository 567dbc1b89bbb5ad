"""P11/P12: pin the circuit layouts (C17-C19) with a float64 slot simulator
(rotation = np.roll, exact products) against numpy matmul, a direct sliding-window
convolution and torch.nn.functional.conv2d; then pin the oracle's encrypted CNN
against two independent float networks (numpy and torch CPU)."""
import numpy as np
import pytest
import torch

from oracle import circuits as C
from synthetic import CFG4, cnn_weights, mnist_like_images, vecmat_inputs

NS = 4096


def mock_vec_mat(x, W, replicate_out):
    D = C.vecmat_diagonals(W, NS, replicate_out)
    return sum(np.roll(x, -k) * D[k] for k in range(W.shape[0]))


def mock_conv(slots, kernels, bias, chunk):
    n_ch = kernels.shape[0]
    acc = np.zeros(NS)
    for c in range(n_ch):
        t = slots * C.conv_kernel_slots(kernels[c], chunk, NS)
        for step in C.conv_fold_steps(chunk, NS):
            t = t + np.roll(t, -step)
        acc += t * C.conv_mask_slots(c, n_ch, chunk, NS)
    return acc + C.conv_bias_slots(bias, chunk, NS)


def test_vecmat_layout_cfg1():
    x, W = vecmat_inputs(0)
    y = mock_vec_mat(C.replicate(x, NS), W, False)
    assert np.allclose(y[:10], x @ W, atol=1e-12) and np.all(y[10:] == 0)


def test_vecmat_layout_replicated_output():
    rng = np.random.default_rng(0)
    x, W = rng.normal(size=256), rng.normal(size=(256, 64))
    y = mock_vec_mat(C.replicate(x, NS), W, True)
    assert np.allclose(y, np.tile(x @ W, NS // 64), atol=1e-11)


def test_vecmat_non_power_of_two_and_exhaustion():
    """S:422 n=10, m=7 (PAPER.md:61 non-power-of-two support) and S:418 exhaustion."""
    rng = np.random.default_rng(1)
    x, W = rng.normal(size=10), rng.normal(size=(10, 7))
    y = mock_vec_mat(C.replicate(x, NS), W, False)
    assert np.allclose(y[:7], x @ W, atol=1e-12)
    with pytest.raises(C.ReplicationExhausted):
        C.vecmat_diagonals(rng.normal(size=(3000, 2000)), NS, False)
    with pytest.raises(ValueError):
        C.vecmat_diagonals(rng.normal(size=(10, 7)), NS, True)


def test_im2col_spec_example():
    """3x3 image, 2x2 kernel, stride 1 -> windows [[1,2,4,5],[2,3,5,6],[4,5,7,8],[5,6,8,9]]."""
    img = np.arange(1, 10, dtype=float).reshape(3, 3)
    s = C.im2col_slots(img, 2, 2, 1, 16)
    windows = s.reshape(4, 4).T    # slot = tap * chunk + window; chunk = 4
    assert windows.tolist() == [[1, 2, 4, 5], [2, 3, 5, 6], [4, 5, 7, 8], [5, 6, 8, 9]]


def _direct_conv(img, w, b):
    out = np.zeros((w.shape[0], 8, 8))
    for c in range(w.shape[0]):
        for r in range(8):
            for s in range(8):
                out[c, r, s] = np.sum(w[c, 0] * img[3 * r:3 * r + 7, 3 * s:3 * s + 7]) + b[c]
    return out


def test_conv_layout_vs_direct_and_torch():
    w = cnn_weights(3)
    img = mnist_like_images(1, 4)[0]
    slots = C.im2col_slots(img, 7, 7, 3, NS)
    assert np.all(slots[49 * 64:] == 0)
    y = mock_conv(slots, w.conv_w.reshape(4, 49), w.conv_b, 64)
    direct = _direct_conv(img, w.conv_w, w.conv_b).reshape(-1)
    ref = torch.nn.functional.conv2d(torch.tensor(img)[None, None], torch.tensor(w.conv_w),
                                     torch.tensor(w.conv_b), stride=3).numpy().reshape(-1)
    assert np.allclose(direct, ref, atol=1e-12)
    # C19: the 256-vector (PyTorch flatten order) replicated x16 with period 256
    assert np.allclose(y, np.tile(ref, 16), atol=1e-12)
    assert len(C.conv_fold_steps(64, NS)) == 6    # PAPER.md:64 "log2(N) rotations", N = 64 rows


def float_net_numpy(img, w):
    x = _direct_conv(img, w.conv_w, w.conv_b).reshape(-1) ** 2
    x = (w.fc1_w @ x + w.fc1_b) ** 2
    return w.fc2_w @ x + w.fc2_b


def float_net_torch(img, w):
    t = lambda a: torch.tensor(a, dtype=torch.float64)
    x = torch.nn.functional.conv2d(t(img)[None, None], t(w.conv_w), t(w.conv_b), stride=3)
    x = x.flatten() ** 2
    x = torch.nn.functional.linear(x, t(w.fc1_w), t(w.fc1_b)) ** 2
    return torch.nn.functional.linear(x, t(w.fc2_w), t(w.fc2_b)).numpy()


def test_cnn_float_networks_and_mock_circuit_agree():
    w = cnn_weights(3)
    for img in mnist_like_images(3, 4):
        a, b = float_net_numpy(img, w), float_net_torch(img, w)
        assert np.allclose(a, b, atol=1e-9)
        x = mock_conv(C.im2col_slots(img, 7, 7, 3, NS), w.conv_w.reshape(4, 49), w.conv_b, 64) ** 2
        x = mock_vec_mat(x, w.fc1_w.T, True) + C.vecmat_bias_slots(w.fc1_b, NS, True)
        x = x ** 2
        x = mock_vec_mat(x, w.fc2_w.T, False) + C.vecmat_bias_slots(w.fc2_b, NS, False)
        assert np.allclose(x[:10], a, atol=1e-9)


def test_cnn_headroom_R1():
    """R1: the last level represents |logit| < q0 / (2 * final scale); the plan's FC2 shift must
    leave >= 2x headroom over the float network's logits on the seeded images."""
    w = cnn_weights(3)
    worst = max(np.abs(float_net_numpy(img, w)).max() for img in mnist_like_images(64, 4))
    final_scale = 2.0 ** (26 + C.CNN_PLAN["fc2_shift"]) * 1.02
    assert 2 * worst < 0x7ffe0001 / (2 * final_scale)


@pytest.mark.slow
def test_oracle_cnn_end_to_end():
    """P12: the oracle's decrypted logits vs the float network, 5e-3 abs and argmax (north_star)."""
    from oracle.oracle import OracleContext
    w = cnn_weights(3)
    img = mnist_like_images(1, 4)[0]
    ctx = OracleContext(CFG4.logN, CFG4.bits, CFG4.n_special, CFG4.seed)
    ctx.keygen(C.cnn_rotation_steps())
    out = C.cnn_forward(ctx, C.cnn_encrypt_input(ctx, img, 0), w)
    assert out.level == 0
    z = ctx.decode(ctx.decrypt(out), 10)
    ref = float_net_numpy(img, w)
    assert np.max(np.abs(z - ref)) < 5e-3
    assert np.argmax(z) == np.argmax(ref)


def test_hoisted_fold_is_the_same_sum():
    """The hoisted two-level fold sums rot(t, chunk m) over all m exactly like the log2 rotate-and-add
    fold (slot simulator): 8 x 8 = 64 chunks."""
    rng = np.random.default_rng(0)
    t = rng.normal(size=NS)
    ref = t.copy()
    for step in C.conv_fold_steps(64, NS):
        ref = ref + np.roll(ref, -step)
    u = sum(np.roll(t, -64 * b) for b in range(8))
    s = sum(np.roll(u, -512 * a) for a in range(8))
    assert np.allclose(s, ref, atol=1e-9)


def mock_conv_bsgs(slots, kernels, bias, chunk, g):
    """The one-level conv: v = sum_{b<g} D_b * rot(x, chunk b), then
    sum_{a<n2} rot(v, chunk g a) + bias (slot simulator, rot = np.roll(., -k))."""
    D = C.conv_bsgs_diagonals(kernels, chunk, NS, g)
    v = sum(D[b] * np.roll(slots, -chunk * b) for b in range(g))
    n2 = NS // chunk // g
    return sum(np.roll(v, -chunk * g * a) for a in range(n2)) + C.conv_bias_slots(bias, chunk, NS)


@pytest.mark.parametrize("g", [4, 8, 16, 64])
def test_one_level_conv_is_the_same_conv(g):
    """D_b = sum_c Mask_c * rot(K_c, chunk b) and Mask_c has period C chunks, so the baby-step /
    giant-step form equals the paper's fold-then-mask conv (mock_conv, itself pinned against
    torch conv2d above) whenever C | g; with g = 2 (C does not divide g) it does not."""
    w = cnn_weights(3)
    img = mnist_like_images(1, 4, start=2)[0]
    slots = C.im2col_slots(img, 7, 7, 3, NS)
    k = w.conv_w.reshape(4, -1)
    ref = mock_conv(slots, k, w.conv_b, 64)
    assert np.allclose(mock_conv_bsgs(slots, k, w.conv_b, 64, g), ref, atol=1e-9)
    assert not np.allclose(mock_conv_bsgs(slots, k, w.conv_b, 64, 2), ref, atol=1e-3)


def test_one_level_conv_diagonals_by_hand():
    """conv_bsgs_diagonals against its definition on a tiny layout written out by hand: 16 slots,
    chunk 2 (8 chunks), C = 2 channels of 3 taps, g = 2.  D_b[s] = kernel_c[tap] with
    c = (s / 2) mod 2, tap = s / 2 + b (when < 3)."""
    k = np.array([[1.0, 2.0, 3.0], [10.0, 20.0, 30.0]])
    D = C.conv_bsgs_diagonals(k, 2, 16, 2)
    # chunks 0..7 -> (channel, tap) for b = 0: (0,0) (1,1) (0,2) (1,-) (0,-) ...
    assert D[0].tolist() == [1, 1, 20, 20, 3, 3, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0]
    # b = 1: chunk q reads tap q + 1: (0,1) (1,2) (0,-) ...; chunk 7 wraps to tap 0 of channel 1
    assert D[1].tolist() == [2, 2, 30, 30, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 10, 10]


def test_replicated_vecmat_fold_identity():
    """Replicated-output diagonals are rotation-periodic, D_{k + m t} = rot(D_k, m t), so the first
    m diagonals plus a fold over m t give x @ W replicated (the oracle's vec_mat_bsgs_fold), pinned
    against numpy matmul with the slot simulator; a fold with the wrong step does not."""
    rng = np.random.default_rng(3)
    x, W = rng.normal(size=256), rng.normal(size=(256, 64))
    D = C.vecmat_diagonals(W, NS, True)
    for k in (0, 5, 63):
        for t in (1, 3):
            assert np.array_equal(D[k + 64 * t], np.roll(D[k], -64 * t))
    xr = C.replicate(x, NS)
    yp = sum(np.roll(xr, -k) * D[k] for k in range(64))
    y = sum(np.roll(yp, -64 * t) for t in range(4))
    assert np.allclose(y, np.tile(x @ W, NS // 64), atol=1e-9)
    bad = sum(np.roll(yp, -32 * t) for t in range(4))
    assert not np.allclose(bad, np.tile(x @ W, NS // 64), atol=1e-3)


@pytest.mark.slow
def test_oracle_cnn_fast_schedule_end_to_end():
    """The oracle with the bench's evaluation schedule (one-level conv, folded BSGS FC1, BSGS FC2,
    input one level lower) meets the same 5e-3 / argmax bar against the float network."""
    from oracle.oracle import OracleContext
    w = cnn_weights(3)
    img = mnist_like_images(1, 4, start=9)[0]
    ctx = OracleContext(CFG4.logN, CFG4.bits, CFG4.n_special, CFG4.seed)
    ctx.keygen(C.cnn_rotation_steps(conv_g=C.CONV_G, fc_bsgs=True, fc1_g=C.FC1_G))   # 47 keys
    ct = C.cnn_encrypt_input(ctx, img, 0, C.CNN_PLAN_BSGS)
    out = C.cnn_forward(ctx, ct, w, lazy=True, bsgs=True, conv_g=C.CONV_G, fc1_g=C.FC1_G)
    assert ct.level == ctx.L - 2 and out.level == 0
    z = ctx.decode(ctx.decrypt(out), 10)
    ref = float_net_numpy(img, w)
    assert np.max(np.abs(z - ref)) < 5e-3 and np.argmax(z) == np.argmax(ref)

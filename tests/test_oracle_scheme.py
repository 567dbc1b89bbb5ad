"""Pins of the oracle's scheme layer against exact algebraic identities
(schoolbook products and big-int CRT on tiny N), a library Vandermonde solve, and
homomorphism / rotation-group laws at realistic N.
"""
import numpy as np
import pytest

from conftest import negacyclic_mul
from oracle.oracle import (OCt, OPt, OracleContext, sid, P_ENC_E0, P_ENC_E1, P_ENC_V, P_PK_A,
                           P_PK_E)


def crt(residues, qs):
    Q = 1
    for q in qs:
        Q *= q
    x = 0
    for r, q in zip(residues, qs):
        Qi = Q // q
        x += int(r) * Qi * pow(Qi, -1, q)
    return x % Q, Q


def centered(x, Q):
    return x - Q if 2 * x > Q else x


@pytest.fixture(scope="module")
def tiny():
    """N=32, 3 data primes + 2 special primes of 30 bits."""
    c = OracleContext(5, (30, 30, 30, 30, 30), 2, 9)
    c.keygen([1, 3, -1])
    return c


@pytest.fixture(scope="module")
def mid():
    c = OracleContext(12, (60, 40, 40, 60), 1, 0)
    c.keygen([1, 2, 3, 5, -1, 2048])
    return c


# -------------------------------------------------------------- P6 encode ---
@pytest.mark.parametrize("logN", [4, 5])
def test_encode_matches_vandermonde_solve(logN):
    """m is the unique real polynomial with m(zeta^{5^j}) = D z_j and m(zeta^{-5^j}) = D z_j
    (C6); solve that linear system with numpy.linalg and compare the pre-rounding values."""
    c = OracleContext(logN, (30, 30), 1, 0)
    N, ns = c.N, c.N // 2
    z = np.random.default_rng(logN).uniform(-1, 1, ns)
    scale = 2.0 ** 20
    pre, m = c.encode_coeffs(z, scale)
    zeta = np.exp(1j * np.pi / N)
    roots = [zeta ** pow(5, j, 2 * N) for j in range(ns)] + [zeta ** (-pow(5, j, 2 * N)) for j in range(ns)]
    V = np.array([[r ** i for i in range(N)] for r in roots])
    y = np.concatenate([scale * z, scale * z])
    sol = np.linalg.solve(V, y)
    assert np.max(np.abs(sol.imag)) < 1e-6
    assert np.allclose(pre, sol.real, rtol=0, atol=1e-6)
    assert np.array_equal(m, np.where(pre >= 0, np.floor(pre + 0.5), np.ceil(pre - 0.5)).astype(np.int64))


def test_encode_decode_roundtrip_linearity_and_rotation(mid):
    c = mid
    rng = np.random.default_rng(4)
    z1, z2 = rng.uniform(-1, 1, (2, c.slots))
    D = 2.0 ** 40
    p1, p2 = c.encode(z1, D, 2), c.encode(z2, D, 2)
    assert np.max(np.abs(c.decode(p1) - z1)) < 2.0 ** -30
    s = OPt(c._pw(0, p1.words[None], p2.words[None], 2)[0], 2, D)
    assert np.max(np.abs(c.decode(s) - (z1 + z2))) < 2.0 ** -29
    # decode(phi_{5^k}(m)) = roll(z, -k)  (C6 left rotation)
    for k in (1, 3, c.slots - 1):
        g = pow(5, k, 2 * c.N)
        rw = np.stack([c.automorph_ntt(p1.words[t], t, g) for t in range(3)])
        assert np.max(np.abs(c.decode(OPt(rw, 2, D)) - np.roll(z1, -k))) < 2.0 ** -30
    # phi_{2N-1} conjugates the slots: real slots are unchanged
    rw = np.stack([c.automorph_ntt(p1.words[t], t, 2 * c.N - 1) for t in range(3)])
    assert np.max(np.abs(c.decode(OPt(rw, 2, D)) - z1)) < 2.0 ** -30


# ------------------------------------------------------------- P7 encrypt ---
def test_encrypt_exact_identity(tiny):
    """c0 + c1 s - m = v e + e0 + e1 s (mod Q) exactly, with the oracle's own randomness."""
    c = tiny
    N = c.N
    s_coef, _ = c.secret_key()
    z = np.random.default_rng(1).uniform(-1, 1, c.slots)
    pt = c.encode(z, 2.0 ** 20, 2)
    sid_ = 77
    ct = c.encrypt(pt, sid_)
    v = c.sample_ternary(sid(P_ENC_V, sid_, 0))
    e0 = c.sample_cdt(sid(P_ENC_E0, sid_, 0))
    e1 = c.sample_cdt(sid(P_ENC_E1, sid_, 0))
    e = c.sample_cdt(sid(P_PK_E, 0, 0))
    ve = negacyclic_mul(v, e, N)
    e1s = negacyclic_mul(e1, s_coef, N)
    rhs = [ve[i] + int(e0[i]) + e1s[i] for i in range(N)]
    s_ntt = c.secret_key()[1]
    for i in range(3):
        q = c.q[i]
        lhs = [(int(a) + int(b) * int(s) - int(m)) % q
               for a, b, s, m in zip(ct.words[0, i], ct.words[1, i], s_ntt[i], pt.words[i])]
        assert [int(x) for x in c.intt(i, np.array(lhs, dtype=np.uint64))] == [r % q for r in rhs]
    # the public key's uniform half is the C13 draw
    assert np.array_equal(c.public_key()[1, 1], c.sample_uniform(sid(P_PK_A, 0, 1), 1))


# -------------------------------------------------------------- P10 tensor ---
def test_tensor_exact_identity(tiny):
    c = tiny
    N, lvl = c.N, 2
    rng = np.random.default_rng(5)
    x = OCt(np.stack([np.stack([rng.integers(0, q, N, dtype=np.uint64) for q in c.q[:3]]) for _ in range(2)]), lvl, 1.0)
    y = OCt(np.stack([np.stack([rng.integers(0, q, N, dtype=np.uint64) for q in c.q[:3]]) for _ in range(2)]), lvl, 1.0)
    d = c.tensor(x, y)
    s_coef, _ = c.secret_key()
    s2 = negacyclic_mul(s_coef, s_coef, N)
    for i in range(3):
        q = c.q[i]
        co = lambda w: [int(t) for t in c.intt(i, w)]
        X0, X1, Y0, Y1 = co(x.words[0, i]), co(x.words[1, i]), co(y.words[0, i]), co(y.words[1, i])
        D0, D1, D2 = co(d.words[0, i]), co(d.words[1, i]), co(d.words[2, i])
        lhs = [a + b + cc for a, b, cc in zip(D0, negacyclic_mul(D1, s_coef, N), negacyclic_mul(D2, s2, N))]
        L1 = [a + b for a, b in zip(X0, negacyclic_mul(X1, s_coef, N))]
        L2 = [a + b for a, b in zip(Y0, negacyclic_mul(Y1, s_coef, N))]
        assert [t % q for t in lhs] == negacyclic_mul(L1, L2, N, q)


# ------------------------------------------------------------ P8 keyswitch ---
@pytest.mark.parametrize("which", ["relin", 1, -1])
def test_keyswitch_noise_identity(tiny, which):
    """u0 + u1 s = d s' + small, with |small| <= (K/2 + 1)(1 + ||s||_1) + sum_j |D_j e_j| / P."""
    c = tiny
    N, lvl = c.N, 2
    rng = np.random.default_rng(6)
    d = np.stack([rng.integers(0, q, N, dtype=np.uint64) for q in c.q[:3]])
    s_coef, s_ntt = c.secret_key()
    if which == "relin":
        u = c.keyswitch(d, lvl, None)
        sp = [np.array([(int(a) * int(a)) % c.q[i] for a in s_ntt[i]], dtype=np.uint64) for i in range(3)]
    else:
        u = c.keyswitch(d, lvl, which)
        g = c.galois_elt(which)
        sp = [c.automorph_ntt(s_ntt[i], i, g) for i in range(3)]
    res = []
    for i in range(3):
        q = c.q[i]
        w = [(int(a) + int(b) * int(s) - int(dd) * int(t)) % q
             for a, b, s, dd, t in zip(u[0, i], u[1, i], s_ntt[i], d[i], sp[i])]
        res.append(c.intt(i, np.array(w, dtype=np.uint64)))
    Q = c.q[0] * c.q[1] * c.q[2]
    err = [abs(centered(crt([res[i][n] for i in range(3)], c.q[:3])[0], Q)) for n in range(N)]
    P = c.q[3] * c.q[4]
    bound = (c.K / 2 + 1) * (1 + N) + 3 * N * (max(c.q[:3]) // 2) * 19 / P
    assert max(err) <= bound
    assert max(err) < 2 ** 20  # far below any wrong-index/sign result (~q)


# -------------------------------------------------------------- P9 rescale ---
def test_rescale_is_exact_round_divide(tiny):
    c = tiny
    N, lvl = c.N, 2
    rng = np.random.default_rng(8)
    w = np.stack([np.stack([rng.integers(0, q, N, dtype=np.uint64) for q in c.q[:3]]) for _ in range(2)])
    out = c.rescale(OCt(w, lvl, 2.0 ** 40))
    assert out.level == 1 and out.scale == 2.0 ** 40 / c.q[2]
    ql = c.q[2]
    for p in range(2):
        coeffs = [c.intt(i, w[p, i]) for i in range(3)]
        expect = [[0] * N for _ in range(2)]
        for n in range(N):
            X, _ = crt([coeffs[i][n] for i in range(3)], c.q[:3])
            r = (X + (ql - 1) // 2) // ql       # round(X / q_l), no ties (q_l odd)
            for i in range(2):
                expect[i][n] = r % c.q[i]
        for i in range(2):
            assert np.array_equal(out.words[p, i], c.ntt(i, np.array(expect[i], dtype=np.uint64)))


def test_moddown_divround_two_primes(tiny):
    """C15 with |B| = 2: out = floor((X + h) / B) - u, 0 <= u < 2, per coefficient."""
    c = tiny
    N = c.N
    rng = np.random.default_rng(9)
    keep, drop = [0, 1, 2], [3, 4]
    xk = np.stack([rng.integers(0, c.q[i], N, dtype=np.uint64) for i in keep])
    xd = np.stack([rng.integers(0, c.q[i], N, dtype=np.uint64) for i in drop])
    out = c.divround(keep, drop, xk, xd)
    B = c.q[3] * c.q[4]
    qs = [c.q[i] for i in keep + drop]
    us = set()
    for n in range(N):
        X, _ = crt([xk[0][n], xk[1][n], xk[2][n], xd[0][n], xd[1][n]], qs)
        base = (X + (B - 1) // 2) // B
        found = [u for u in range(2) if all((base - u) % c.q[i] == int(out[i][n]) for i in keep)]
        assert found, f"coefficient {n}: not floor((X+h)/B) - u"
        us.add(found[0])
    assert 0 in us


# ------------------------------------------------------- homomorphism laws ---
def test_homomorphism_add_mul_rotate(mid):
    c = mid
    rng = np.random.default_rng(12)
    D = 2.0 ** 40
    for trial in range(3):
        z1, z2 = rng.uniform(-1, 1, (2, c.slots))
        a = c.encrypt(c.encode(z1, D, 2), 2 * trial)
        b = c.encrypt(c.encode(z2, D, 2), 2 * trial + 1)
        dec = lambda ct, n=None: c.decode(c.decrypt(ct), n)
        assert np.max(np.abs(dec(a) - z1)) < 1e-6
        assert np.max(np.abs(dec(c.add(a, b)) - (z1 + z2))) < 1e-6
        assert np.max(np.abs(dec(c.sub(a, b)) - (z1 - z2))) < 1e-6
        assert np.max(np.abs(dec(c.negate(a)) + z1)) < 1e-6
        m = c.rescale(c.relinearize(c.tensor(a, b)))
        assert m.level == 1 and np.max(np.abs(dec(m) - z1 * z2)) < 1e-6
        pm = c.rescale(c.mul_plain(a, c.encode(z2, float(c.q[2]), 2)))
        assert pm.scale == D and np.max(np.abs(dec(pm) - z1 * z2)) < 1e-6
        for k in (1, 5, -1):
            assert np.max(np.abs(dec(c.rotate(a, k)) - np.roll(z1, -k))) < 1e-6
        # group action rot(rot(v,2),3) == rot(v,5); rotation by n_s is the identity
        r23 = c.rotate(c.rotate(a, 2), 3)
        assert np.max(np.abs(dec(r23) - dec(c.rotate(a, 5)))) < 1e-6
        assert np.max(np.abs(dec(c.rotate(a, c.slots)) - z1)) < 1e-6


def test_depth_accounting():
    """A fresh ciphertext at an L-prime chain admits exactly L-1 rescaled squarings."""
    c = OracleContext(11, (60, 40, 40, 40, 60), 1, 1)
    c.keygen([])
    x = np.random.default_rng(0).uniform(-1, 1, c.slots)
    ct = c.encrypt(c.encode(x, 2.0 ** 40, c.L - 1), 0)
    for i in range(c.L - 1):
        ct = c.square(ct)
    assert ct.level == 0
    assert np.max(np.abs(c.decode(c.decrypt(ct)) - x ** (2 ** (c.L - 1)))) < 1e-4
    with pytest.raises(ValueError):
        c.square(ct)


# ---------------------------------------------- lazy-ModDown vec_mat pins ---
def test_vec_mat_lazy_n1_equals_plain_exactly():
    """With a single diagonal there is no rotation: ModDown(P D_0 c) must equal D_0 c exactly
    (C15: ModDown(P X + Y) = X + ModDown(Y)), so vec_mat_lazy == vec_mat word for word."""
    from oracle import circuits as OC
    c = OracleContext(11, (50, 40, 40, 50, 50), 2, 5)
    c.keygen([1])
    rng = np.random.default_rng(1)
    W = rng.normal(0, 0.1, (1, 1))
    ct = c.encrypt(c.encode(rng.uniform(-1, 1, c.slots), 2.0 ** 30, 2), 0)
    a = OC.vec_mat(c, ct, W, None, replicate_out=True)
    b = OC.vec_mat_lazy(c, ct, W, None, replicate_out=True)
    assert np.array_equal(a.words, b.words) and a.scale == b.scale


@pytest.mark.parametrize("rep", [False, True])
def test_vec_mat_lazy_matches_matmul(rep):
    """Decrypted lazy vec_mat vs numpy x @ W (float definition) and vs the per-rotation-ModDown
    vec_mat (both approximate the same product; they differ only by rounding noise)."""
    from oracle import circuits as OC
    c = OracleContext(12, (60, 40, 40, 60), 1, 0)
    n, m = 16, (16 if rep else 5)
    c.keygen(range(1, n))
    rng = np.random.default_rng(2)
    x, W, bias = rng.uniform(-1, 1, n), rng.normal(0, 0.1, (n, m)), rng.normal(0, 0.1, m)
    ct = c.encrypt(c.encode(OC.replicate(x, c.slots), 2.0 ** 40, 2), 3)
    y_lazy = c.decode(c.decrypt(OC.vec_mat_lazy(c, ct, W, bias, rep)), m)
    y_plain = c.decode(c.decrypt(OC.vec_mat(c, ct, W, bias, rep)), m)
    ref = x @ W + bias
    assert np.max(np.abs(y_lazy - ref)) < 1e-6
    assert np.max(np.abs(y_lazy - y_plain)) < 1e-6


# ------------------------------------ SURVEY 8(f) #2/#4 circuit pins (float) ---
def test_dot_power_polyval_circuits_vs_float():
    """dot / dot_plain / power / polyval compositions decrypt to numpy's values (the definitions)."""
    from oracle import circuits as OC
    c = OracleContext(12, (60, 40, 40, 40, 60), 1, 7)
    c.keygen([1, 2, 4, 8, 16, 32])
    rng = np.random.default_rng(3)
    n = 37
    x, y = np.zeros(c.slots), np.zeros(c.slots)
    x[:n], y[:n] = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    lvl = c.L - 1
    cx, cy = c.encrypt(c.encode(x, 2.0 ** 40, lvl), 1), c.encrypt(c.encode(y, 2.0 ** 40, lvl), 2)
    assert abs(c.decode(c.decrypt(OC.dot(c, cx, cy, n)), 1)[0] - x @ y) < 1e-6
    assert abs(c.decode(c.decrypt(OC.dot_plain(c, cx, y, n)), 1)[0] - x @ y) < 1e-6
    for p in (2, 3, 4):
        r = OC.power(c, cx, p)
        assert r.level == lvl - (p - 1).bit_length()          # depth ceil(log2 p)
        assert np.max(np.abs(c.decode(c.decrypt(r), n) - x[:n] ** p)) < 1e-6
    r = OC.polyval(c, cx, [0.0, 1.0, 2.0])                      # Table 4: 2x^2 + x
    assert np.max(np.abs(c.decode(c.decrypt(r), n) - (2 * x[:n] ** 2 + x[:n]))) < 1e-6
    r = OC.polyval(c, cx, [0.5, -1.0, 0.25, 0.125])
    assert np.max(np.abs(c.decode(c.decrypt(r), n) - (0.5 - x[:n] + 0.25 * x[:n] ** 2 + 0.125 * x[:n] ** 3))) < 1e-6


def test_vec_mat_bsgs_pins():
    """BSGS vec_mat: with one giant step (g >= n) it IS vec_mat_lazy (word for word); otherwise it
    decrypts to x @ W (float definition) like the other two forms."""
    from oracle import circuits as OC
    c = OracleContext(12, (60, 40, 40, 60), 1, 0)
    n, m = 16, 16
    c.keygen(range(1, n))
    rng = np.random.default_rng(4)
    x, W, bias = rng.uniform(-1, 1, n), rng.normal(0, 0.1, (n, m)), rng.normal(0, 0.1, m)
    ct = c.encrypt(c.encode(OC.replicate(x, c.slots), 2.0 ** 40, 2), 3)
    one = OC.vec_mat_bsgs(c, ct, W, bias, True, g=16)
    assert np.array_equal(one.words, OC.vec_mat_lazy(c, ct, W, bias, True).words)
    for g in (4, 8):
        y = c.decode(c.decrypt(OC.vec_mat_bsgs(c, ct, W, bias, True, g=g)), m)
        assert np.max(np.abs(y - (x @ W + bias))) < 1e-6
    # E construction: rot(E[k2][k1], g k2) = D_{k1 + g k2}
    D = OC.vecmat_diagonals(W, c.slots, True)
    E = OC.bsgs_diagonals(D, 4)
    assert np.array_equal(np.roll(E[2, 1], -8), D[9])


def test_hoisted_fold_oracle_pins():
    """Oracle hoisted fold: decrypts to the log2 fold's values (same sum), and with n1 = #chunks
    (one level) on two chunks it equals a single lazy vec_mat with all-one diagonals."""
    from oracle import circuits as OC
    c = OracleContext(11, (50, 40, 40, 50), 1, 3)
    chunk, ns = 64, 1024
    c.keygen(sorted(set(OC.conv_fold_steps(chunk, ns)) | {64 * b for b in range(1, 4)} | {256 * a for a in range(1, 4)}))
    z = np.random.default_rng(1).uniform(-1, 1, ns)
    ct = c.encrypt(c.encode(z, 2.0 ** 30, 2), 0)
    folded = ct
    for step in OC.conv_fold_steps(chunk, ns):
        folded = c.add(folded, c.rotate(folded, step))
    h = OC.hoisted_fold(c, ct, chunk, 4)
    assert h.level == ct.level and h.scale == ct.scale
    # both forms compute the same sum of 16 rotated copies; their errors are CKKS noise only:
    # fresh noise ~340 sqrt(N) / 2^30 ~ 1.4e-5 per slot, summed over 16 copies -> <= ~2e-4
    ref = sum(np.roll(z, -64 * m) for m in range(16))
    assert np.max(np.abs(c.decode(c.decrypt(h)) - ref)) < 2e-4
    assert np.max(np.abs(c.decode(c.decrypt(folded)) - ref)) < 2e-4


def test_one_level_conv_oracle_pin():
    """Oracle im2col_conv_bsgs (C = 4 channels, g = 4 baby steps x 4 giant steps on 16 chunks, 2x2
    kernels) decrypts to the exact slot convolution within CKKS noise, consumes one level, and
    agrees with the paper's two-level conv order."""
    from oracle import circuits as OC
    c = OracleContext(11, (50, 40, 40, 50), 1, 5)
    chunk, ns, g = 64, 1024, 4
    c.keygen(sorted(set(OC.conv_fold_steps(chunk, ns)) | {chunk * b for b in range(1, g)}
                    | {chunk * g * a for a in range(1, ns // chunk // g)}))
    rng = np.random.default_rng(7)
    z = np.zeros(ns)
    z[: 4 * chunk] = rng.uniform(-1, 1, 4 * chunk)      # 4 taps x 64 windows
    k = rng.uniform(-1, 1, (4, 4))
    bias = rng.uniform(-0.5, 0.5, 4)
    ref = np.zeros(ns)
    for ch in range(4):
        t = z * OC.conv_kernel_slots(k[ch], chunk, ns)
        ref += sum(np.roll(t, -chunk * m) for m in range(ns // chunk)) * OC.conv_mask_slots(ch, 4, chunk, ns)
    ref += OC.conv_bias_slots(bias, chunk, ns)
    ct = c.encrypt(c.encode(z, 2.0 ** 30, 2), 0)
    new = OC.im2col_conv_bsgs(c, ct, k, bias, chunk, g, 0)
    old = OC.im2col_conv(c, ct, k, bias, chunk, 0, 0)
    assert new.level == 1 and old.level == 0
    assert new.scale == ct.scale * (float(c.q[2]) / c.q[2])
    zn, zo = c.decode(c.decrypt(new)), c.decode(c.decrypt(old))
    # fresh noise ~1.4e-5 per slot (N = 2^11, scale 2^30) times |k| <= 1 over 4 taps, plus rescale
    # and key-switch rounding: ~3e-5 measured for the paper's order
    assert np.max(np.abs(zn - ref)) < 2e-4 and np.max(np.abs(zo - ref)) < 2e-4


def test_vec_mat_bsgs_fold_oracle_pin():
    """Oracle vec_mat_bsgs_fold (n 64 -> m 16, g 8: 2 groups, fold 4) decrypts to x @ W replicated
    (numpy) within CKKS noise and to the same values as the plain diagonal method (vec_mat)."""
    from oracle import circuits as OC
    c = OracleContext(11, (50, 40, 40, 50), 1, 9)
    ns, n, m, g = 1024, 64, 16, 8
    c.keygen(sorted(set(range(1, n)) | {16, 32, 48}))
    rng = np.random.default_rng(11)
    x, W, bias = rng.uniform(-1, 1, n), rng.normal(0, 0.2, (n, m)), rng.uniform(-0.5, 0.5, m)
    ct = c.encrypt(c.encode(OC.replicate(x, ns), 2.0 ** 30, 2), 0)
    f = OC.vec_mat_bsgs_fold(c, ct, W, bias, 0, g=g)
    p = OC.vec_mat(c, ct, W, bias, True, 0)
    assert f.level == p.level == 1 and f.scale == p.scale
    ref = np.tile(x @ W + bias, ns // m)
    zf, zp = c.decode(c.decrypt(f)), c.decode(c.decrypt(p))
    # fresh noise ~1.4e-5 per slot times |W| summed over 64 terms, plus key-switch and rescale rounding
    assert np.max(np.abs(zf - ref)) < 2e-4 and np.max(np.abs(zp - ref)) < 2e-4


def test_symmetric_encrypt_oracle_pin():
    """Oracle symmetric encryption: decrypt - m is the NTT of ONE small integer
    polynomial e (the same in every limb, |e| within the CDT's range, std ~ sigma = 3.2); c1 depends
    only on the public (a_seed, stream): another context seed (other secret key) gives the same c1,
    another a_seed a different one; the ciphertext decodes to the message."""
    c = OracleContext(10, (50, 40, 40), 1, 21)
    c.keygen([])
    z = np.random.default_rng(5).uniform(-1, 1, c.slots)
    pt = c.encode(z, 2.0 ** 30, 1)
    ct = c.encrypt_symmetric(pt, 7, 0xABCDEF)
    d = c.decrypt(ct)
    es = []
    for i in range(2):
        q = int(c.q[i])
        diff = np.array([(int(a) - int(b)) % q for a, b in zip(d.words[i], pt.words[i])], dtype=np.uint64)
        e = np.array([int(v) if int(v) <= q // 2 else int(v) - q for v in c.intt(i, diff)])
        es.append(e)
    assert np.array_equal(es[0], es[1])
    assert np.max(np.abs(es[0])) <= 41 and 2.5 < np.std(es[0]) < 4.0
    c2 = OracleContext(10, (50, 40, 40), 1, 22)
    c2.keygen([])
    ct2 = c2.encrypt_symmetric(c2.encode(z, 2.0 ** 30, 1), 7, 0xABCDEF)
    assert np.array_equal(ct2.words[1], ct.words[1]) and not np.array_equal(ct2.words[0], ct.words[0])
    assert not np.array_equal(c.encrypt_symmetric(pt, 7, 0xABCDEE).words[1], ct.words[1])
    assert np.max(np.abs(c.decode(c.decrypt(ct)) - z)) < 1e-4


def test_seeded_wire_reference_packer():
    """oracle/wire.pack_seeded: header fields at their offsets (magic, size 2, a_seed and stream in
    the tail) and a c0-only payload, half the full form's."""
    import struct
    from oracle import wire
    rng = np.random.default_rng(2)
    q = [1073479681, 1073184769]
    c0 = np.stack([np.stack([rng.integers(0, qi, 64, dtype=np.uint64) for qi in q]) for _ in range(3)])
    blob = wire.pack_seeded(c0, q, 1, 2.0 ** 20, 0x1122334455667788, 9)
    assert blob[:8] == b"HECKKSS1"
    log2n, B, size, level, scale, pay, nl, a_seed, stream = struct.unpack("<IIIIdQIQQ", blob[8:60])
    assert (log2n, B, size, level, scale, nl) == (6, 3, 2, 1, 2.0 ** 20, 2)
    assert (a_seed, stream) == (0x1122334455667788, 9) and blob[60:64] == bytes(4)
    full = wire.pack(np.stack([c0, c0], axis=1), q, 1, 2.0 ** 20)
    assert pay == len(blob) - 64 == (len(full) - 64) // 2 == 3 * 64 * 60 // 8

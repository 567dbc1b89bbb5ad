"""GPU parity of the SURVEY §8(f) #2/#4 circuits (PAPER.md:166-171 power / polyval, :170 dot, Table 4
polyval 2x^2+x, Table 5 dot / dot_plain) against the oracle's compositions in oracle/circuits.py:
word for word where no float encoding is involved (dot, power, mod_switch, the dot_plain chain from
an injected oracle plaintext), and within tolerance of numpy for the all-GPU forms."""
import numpy as np
import pytest

from oracle import circuits as OC
from oracle.oracle import OracleContext

pytestmark = pytest.mark.gpu

PARAMS = {"q64": (12, (60, 40, 40, 40, 60), 1, 7), "q32": (12, (31, 26, 26, 26, 26, 31), 1, 7)}
STEPS = [1, 2, 4, 8, 16, 32]


@pytest.fixture(scope="module", params=list(PARAMS))
def pair(request):
    from paper_2104_03152_b200 import Context
    logN, bits, K, seed = PARAMS[request.param]
    o = OracleContext(logN, bits, K, seed)
    o.keygen(STEPS)
    g = Context(logN, bits, K, seed)
    g.he_keygen(STEPS)
    scale = 2.0 ** (40 if request.param == "q64" else 26)
    return o, g, scale


def _inputs(o, g, scale, n=37):
    rng = np.random.default_rng(5)
    x, y = np.zeros(o.slots), np.zeros(o.slots)
    x[:n], y[:n] = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    lvl = o.L - 1
    ox, oy = o.encrypt(o.encode(x, scale, lvl), 1), o.encrypt(o.encode(y, scale, lvl), 2)
    gx, gy = g.he_ct_import_words(ox.words[None], lvl, scale), g.he_ct_import_words(oy.words[None], lvl, scale)
    return x, y, ox, oy, gx, gy, n


def test_mod_switch_dot_power_bit_exact(pair):
    o, g, scale = pair
    x, y, ox, oy, gx, gy, n = _inputs(o, g, scale)
    assert np.array_equal(g.he_mod_switch_to(gx, 1).words()[0], OC.mod_switch(o, ox, 1).words)
    d = g.he_dot(gx, gy, n)
    ref = OC.dot(o, ox, oy, n)
    assert np.array_equal(d.words()[0], ref.words) and d.scale == ref.scale
    tol = 1e-6 if scale > 2 ** 30 else 5e-3
    assert abs(g.he_decode(g.he_decrypt(d), 1)[0, 0] - x @ y) < tol
    for p in (2, 3, 4, 5):
        r = g.he_power(gx, p)
        rr = OC.power(o, ox, p)
        assert np.array_equal(r.words()[0], rr.words), p
        assert r.level == o.L - 1 - (p - 1).bit_length()


def test_dot_plain_chain_bit_exact_and_all_gpu(pair):
    o, g, scale = pair
    x, y, ox, oy, gx, gy, n = _inputs(o, g, scale)
    lvl = o.L - 1
    _, m = o.encode_coeffs(y, float(o.q[lvl]))
    t = g.he_rescale(g.he_mul_plain(gx, g.he_pt_from_int_coeffs(m, float(o.q[lvl]), lvl)))
    s = 1
    while s < n:
        t = g.he_add(t, g.he_rotate(t, s))
        s <<= 1
    ref = OC.dot_plain(o, ox, y, n)
    assert np.array_equal(t.words()[0], ref.words)
    tol = 1e-6 if scale > 2 ** 30 else 5e-3
    d = g.he_dot_plain(gx, y, n)
    assert abs(g.he_decode(g.he_decrypt(d), 1)[0, 0] - x @ y) < tol


@pytest.mark.parametrize("coeffs", [[0.0, 1.0, 2.0], [0.5, -1.0, 0.25, 0.125]])
def test_polyval(pair, coeffs):
    """Table 4 polyval(2x^2 + x) and a cubic: words equal to the oracle's (the constant plaintexts
    round identically: their only nonzero coefficient is scale * c); values vs numpy."""
    o, g, scale = pair
    x, y, ox, oy, gx, gy, n = _inputs(o, g, scale)
    r = g.he_polyval(gx, coeffs)
    rr = OC.polyval(o, ox, coeffs)
    assert np.array_equal(r.words()[0], rr.words) and r.level == rr.level
    ref = sum(c * x[:n] ** i for i, c in enumerate(coeffs))
    tol = 1e-6 if scale > 2 ** 30 else 5e-3
    assert np.max(np.abs(g.he_decode(g.he_decrypt(r), n)[0] - ref)) < tol

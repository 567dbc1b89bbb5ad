"""GPU parity of the ring layer (BASELINE config 2):
parameters, NTT / INTT, pointwise modmul and the fused ring product, called
through the C-ABI and compared word for word with the CPU oracle."""
import numpy as np
import pytest

from oracle.oracle import OracleContext
from synthetic import CFG1, CFG3, CFG4, CFG5B, CFG2_PRIME_BITS, uniform_residues

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    return torch


def gpu_ctx(logN, bits, K, seed):
    from paper_2104_03152_b200 import Context
    return Context(logN, bits, K, seed)


@pytest.mark.parametrize("cfg", [CFG1, CFG3, CFG4, CFG5B], ids=lambda c: c.name)
def test_params_match_oracle(cfg):
    o = OracleContext(cfg.logN, cfg.bits, cfg.n_special, cfg.seed)
    g = gpu_ctx(cfg.logN, cfg.bits, cfg.n_special, cfg.seed)
    assert np.array_equal(g.primes, o.primes)
    assert np.array_equal(g.psis, o.psis)
    assert np.array_equal(g.he_context_cdt(), o.cdt)


def _to_dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


def _from_dev(t):
    return t.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("logN,L,B,small", [(10, 3, 5, False), (13, 4, 3, False), (14, 8, 2, False),
                                            (15, 4, 2, False), (10, 3, 3, True), (13, 4, 3, True),
                                            (14, 3, 2, True)])
def test_ntt_forward_inverse_bit_exact(torch_cuda, logN, L, B, small):
    """small: every prime < 2^31 -> the 32-bit arithmetic engine (k_ntt32) runs."""
    torch = torch_cuda
    bits = (31, 26, 30, 20, 28, 31)[:L] if small else CFG2_PRIME_BITS(L)
    o = OracleContext(logN, bits, 0, 1)
    g = gpu_ctx(logN, bits, 0, 1)
    N = 1 << logN
    a = uniform_residues(o.q, N, B, seed=1)
    # edge rows: zeros, all q-1
    a[0, 0, :] = 0
    a[-1, -1, :] = np.uint64(o.q[L - 1] - 1)
    d = _to_dev(torch, a)
    g.he_ntt_forward(d, B, L)
    got = _from_dev(d)
    for b in range(B):
        for i in range(L):
            assert np.array_equal(got[b, i], o.ntt(i, a[b, i])), (b, i)
    g.he_ntt_inverse(d, B, L)
    assert np.array_equal(_from_dev(d), a)


@pytest.mark.parametrize("logN,L,B", [(10, 3, 4), (13, 4, 3), (15, 2, 2)])
def test_modmul_and_fused_ring_product(torch_cuda, logN, L, B):
    torch = torch_cuda
    bits = CFG2_PRIME_BITS(L)
    o = OracleContext(logN, bits, 0, 1)
    g = gpu_ctx(logN, bits, 0, 1)
    N = 1 << logN
    a = uniform_residues(o.q, N, B, seed=2)
    b = uniform_residues(o.q, N, B, seed=3)
    out = torch.empty((B, L, N), dtype=torch.int64, device="cuda")
    g.he_modmul(_to_dev(torch, a), _to_dev(torch, b), out, B, L)
    got = _from_dev(out)
    for i in range(L):
        q = o.q[i]
        ref = np.array([(int(x) * int(y)) % q for x, y in zip(a[:, i].ravel(), b[:, i].ravel())],
                       dtype=np.uint64).reshape(B, N)
        assert np.array_equal(got[:, i], ref)
    # fused INTT(NTT(a) . b): the oracle composes its own NTT, big-int products and INTT
    g.he_ntt_mul_intt(_to_dev(torch, a), _to_dev(torch, b), out, B, L)
    got = _from_dev(out)
    for bb in range(B):
        for i in range(L):
            q = o.q[i]
            fa = o.ntt(i, a[bb, i])
            prod = np.array([(int(x) * int(y)) % q for x, y in zip(fa, b[bb, i])], dtype=np.uint64)
            assert np.array_equal(got[bb, i], o.intt(i, prod)), (bb, i)

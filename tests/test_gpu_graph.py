"""CUDA-graph recording of a call sequence (he_graph_begin / end / launch / free; include/he_ckks.h):
replays equal eager execution word for word on fresh inputs, handles created while recording hold
the replay's results, the launch counter counts replayed kernels, and a host read-back while
recording fails cleanly (the context stays usable)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("bits", [(50, 40, 40, 50), (31, 26, 26, 31)])
def test_graph_replay_equals_eager(bits):
    import torch
    from paper_2104_03152_b200 import Context, HEError
    dev = torch.device("cuda", 0)
    c = Context(12, bits, 1, 5)
    c.he_set_stream(torch.cuda.current_stream(dev))
    c.he_keygen([1, 2, 3, 4, 5, 6, 7])
    lvl = c.L - 1
    scale = 2.0 ** (40 if bits[0] > 31 else 26)
    rng = np.random.default_rng(1)
    W = rng.normal(0, 0.1, (8, 4))
    D, _ = c.he_vec_mat_encode(W, None, False, 0, lvl, float(c.q[lvl]), lazy=False)
    z_dev = torch.zeros((2, c.slots), dtype=torch.float64, device=dev)
    out = torch.zeros((2, 4), dtype=torch.float64, device=dev)

    def seq():
        ct = c.he_encrypt(c.he_encode(z_dev, scale, lvl), 7)
        r = c.he_rotate(ct, 3)
        y = c.he_vec_mat_pt(r, D)
        c.he_decode(c.he_decrypt(y), 4, out=out)
        return r, y

    c.he_graph_begin()
    r_g, y_g = seq()
    g = c.he_graph_end()
    assert g.kernels > 0
    for trial in range(2):
        x = rng.uniform(-1, 1, (2, 8))
        z_dev.copy_(torch.from_numpy(np.tile(x, (1, c.slots // 8))))
        n0 = c.he_launch_count()
        g.launch()
        torch.cuda.synchronize()
        assert c.he_launch_count() - n0 == g.kernels
        got_r, got_y, got_out = r_g.words(), y_g.words(), out.clone()
        r_e, y_e = seq()
        torch.cuda.synchronize()
        assert np.array_equal(got_r, r_e.words()), trial
        assert np.array_equal(got_y, y_e.words()), trial
        assert torch.equal(got_out, out), trial
        ref = np.roll(np.tile(x, (1, c.slots // 8)), -3, axis=1)[:, :8] @ W
        assert np.max(np.abs(got_out.cpu().numpy() - ref)) < 1e-3
    del r_g, y_g
    g.free()
    # a host read-back while recording fails, and so does he_graph_end; the context stays usable
    c.he_graph_begin()
    ct = c.he_encrypt(c.he_encode(z_dev, scale, lvl), 9)
    with pytest.raises(HEError):
        c.he_decode(c.he_decrypt(ct), 4)   # host output: synchronises
    with pytest.raises(HEError):
        c.he_graph_end()
    with pytest.raises(HEError):
        c.he_graph_end()                   # not recording any more
    v = c.he_decode(c.he_decrypt(c.he_encrypt(c.he_encode(z_dev, scale, lvl), 9)), 4)
    assert np.max(np.abs(v - z_dev[:, :4].cpu().numpy())) < 1e-3

"""Oracle circuits: vec_mat (diagonal method), im2col conv, the paper's CNN.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* vec_mat — PAPER.md:58-61 ("a variant of the encrypted vector-plain matrix
  multiplication proposed by halevi", "replicating the input vector as many
  times as possible into ciphertext slots and only left ciphertext
  rotations"); layout = SURVEY C17.
* im2col conv — PAPER.md:57, 64, 189-213 ("convolution windows as rows ...
  flatten it as a vector via a vertical scan", "one multiplication operation
  and log2(N) rotations and additions"); layout = SURVEY C18/C19.
* CNN — PAPER.md:98: conv 7x7 stride 3, 4 kernels -> x^2 -> FC 256->64 -> x^2
  -> FC 64->10; 6 multiplicative levels.

Every slot-layout helper here is plain numpy indexing written from C17-C19;
``tests/test_layouts.py`` pins them with a float slot simulator against numpy
matmul and torch conv2d.
"""
from __future__ import annotations

import numpy as np

from .oracle import OCt, OracleContext


class ReplicationExhausted(ValueError):
    pass


# ------------------------------------------------------------ layouts ---
def vecmat_diagonals(W: np.ndarray, ns: int, replicate_out: bool) -> np.ndarray:
    """C17: D_k[j] = W[(j+k) mod n][j'] (W is in x out), j' = j mod m when the
    output is replicated, else j' = j for j < m and 0 beyond."""
    n, m = W.shape
    if replicate_out and (ns % n or ns % m):
        raise ValueError("replicated output needs n | slots and m | slots")
    j = np.arange(ns)
    span = (ns // n) * n
    D = np.zeros((n, ns))
    for k in range(n):
        live = np.ones(ns, bool) if replicate_out else (j < m)
        if ns % n and np.any(live & (j + k >= span)):
            raise ReplicationExhausted(f"diagonal {k} reads past the replicated span")
        jp = (j % m) if replicate_out else np.minimum(j, m - 1)
        D[k] = np.where(live, W[(j + k) % n, jp], 0.0)
    return D


def vecmat_bias_slots(bias: np.ndarray, ns: int, replicate_out: bool) -> np.ndarray:
    m = bias.shape[0]
    j = np.arange(ns)
    if replicate_out:
        return bias[j % m].astype(np.float64)
    out = np.zeros(ns)
    out[:m] = bias
    return out


def replicate(x: np.ndarray, ns: int) -> np.ndarray:
    """Client-side replication of an n-vector as many times as fits."""
    n = x.shape[0]
    out = np.zeros(ns)
    r = ns // n
    out[: r * n] = np.tile(x, r)
    return out


def conv_geometry(H: int, W: int, kh: int, kw: int, stride: int):
    oh, ow = (H - kh) // stride + 1, (W - kw) // stride + 1
    windows = oh * ow
    chunk = 1 << (windows - 1).bit_length()
    return oh, ow, windows, chunk


def im2col_slots(img: np.ndarray, kh: int, kw: int, stride: int, ns: int) -> np.ndarray:
    """C18: windows in row-major order of output positions, taps row-major;
    slot = tap * chunk + window (vertical scan of the windows x taps matrix)."""
    H, W = img.shape
    oh, ow, windows, chunk = conv_geometry(H, W, kh, kw, stride)
    if kh * kw * chunk > ns:
        raise ValueError("im2col matrix does not fit the slots")
    out = np.zeros(ns)
    for r in range(oh):
        for c in range(ow):
            w = r * ow + c
            patch = img[r * stride: r * stride + kh, c * stride: c * stride + kw].reshape(-1)
            out[np.arange(kh * kw) * chunk + w] = patch
    return out


def conv_kernel_slots(kernel: np.ndarray, chunk: int, ns: int) -> np.ndarray:
    """C18: K[tap * chunk + w] = kernel[tap] (kernel value replicated along its chunk)."""
    taps = kernel.reshape(-1)
    out = np.zeros(ns)
    for t, v in enumerate(taps):
        out[t * chunk:(t + 1) * chunk] = v
    return out


def conv_mask_slots(c: int, n_ch: int, chunk: int, ns: int) -> np.ndarray:
    """C19: Mask_c = 1 on slots whose chunk index q satisfies q mod C_out = c."""
    q = np.arange(ns) // chunk
    return (q % n_ch == c).astype(np.float64)


def conv_bias_slots(bias: np.ndarray, chunk: int, ns: int) -> np.ndarray:
    q = np.arange(ns) // chunk
    return bias[q % bias.shape[0]].astype(np.float64)


def conv_fold_steps(chunk: int, ns: int) -> list:
    """C19: fold by chunk * 2^r, r = 0 .. log2(ns/chunk) - 1."""
    n_chunks = ns // chunk
    return [chunk << r for r in range(n_chunks.bit_length() - 1)]


# ------------------------------------------------------------ circuits ---
def _shifted(q: int, shift: int) -> float:
    """Plaintext scale q * 2^shift (exact in double for |shift| < 1000)."""
    return float(q) * 2.0 ** shift


def vec_mat(ctx: OracleContext, ct: OCt, W: np.ndarray, bias: np.ndarray | None,
            replicate_out: bool, pt_scale_shift: int = 0) -> OCt:
    """Step 11: acc = sum_k mul_plain(rot(x, k), D_k); rescale once; + bias.
    D_k is encoded at scale q_l / 2^shift (l = ct level) so that the rescale by
    q_l returns the ciphertext to its input scale / 2^shift (C14)."""
    ns = ctx.slots
    D = vecmat_diagonals(W, ns, replicate_out)
    lvl = ct.level
    pscale = _shifted(ctx.q[lvl], -pt_scale_shift)
    acc = None
    for k in range(W.shape[0]):
        r = ct if k == 0 else ctx.rotate(ct, k)
        t = ctx.mul_plain(r, ctx.encode(D[k], pscale, lvl))
        acc = t if acc is None else ctx.add(acc, t)
    acc = ctx.rescale(acc)
    if bias is not None:
        acc = ctx.add_plain(acc, ctx.encode(vecmat_bias_slots(bias, ns, replicate_out),
                                            acc.scale, acc.level))
    return acc


def vec_mat_lazy(ctx: OracleContext, ct: OCt, W: np.ndarray, bias: np.ndarray | None,
                 replicate_out: bool, pt_scale_shift: int = 0) -> OCt:
    """vec_mat with the diagonals' rotations sharing ONE ModDown (lazy ModDown,
    DESIGN.md §3): same diagonals, scales and bias as vec_mat (C17); D_k is
    encoded on the data limbs and the special limbs.  Rescale once, + bias."""
    ns = ctx.slots
    D = vecmat_diagonals(W, ns, replicate_out)
    lvl = ct.level
    pscale = _shifted(ctx.q[lvl], -pt_scale_shift)
    Dqp = np.stack([ctx.coeffs_to_pt_qp(ctx.encode_coeffs(D[k], pscale)[1], lvl) for k in range(W.shape[0])])
    acc = OCt(ctx.vec_mat_lazy_acc(ct, Dqp), lvl, ct.scale * pscale)
    acc = ctx.rescale(acc)
    if bias is not None:
        acc = ctx.add_plain(acc, ctx.encode(vecmat_bias_slots(bias, ns, replicate_out), acc.scale, acc.level))
    return acc


def hoisted_fold(ctx: OracleContext, t: OCt, chunk: int, n1: int) -> OCt:
    """sum_{m < ns/chunk} rot(t, chunk m) as two hoisted lazy-ModDown sums (DESIGN.md §3 'hoisted
    conv fold'): u = sum_{b < n1} rot(t, chunk b), then sum_{a < n2} rot(u, chunk n1 a), n1 n2 =
    ns/chunk.  The diagonals are the plaintext polynomial 1 (the constant-1 slots encoded at scale 1,
    i.e. m = 1 exactly), so the ciphertext scale is unchanged."""
    n_chunks = ctx.slots // chunk
    assert n_chunks % n1 == 0
    n2 = n_chunks // n1
    one = np.zeros((ctx.N,), dtype=np.int64)
    one[0] = 1
    for n, step in ((n1, chunk), (n2, chunk * n1)):
        if n == 1:
            continue
        D = np.stack([ctx.coeffs_to_pt_qp(one, t.level)] * n)
        t = OCt(ctx.vec_mat_lazy_acc(t, D, step), t.level, t.scale)
    return t


def rot_sum(ctx: OracleContext, t: OCt, n: int, step: int) -> OCt:
    """sum_{k < n} rot(t, step k) with ONE lazy ModDown: the lazy vec_mat with unit diagonals (the
    plaintext polynomial 1, i.e. the constant-1 slots encoded at scale 1, m = 1 exactly), so the
    ciphertext scale is unchanged."""
    if n == 1:
        return t
    one = np.zeros((ctx.N,), dtype=np.int64)
    one[0] = 1
    D = np.stack([ctx.coeffs_to_pt_qp(one, t.level)] * n)
    return OCt(ctx.vec_mat_lazy_acc(t, D, step), t.level, t.scale)


def conv_bsgs_diagonals(kernels: np.ndarray, chunk: int, ns: int, g: int) -> np.ndarray:
    """D_b = sum_c Mask_c * rot(K_c, chunk b), b < g (slot vectors; rot = left rotation,
    rot(v, k)[s] = v[s + k]).  Written from C18/C19: K_c and Mask_c as conv_kernel_slots /
    conv_mask_slots."""
    n_ch = kernels.shape[0]
    D = np.zeros((g, ns))
    for b in range(g):
        for c in range(n_ch):
            D[b] += conv_mask_slots(c, n_ch, chunk, ns) * np.roll(conv_kernel_slots(kernels[c], chunk, ns),
                                                                  -chunk * b)
    return D


def im2col_conv_bsgs(ctx: OracleContext, ct: OCt, kernels: np.ndarray, bias: np.ndarray | None,
                     chunk: int, g: int, pt_shift: int = 0) -> OCt:
    """The im2col conv (C18/C19) as ONE level (DESIGN.md §3 'conv as a baby-step/giant-step
    product').  The paper's result is out = sum_c Mask_c * sum_{m < n_chunks} rot(ct * K_c, chunk m)
    (+ bias).  Slot products commute with rotations applied to both factors, and Mask_c has
    period C chunks, so for C | g and m = b + g a:
        out = sum_{a < n2} rot(v, chunk g a),  v = sum_{b < g} D_b * rot(ct, chunk b)
    with D_b = conv_bsgs_diagonals.  v is the lazy vec_mat (one ModDown) with the g QP diagonals
    D_b at scale q_l 2^pt_shift and rotation step chunk; rescale once; the giant steps are a
    unit-diagonal rotation sum (rot_sum); + bias."""
    ns = ctx.slots
    n_ch = kernels.shape[0]
    n_chunks = ns // chunk
    assert g % n_ch == 0 and n_chunks % g == 0
    lvl = ct.level
    pscale = _shifted(ctx.q[lvl], pt_shift)
    D = conv_bsgs_diagonals(kernels, chunk, ns, g)
    Dqp = np.stack([ctx.coeffs_to_pt_qp(ctx.encode_coeffs(D[b], pscale)[1], lvl) for b in range(g)])
    v = ctx.rescale(OCt(ctx.vec_mat_lazy_acc(ct, Dqp, chunk), lvl, ct.scale * pscale))
    out = rot_sum(ctx, v, n_chunks // g, chunk * g)
    if bias is not None:
        out = ctx.add_plain(out, ctx.encode(conv_bias_slots(bias, chunk, ns), out.scale, out.level))
    return out


def im2col_conv(ctx: OracleContext, ct: OCt, kernels: np.ndarray, bias: np.ndarray | None,
                chunk: int, kernel_shift: int = 0, mask_shift: int = 0, fold_n1: int = 0) -> OCt:
    """Steps 12 (C18/C19): per channel t_c = rescale(ct * K_c), log2(#chunks)
    rounds t_c += rot(t_c, chunk 2^r); sum_c t_c * Mask_c; rescale; + bias."""
    ns = ctx.slots
    n_ch = kernels.shape[0]
    lvl = ct.level
    ts = []
    for c in range(n_ch):
        K = conv_kernel_slots(kernels[c], chunk, ns)
        t = ctx.rescale(ctx.mul_plain(ct, ctx.encode(K, _shifted(ctx.q[lvl], kernel_shift), lvl)))
        if fold_n1:     # hoisted two-level fold (same sum, different rounding)
            t = hoisted_fold(ctx, t, chunk, fold_n1)
        else:           # log2(#chunks) rotate-and-add rounds
            for step in conv_fold_steps(chunk, ns):
                t = ctx.add(t, ctx.rotate(t, step))
        ts.append(t)
    lvl2 = ts[0].level
    acc = None
    for c in range(n_ch):
        M = conv_mask_slots(c, n_ch, chunk, ns)
        p = ctx.mul_plain(ts[c], ctx.encode(M, _shifted(ctx.q[lvl2], mask_shift), lvl2))
        acc = p if acc is None else ctx.add(acc, p)
    acc = ctx.rescale(acc)
    if bias is not None:
        acc = ctx.add_plain(acc, ctx.encode(conv_bias_slots(bias, chunk, ns), acc.scale,
                                            acc.level))
    return acc



# Scale schedule of the CNN (R1/R2): log2 of the input scale and
# the plaintext-scale shifts relative to the prime each following rescale drops.
CNN_PLAN = dict(in_log2=30, conv_shift=0, mask_shift=-4, fc1_shift=0, fc2_shift=-4)
# With the one-level conv (im2col_conv_bsgs) the input is encrypted one level lower (level L-2,
# the circuit then ends at level 0) and the conv plaintext carries the whole conv shift; the final
# scale is the same 2^22 (2 (2 (30 - 2) - 26 - 4) - 26 - 4 = 22).
CNN_PLAN_BSGS = dict(in_log2=30, conv_shift=-2, fc1_shift=-4, fc2_shift=-4, in_level_drop=1)
CONV_G = 8          # baby steps of the one-level conv: 8 chunks x 8 giant steps
FC1_G = 32          # baby steps of the folded FC1 (vec_mat_bsgs_fold): 32 x 2 groups, fold 4
FC2_M = 16          # folded FC2: outputs padded to 16, 16 diagonals (one group), fold 4


def cnn_rotation_steps(ns: int = 4096, chunk: int = 64, fold_n1: int = 0, conv_g: int = 0,
                       fc_bsgs: bool = False, fc1_g: int = 0) -> list:
    """A-rot: exactly the circuit's steps.  FC: 1..255 (FC2's 1..63 are a subset), or with
    fc_bsgs the baby steps 1..g-1 and giant steps g k2 of FC1 (n 256, g 64) and FC2 (n 64, g 16).
    Conv: the log2 fold steps chunk 2^r, or chunk b and chunk n1 a (hoisted fold, fold_n1), or
    chunk b and chunk g a (one-level conv, conv_g)."""
    if fc_bsgs:
        def bsgs(n, g):         # baby steps 1..g-1, giant steps g k2
            return set(range(1, g)) | {g * k2 for k2 in range(1, (n + g - 1) // g)}
        # FC1 (n 256 -> m 64): plain BSGS with g = n/4, or folded with g = fc1_g over the first m
        # diagonals (giant g k2 < m) and the fold m t < n; FC2 (n 64): g = 16
        fc1 = bsgs(64, fc1_g) | {64, 128, 192} if fc1_g else bsgs(256, 64)
        steps = fc1 | bsgs(64, 16)
    else:
        steps = set(range(1, 256))
    n1 = conv_g or fold_n1
    if n1:
        n2 = ns // chunk // n1
        steps |= {chunk * b for b in range(1, n1)} | {chunk * n1 * a for a in range(1, n2)}
    else:
        steps |= set(conv_fold_steps(chunk, ns))
    return sorted(steps)


def cnn_encrypt_input(ctx: OracleContext, img: np.ndarray, stream_id: int, plan=None) -> OCt:
    plan = plan or CNN_PLAN
    slots = im2col_slots(img, 7, 7, 3, ctx.slots)
    level = ctx.L - 1 - plan.get("in_level_drop", 0)
    return ctx.encrypt(ctx.encode(slots, 2.0 ** plan["in_log2"], level), stream_id)


def cnn_forward(ctx: OracleContext, ct: OCt, w, plan=None, lazy: bool = False, bsgs: bool = False,
                fold_n1: int = 0, conv_g: int = 0, fc1_g: int = 0) -> OCt:
    """The paper's network; lazy=True uses vec_mat_lazy for FC1/FC2, bsgs=True
    vec_mat_bsgs (baby step n/4); fold_n1 > 0 the hoisted conv fold; conv_g > 0 the one-level
    conv (im2col_conv_bsgs, plan CNN_PLAN_BSGS, input from cnn_encrypt_input with that plan);
    fc1_g > 0 (with bsgs) FC1 as vec_mat_bsgs_fold with baby step fc1_g and FC2 folded with its
    outputs padded to FC2_M."""
    plan = plan or (CNN_PLAN_BSGS if conv_g else CNN_PLAN)

    def vm(x, W, b, rep, shift):
        if bsgs:
            return vec_mat_bsgs(ctx, x, W, b, rep, shift, g=W.shape[0] // 4)
        return (vec_mat_lazy if lazy else vec_mat)(ctx, x, W, b, rep, shift)
    if conv_g:
        x = im2col_conv_bsgs(ctx, ct, w.conv_w.reshape(w.conv_w.shape[0], -1), w.conv_b, 64, conv_g,
                             plan["conv_shift"])
    else:
        x = im2col_conv(ctx, ct, w.conv_w.reshape(w.conv_w.shape[0], -1), w.conv_b, 64,
                        plan["conv_shift"], plan["mask_shift"], fold_n1=fold_n1)
    x = ctx.square(x)
    if bsgs and fc1_g:
        x = vec_mat_bsgs_fold(ctx, x, w.fc1_w.T, w.fc1_b, -plan["fc1_shift"], g=fc1_g)
    else:
        x = vm(x, w.fc1_w.T, w.fc1_b, True, -plan["fc1_shift"])
    x = ctx.square(x)
    if bsgs and fc1_g:
        # FC2 with its 10 outputs padded to 16 columns (zero weights and bias): the output is then
        # replicated with period 16 | 64 and folds like FC1 (16 diagonals, fold 4); slots 0..9 hold
        # the logits as before (DESIGN.md §3 'folded FC layers')
        W2, b2 = pad_columns(w.fc2_w.T, w.fc2_b, FC2_M)
        x = vec_mat_bsgs_fold(ctx, x, W2, b2, -plan["fc2_shift"], g=FC2_M)
    else:
        x = vm(x, w.fc2_w.T, w.fc2_b, False, -plan["fc2_shift"])
    return x


def pad_columns(W: np.ndarray, b: np.ndarray, m: int):
    """W (n x m0) and bias (m0) padded with zero columns / entries to m >= m0 outputs."""
    n, m0 = W.shape
    Wp = np.zeros((n, m))
    Wp[:, :m0] = W
    bp = np.zeros(m)
    bp[:m0] = b
    return Wp, bp


# ------------------------------------------------------------ config 5b ---
def deep_chain(ctx: OracleContext, ct: OCt, pts: np.ndarray, rot_steps=(1, 2, 4, 8)) -> OCt:
    """A-cfg5b: for t < len(pts): ct <- rescale(ct * pt_t) with pt_t encoded at the
    scale q_l of the prime the rescale drops (C3, so the ciphertext scale is unchanged); then
    ct <- ct + rot(ct, s) for s in rot_steps."""
    for z in pts:
        lvl = ct.level
        ct = ctx.rescale(ctx.mul_plain(ct, ctx.encode(z, float(ctx.q[lvl]), lvl)))
    for s in rot_steps:
        ct = ctx.add(ct, ctx.rotate(ct, s))
    return ct


# ------------------------------------------- SURVEY 8(f) #2 / #4 circuits ---
def mod_switch(ctx: OracleContext, ct: OCt, level: int) -> OCt:
    """Drop limbs level+1..: the ciphertext mod Q_level decrypts to the same message (|m| < Q_level/2);
    the scale is unchanged."""
    assert level <= ct.level
    return OCt(ct.words[:, : level + 1].copy(), level, ct.scale)


def mul_relin_rescale(ctx: OracleContext, a: OCt, b: OCt) -> OCt:
    """ct x ct at the lower of the two levels: tensor, relinearize, rescale (C14)."""
    lvl = min(a.level, b.level)
    return ctx.rescale(ctx.relinearize(ctx.tensor(mod_switch(ctx, a, lvl), mod_switch(ctx, b, lvl))))


def fold_sum(ctx: OracleContext, ct: OCt, n: int) -> OCt:
    """Rotate-and-add by 1, 2, 4, ... < n (n rounded up to a power of two): slot 0 = sum of slots 0..n-1
    (zeros beyond n)."""
    s = 1
    while s < n:
        ct = ctx.add(ct, ctx.rotate(ct, s))
        s <<= 1
    return ct


def dot(ctx: OracleContext, a: OCt, b: OCt, n: int) -> OCt:
    """Encrypted dot product (Table 5 'dot'): sum_i a_i b_i into slot 0."""
    return fold_sum(ctx, mul_relin_rescale(ctx, a, b), n)


def dot_plain(ctx: OracleContext, a: OCt, z: np.ndarray, n: int) -> OCt:
    """Encrypted x plain dot product (Table 5 'dot_plain'): z encoded at q_l so the rescale restores
    the ciphertext scale."""
    lvl = a.level
    t = ctx.rescale(ctx.mul_plain(a, ctx.encode(z, float(ctx.q[lvl]), lvl)))
    return fold_sum(ctx, t, n)


def powers(ctx: OracleContext, x: OCt, d: int) -> dict:
    """x^1..x^d at minimal depth: x^(2^k) by squaring; x^i = x^(2^k) * x^(i - 2^k), 2^k < i < 2^(k+1)
    (depth ceil(log2 i), PAPER.md:58 'depth-optimal')."""
    P = {1: x}
    k = 1
    while 2 * k <= d:
        P[2 * k] = ctx.square(P[k])
        k *= 2
    for i in range(2, d + 1):
        if i not in P:
            hi = 1 << (i.bit_length() - 1)
            P[i] = mul_relin_rescale(ctx, P[hi], P[i - hi])
    return P


def power(ctx: OracleContext, x: OCt, p: int) -> OCt:
    return powers(ctx, x, p)[p]


def polyval(ctx: OracleContext, x: OCt, coeffs) -> OCt:
    """sum_i c_i x^i (Table 4 'polyval').  Every term c_i x^i (i >= 1) is formed at the
    level l_d of x^d: mod-switch x^i to l_d, multiply by c_i encoded at scale S q_{l_d} / scale(x^i)
    (S = scale of x^d), rescale -> level l_d - 1, scale ~= S.  The tracked scales of the terms agree
    only up to double rounding, so the terms are summed at the first term's scale;
    c_0 is added at that scale."""
    coeffs = [float(c) for c in coeffs]
    d = len(coeffs) - 1
    assert d >= 1
    P = powers(ctx, x, d)
    ld, S = P[d].level, P[d].scale
    acc = None
    for i in range(1, d + 1):
        if coeffs[i] == 0.0:
            continue
        xi = mod_switch(ctx, P[i], ld)
        sc = S * float(ctx.q[ld]) / xi.scale
        t = ctx.rescale(ctx.mul_plain(xi, ctx.encode(np.full(ctx.slots, coeffs[i]), sc, ld)))
        if acc is None:
            acc = t
        else:
            acc = OCt(ctx._pw(0, acc.words, t.words, acc.level), acc.level, acc.scale)
    if coeffs[0] != 0.0:
        acc = ctx.add_plain(acc, ctx.encode(np.full(ctx.slots, coeffs[0]), acc.scale, acc.level))
    return acc


# ------------------------------------------ BSGS vec_mat ---
def bsgs_diagonals(D: np.ndarray, g: int) -> np.ndarray:
    """Baby-step/giant-step diagonals: E[k2][k1] = rot(D_{k1 + g k2}, -g k2) (zero past n), so that
    rot(sum_k1 E[k2][k1] (.) rot(x, k1), g k2) = sum_k1 D_{k1 + g k2} (.) rot(x, k1 + g k2)."""
    n, ns = D.shape
    n2 = -(-n // g)
    E = np.zeros((n2, g, ns))
    for k2 in range(n2):
        for k1 in range(g):
            k = k1 + g * k2
            if k < n:
                E[k2, k1] = np.roll(D[k], g * k2)      # rot(v, -s) = np.roll(v, s)
    return E


def vec_mat_bsgs(ctx: OracleContext, ct: OCt, W: np.ndarray, bias: np.ndarray | None,
                 replicate_out: bool, pt_scale_shift: int = 0, g: int = 64) -> OCt:
    """vec_mat by baby steps k1 < g (one lazy-ModDown accumulation per giant step k2, all sharing the
    rotations of x by k1) and giant steps (a full rotation of each inner sum by g k2), then one
    rescale and the bias: sum_k2 rot(inner_k2, g k2) = sum_k D_k (.) rot(x, k) (C17)."""
    ns = ctx.slots
    D = vecmat_diagonals(W, ns, replicate_out)
    E = bsgs_diagonals(D, g)
    lvl = ct.level
    pscale = _shifted(ctx.q[lvl], -pt_scale_shift)
    acc = None
    for k2 in range(E.shape[0]):
        Eqp = np.stack([ctx.coeffs_to_pt_qp(ctx.encode_coeffs(E[k2, k1], pscale)[1], lvl) for k1 in range(g)])
        inner = OCt(ctx.vec_mat_lazy_acc(ct, Eqp), lvl, ct.scale * pscale)
        if k2:
            inner = ctx.rotate(inner, g * k2)
        acc = inner if acc is None else ctx.add(acc, inner)
    acc = ctx.rescale(acc)
    if bias is not None:
        acc = ctx.add_plain(acc, ctx.encode(vecmat_bias_slots(bias, ns, replicate_out), acc.scale, acc.level))
    return acc


def vec_mat_bsgs_fold(ctx: OracleContext, ct: OCt, W: np.ndarray, bias: np.ndarray | None,
                      pt_scale_shift: int = 0, g: int = 32) -> OCt:
    """vec_mat with replicated output (C17) when m | n: the diagonals are rotation-periodic,
    D_{k + m t}[j] = W[(j + k + m t) mod n][j mod m] = rot(D_k, m t)[j], so
        sum_{k < n} D_k (.) rot(x, k) = sum_{t < n/m} rot(y', m t),  y' = sum_{k < m} D_k (.) rot(x, k)
    (the rectangular "hybrid" diagonal method).  y' by baby-step/giant-step over the first m
    diagonals (g | m, m/g groups, as vec_mat_bsgs), then the n/m-term sum as one unit-diagonal
    rotation sum (rot_sum, one lazy ModDown), one rescale, + bias."""
    n, m = W.shape
    assert n % m == 0 and m % g == 0
    ns = ctx.slots
    D = vecmat_diagonals(W, ns, True)[:m]
    E = bsgs_diagonals(D, g)
    lvl = ct.level
    pscale = _shifted(ctx.q[lvl], -pt_scale_shift)
    acc = None
    for k2 in range(E.shape[0]):
        Eqp = np.stack([ctx.coeffs_to_pt_qp(ctx.encode_coeffs(E[k2, k1], pscale)[1], lvl) for k1 in range(g)])
        inner = OCt(ctx.vec_mat_lazy_acc(ct, Eqp), lvl, ct.scale * pscale)
        if k2:
            inner = ctx.rotate(inner, g * k2)
        acc = inner if acc is None else ctx.add(acc, inner)
    acc = rot_sum(ctx, acc, n // m, m)
    acc = ctx.rescale(acc)
    if bias is not None:
        acc = ctx.add_plain(acc, ctx.encode(vecmat_bias_slots(bias, ns, True), acc.scale, acc.level))
    return acc

"""The paper's encrypted CNN driven through the C-ABI.

conv 7x7 stride 3, 4 kernels (im2col) -> x^2 -> FC 256->64
-> x^2 -> FC 64->10, one image per ciphertext, a batch of images per call.
Every step is a C-ABI call (include/he_ckks.h); this module only sequences
the calls and holds the resident weight plaintexts (encoded once).

Scale schedule: input encoded at 2^30; conv
kernels at q_l (shift 0), masks at q_{l-1} 2^-4, FC1 diagonals at q_l, FC2
diagonals at q_l 2^-4.  With the one-level conv (PLAN_BSGS): input at level
L-2, conv diagonals at q_l 2^-2, FC1 at q_l 2^-4, FC2 at q_l 2^-4.  Rotation keys: exactly the circuit's steps (A-rot).
"""
from __future__ import annotations

import numpy as np

from .ckks import Context, he_im2col_encode_batch

PLAN = dict(in_log2=30, kernel_shift=0, mask_shift=-4, fc1_shift=0, fc2_shift=4)
# One-level conv (he_im2col_conv_bsgs_pt; oracle CNN_PLAN_BSGS): the input is encrypted one level
# lower, the conv plaintext is at q_l 2^conv_shift, FC1 at q_l 2^fc1_shift, FC2 at q_l 2^-fc2_shift.
PLAN_BSGS = dict(in_log2=30, conv_shift=-2, fc1_shift=-4, fc2_shift=4, in_level_drop=1)
CONV_G = 8          # one-level conv: 8 baby steps (chunks) x 8 giant steps
FC1_G = 32          # folded FC1 (he_vec_mat_encode_bsgs_fold): baby step 32, 2 groups, fold 4
FC2_M = 16          # folded FC2: outputs padded to 16 columns, 16 diagonals (one group), fold 4
CHUNK = 64          # next power of two >= 64 windows (C18)
KH = KW = 7
STRIDE = 3


FOLD_N1 = 8        # hoisted conv fold: 8 x 8 chunks


def rotation_steps(ns: int = 4096, chunk: int = CHUNK, fold_n1: int = 0, conv_g: int = 0,
                   fc_bsgs: bool = False, fc1_g: int = 0) -> list:
    """A-rot, exactly the circuit's steps.  FC: 1..255, or with fc_bsgs the baby steps 1..g-1 and
    giant steps g k2 of FC1 (n 256, g 64) and FC2 (n 64, g 16).  Conv: chunk 2^r (log2 fold), or
    chunk b and chunk n1 a (hoisted fold) / chunk b and chunk g a (one-level conv)."""
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
        s = chunk
        while s < ns:
            steps.add(s)
            s <<= 1
    return sorted(steps)


class EncryptedCNN:
    """conv_w [4,1,7,7], conv_b [4], fc1_w [64,256], fc1_b [64], fc2_w [10,64], fc2_b [10] (PyTorch layouts)."""

    def __init__(self, ctx: Context, w, plan=None, lazy: bool = True, bsgs: bool = True, fold_n1: int = 0,
                 conv_g: int = 0, fc1_g: int = 0):
        """FC layers: bsgs (default) = baby-step/giant-step with lazy ModDown (oracle vec_mat_bsgs,
        baby step n/4); lazy = one ModDown per vec_mat (oracle vec_mat_lazy); neither = one ModDown
        per rotation (oracle vec_mat); bsgs with fc1_g > 0 = FC1 folded (oracle vec_mat_bsgs_fold,
        baby step fc1_g).  Conv: conv_g > 0 = the one-level conv (plan PLAN_BSGS), else fold_n1 > 0
        = the hoisted two-level fold, else the paper's log2 fold."""
        self.ctx, self.lazy, self.fold_n1, self.conv_g = ctx, lazy, fold_n1, conv_g
        self.plan = dict(plan or (PLAN_BSGS if conv_g else PLAN))
        self.bsgs = bsgs and lazy
        L = ctx.L
        self.top = L - 1 - self.plan.get("in_level_drop", 0)
        in_scale = 2.0 ** self.plan["in_log2"]
        k = np.asarray(w.conv_w, dtype=np.float64).reshape(w.conv_w.shape[0], KH, KW)
        if conv_g:
            self.conv_d, self.conv_b = ctx.he_im2col_conv_bsgs_encode(
                k, w.conv_b, CHUNK, conv_g, self.plan["conv_shift"], self.top, in_scale)
            s = in_scale * self.conv_d.scale / ctx.q[self.top]
            lvl = self.top - 1
        else:
            self.conv_k, self.conv_m, self.conv_b = ctx.he_im2col_conv_encode(
                k, w.conv_b, CHUNK, self.plan["kernel_shift"], self.plan["mask_shift"], self.top, in_scale)
            # scale after conv and square (tracked exactly like the library does)
            s = in_scale * self.conv_k.scale / ctx.q[self.top]
            s = s * self.conv_m.scale / ctx.q[self.top - 1]
            lvl = self.top - 2
        s = s * s / ctx.q[lvl]          # square: tensor, relin, rescale
        lvl -= 1
        fold = bool(self.bsgs and fc1_g)
        g1 = fc1_g if fold else (np.asarray(w.fc1_w).shape[1] // 4 if self.bsgs else 0)
        self.fc1_d, self.fc1_b = ctx.he_vec_mat_encode(np.asarray(w.fc1_w).T, w.fc1_b, True,
                                                       -self.plan["fc1_shift"], lvl, s, lazy=lazy, bsgs_g=g1,
                                                       fold=fold)
        s = s * self.fc1_d.scale / ctx.q[lvl]
        lvl -= 1
        s = s * s / ctx.q[lvl]
        lvl -= 1
        if fold:    # FC2 outputs padded to FC2_M zero columns: replicated with period 16, folded
            W2 = np.zeros((np.asarray(w.fc2_w).shape[1], FC2_M))
            W2[:, :np.asarray(w.fc2_w).shape[0]] = np.asarray(w.fc2_w).T
            b2 = np.zeros(FC2_M)
            b2[:len(w.fc2_b)] = w.fc2_b
            self.fc2_d, self.fc2_b = ctx.he_vec_mat_encode(W2, b2, True, self.plan["fc2_shift"], lvl, s,
                                                           lazy=lazy, bsgs_g=FC2_M, fold=True)
        else:
            g2 = np.asarray(w.fc2_w).shape[1] // 4 if self.bsgs else 0
            self.fc2_d, self.fc2_b = ctx.he_vec_mat_encode(np.asarray(w.fc2_w).T, w.fc2_b, False,
                                                           self.plan["fc2_shift"], lvl, s, lazy=lazy, bsgs_g=g2)
        self.n_out = int(np.asarray(w.fc2_w).shape[0])

    def im2col(self, imgs: np.ndarray) -> np.ndarray:
        return he_im2col_encode_batch(imgs, KH, KW, STRIDE, self.ctx.slots)

    def encrypt(self, imgs: np.ndarray, stream_id: int = 0):
        """Client side: im2col (host) -> encode -> encrypt, images [B][28][28]."""
        slots = self.im2col(np.asarray(imgs, dtype=np.float64))
        return self.ctx.he_encode_encrypt(slots, 2.0 ** self.plan["in_log2"], self.top, stream_id)

    def forward(self, ct):
        """Server side: conv -> square -> FC1 -> square -> FC2."""
        c = self.ctx
        if self.conv_g:
            x = c.he_im2col_conv_bsgs_pt(ct, self.conv_d, self.conv_b, CHUNK, self.conv_g)
        elif self.fold_n1:
            x = c.he_im2col_conv_hoisted_pt(ct, self.conv_k, self.conv_m, self.conv_b, CHUNK, self.fold_n1)
        else:
            x = c.he_im2col_conv_pt(ct, self.conv_k, self.conv_m, self.conv_b, CHUNK)
        x = c.he_square(x)
        x = c.he_vec_mat_pt(x, self.fc1_d, self.fc1_b)
        x = c.he_square(x)
        return c.he_vec_mat_pt(x, self.fc2_d, self.fc2_b)

    def decrypt(self, ct) -> np.ndarray:
        """Client side: decrypt -> decode -> the first n_out slots per image."""
        return self.ctx.he_decode(self.ctx.he_decrypt(ct), self.n_out)

"""Python harness of the CPU oracle — TEST INFRASTRUCTURE ONLY.

Loads ``oracle/liboracle.so`` (built from ``oracle/ckks_oracle.cpp`` by
``__graft_entry__.build()`` or :func:`build_oracle`) with ctypes and wraps it
with numpy arrays.  The algorithms are SURVEY.md §8(c) "Oracle algorithm, step
by step" (CKKS of Cheon et al., which TenSEAL uses through SEAL).

The only arithmetic written here (not in C++) is the CDT table of convention
C11, computed with mpmath at 60 significant digits, and the ciphertext scale
bookkeeping (exact double products / quotients, C14).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ckks_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

U64P = ctypes.POINTER(ctypes.c_uint64)
I64P = ctypes.POINTER(ctypes.c_int64)
U32P = ctypes.POINTER(ctypes.c_uint32)
DP = ctypes.POINTER(ctypes.c_double)
IP = ctypes.POINTER(ctypes.c_int)

SIGMA = 3.2      # C11 / BASELINE configs: "error discrete Gaussian sigma=3.2"
CDT_BOUND = 19   # floor(6 sigma)


def build_oracle(force: bool = False) -> str:
    """Compile the oracle with plain g++ (no CUDA, no shared headers)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-pthread",
                               _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build_oracle())
        L.orc_create.restype = ctypes.c_void_p
        L.orc_create.argtypes = [ctypes.c_int, ctypes.c_int, IP, ctypes.c_int, ctypes.c_uint64,
                                 U64P, ctypes.c_int]
        L.orc_destroy.argtypes = [ctypes.c_void_p]
        for name in ["orc_dims"]:
            getattr(L, name).argtypes = [ctypes.c_void_p, IP]
        L.orc_primes.argtypes = [ctypes.c_void_p, U64P]
        L.orc_psis.argtypes = [ctypes.c_void_p, U64P]
        L.orc_select_primes.argtypes = [ctypes.c_int, ctypes.c_int, IP, U64P]
        L.orc_min_psi.restype = ctypes.c_uint64
        L.orc_min_psi.argtypes = [ctypes.c_uint64, ctypes.c_int]
        L.orc_is_prime.argtypes = [ctypes.c_uint64]
        L.orc_ntt_raw.argtypes = [U64P, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64]
        L.orc_intt_raw.argtypes = [U64P, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64]
        L.orc_philox.argtypes = [U32P, U32P, U32P]
        L.orc_ntt.argtypes = [ctypes.c_void_p, ctypes.c_int, U64P]
        L.orc_intt.argtypes = [ctypes.c_void_p, ctypes.c_int, U64P]
        L.orc_sample_ternary.argtypes = [ctypes.c_void_p, ctypes.c_uint64, I64P]
        L.orc_sample_cdt.argtypes = [ctypes.c_void_p, ctypes.c_uint64, I64P]
        L.orc_sample_uniform.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, U64P]
        L.orc_sid.restype = ctypes.c_uint64
        L.orc_sid.argtypes = [ctypes.c_uint64] * 3
        L.orc_galois_elt.restype = ctypes.c_uint64
        L.orc_galois_elt.argtypes = [ctypes.c_void_p, ctypes.c_int]
        L.orc_keygen.argtypes = [ctypes.c_void_p, IP, ctypes.c_int, ctypes.c_int]
        L.orc_sk.argtypes = [ctypes.c_void_p, I64P, U64P]
        L.orc_pk.argtypes = [ctypes.c_void_p, U64P]
        L.orc_relin_key.argtypes = [ctypes.c_void_p, U64P]
        L.orc_galois_key.argtypes = [ctypes.c_void_p, ctypes.c_int, U64P]
        L.orc_encode.argtypes = [ctypes.c_void_p, DP, ctypes.c_int, ctypes.c_double, DP, I64P]
        L.orc_coeffs_to_pt.argtypes = [ctypes.c_void_p, I64P, ctypes.c_int, U64P]
        L.orc_decode.argtypes = [ctypes.c_void_p, U64P, ctypes.c_int, ctypes.c_double,
                                 ctypes.c_int, DP, DP]
        L.orc_encrypt.argtypes = [ctypes.c_void_p, U64P, ctypes.c_int, ctypes.c_uint64, U64P]
        L.orc_encrypt_symmetric.argtypes = [ctypes.c_void_p, U64P, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                            U64P]
        L.orc_decrypt.argtypes = [ctypes.c_void_p, U64P, ctypes.c_int, ctypes.c_int, U64P]
        L.orc_pointwise.argtypes = [ctypes.c_void_p, ctypes.c_int, U64P, U64P, ctypes.c_int,
                                    ctypes.c_int, ctypes.c_int, U64P]
        L.orc_tensor.argtypes = [ctypes.c_void_p, U64P, U64P, ctypes.c_int, U64P]
        L.orc_keyswitch.argtypes = [ctypes.c_void_p, U64P, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, U64P]
        L.orc_relinearize.argtypes = [ctypes.c_void_p, U64P, ctypes.c_int, U64P]
        L.orc_rotate.argtypes = [ctypes.c_void_p, U64P, ctypes.c_int, ctypes.c_int, U64P]
        L.orc_automorph_ntt.argtypes = [ctypes.c_void_p, U64P, ctypes.c_int, ctypes.c_uint64,
                                        U64P]
        L.orc_rescale.argtypes = [ctypes.c_void_p, U64P, ctypes.c_int, ctypes.c_int, U64P]
        L.orc_vec_mat_lazy.argtypes = [ctypes.c_void_p, U64P, ctypes.c_int, U64P, ctypes.c_int, U64P]
        L.orc_vec_mat_lazy_step.argtypes = [ctypes.c_void_p, U64P, ctypes.c_int, U64P, ctypes.c_int, ctypes.c_int,
                                            U64P]
        L.orc_coeffs_to_pt_qp.argtypes = [ctypes.c_void_p, I64P, ctypes.c_int, U64P]
        L.orc_divround.argtypes = [ctypes.c_void_p, IP, ctypes.c_int, IP, ctypes.c_int, U64P,
                                   U64P, U64P]
        _lib = L
    return _lib


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint64)


def cdt_table(sigma: float = SIGMA, bound: int = CDT_BOUND) -> np.ndarray:
    """C11: T[k] = floor(2^63 * Pr(|X| <= k)), X discrete Gaussian with
    rho(x) = exp(-x^2 / (2 sigma^2)) on |x| <= bound, in 60-digit arithmetic."""
    import mpmath
    with mpmath.workdps(60):
        s = mpmath.mpf(str(sigma))
        rho = [mpmath.e ** (-(mpmath.mpf(x) ** 2) / (2 * s * s)) for x in range(bound + 1)]
        total = rho[0] + 2 * sum(rho[1:])
        out = []
        run = mpmath.mpf(0)
        for k in range(bound + 1):
            run += rho[0] if k == 0 else 2 * rho[k]
            out.append(int(mpmath.floor(mpmath.mpf(2) ** 63 * run / total)))
    out[-1] = 1 << 63   # Pr(|X| <= bound) = 1 exactly
    return np.array(out, dtype=np.uint64)


# C9 purposes
P_S, P_PK_A, P_PK_E, P_RLK_A, P_RLK_E, P_GK_A, P_GK_E, P_ENC_V, P_ENC_E0, P_ENC_E1 = range(1, 11)


def sid(purpose: int, obj: int, prime: int) -> int:
    return (purpose << 56) | (obj << 16) | prime


@dataclass
class OCt:
    """Oracle ciphertext: words [size][level+1][N] (NTT domain, C5)."""
    words: np.ndarray
    level: int
    scale: float

    @property
    def size(self) -> int:
        return self.words.shape[0]


@dataclass
class OPt:
    words: np.ndarray   # [level+1][N]
    level: int
    scale: float


class OracleContext:
    """Oracle CKKS context: params (C2/C4), keys (C9–C12), scheme ops."""

    def __init__(self, logN: int, bits, n_special: int, seed: int):
        self.lib = lib()
        bits = list(bits)
        b = (ctypes.c_int * len(bits))(*bits)
        self.cdt = cdt_table()
        self.h = self.lib.orc_create(logN, len(bits), b, n_special, seed,
                                     _p(self.cdt, U64P), len(self.cdt))
        if not self.h:
            raise ValueError("oracle: invalid parameters")
        dims = (ctypes.c_int * 4)()
        self.lib.orc_dims(self.h, dims)
        self.logN, self.N, self.L, self.K = dims[0], dims[1], dims[2], dims[3]
        self.seed = seed
        self.primes = np.zeros(self.L + self.K, dtype=np.uint64)
        self.lib.orc_primes(self.h, _p(self.primes, U64P))
        self.psis = np.zeros(self.L + self.K, dtype=np.uint64)
        self.lib.orc_psis(self.h, _p(self.psis, U64P))
        self.q = [int(x) for x in self.primes]
        self.steps: list[int] = []

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.orc_destroy(self.h)
        except Exception:
            pass

    @property
    def slots(self) -> int:
        return self.N // 2

    # ------------------------------------------------------------ ring ---
    def ntt(self, t: int, a) -> np.ndarray:
        a = _u64(a).copy()
        self.lib.orc_ntt(self.h, t, _p(a, U64P))
        return a

    def intt(self, t: int, a) -> np.ndarray:
        a = _u64(a).copy()
        self.lib.orc_intt(self.h, t, _p(a, U64P))
        return a

    def galois_elt(self, k: int) -> int:
        return int(self.lib.orc_galois_elt(self.h, k))

    def automorph_ntt(self, a, t: int, g: int) -> np.ndarray:
        a = _u64(a)
        out = np.zeros(self.N, dtype=np.uint64)
        self.lib.orc_automorph_ntt(self.h, _p(a, U64P), t, g, _p(out, U64P))
        return out

    # -------------------------------------------------------- sampling ---
    def sample_ternary(self, s: int) -> np.ndarray:
        out = np.zeros(self.N, dtype=np.int64)
        self.lib.orc_sample_ternary(self.h, s, _p(out, I64P))
        return out

    def sample_cdt(self, s: int) -> np.ndarray:
        out = np.zeros(self.N, dtype=np.int64)
        self.lib.orc_sample_cdt(self.h, s, _p(out, I64P))
        return out

    def sample_uniform(self, s: int, t: int) -> np.ndarray:
        out = np.zeros(self.N, dtype=np.uint64)
        self.lib.orc_sample_uniform(self.h, s, t, _p(out, U64P))
        return out

    # ------------------------------------------------------------ keys ---
    def keygen(self, steps=(), nthreads: int | None = None) -> None:
        steps = [int(s) for s in steps]
        for s in steps:
            if s == 0 or abs(s) > self.slots:
                raise ValueError(f"invalid rotation step {s}")
        arr = (ctypes.c_int * max(1, len(steps)))(*steps)
        nthreads = nthreads or os.cpu_count() or 1
        if self.lib.orc_keygen(self.h, arr, len(steps), nthreads) != 0:
            raise RuntimeError("oracle keygen failed")
        self.steps = steps

    def secret_key(self):
        c = np.zeros(self.N, dtype=np.int64)
        w = np.zeros((self.L + self.K, self.N), dtype=np.uint64)
        self.lib.orc_sk(self.h, _p(c, I64P), _p(w, U64P))
        return c, w

    def public_key(self) -> np.ndarray:
        out = np.zeros((2, self.L, self.N), dtype=np.uint64)
        self.lib.orc_pk(self.h, _p(out, U64P))
        return out

    def relin_key(self) -> np.ndarray:
        out = np.zeros((self.L, 2, self.L + self.K, self.N), dtype=np.uint64)
        self.lib.orc_relin_key(self.h, _p(out, U64P))
        return out

    def galois_key(self, step: int) -> np.ndarray:
        out = np.zeros((self.L, 2, self.L + self.K, self.N), dtype=np.uint64)
        if self.lib.orc_galois_key(self.h, step, _p(out, U64P)) != 0:
            raise KeyError(step)
        return out

    # ---------------------------------------------------- encode/decode ---
    def encode_coeffs(self, z, scale: float):
        """C6/C7: returns (pre-rounding float values, int64 coefficients)."""
        z = np.ascontiguousarray(z, dtype=np.float64)
        if z.size > self.slots:
            raise ValueError("too many values")
        pre = np.zeros(self.N, dtype=np.float64)
        m = np.zeros(self.N, dtype=np.int64)
        rc = self.lib.orc_encode(self.h, _p(z, DP), z.size, float(scale), _p(pre, DP), _p(m, I64P))
        if rc != 0:
            raise OverflowError("encode: |scale*z| >= 2^62")
        return pre, m

    def coeffs_to_pt(self, m, level: int, scale: float) -> OPt:
        m = np.ascontiguousarray(m, dtype=np.int64)
        out = np.zeros((level + 1, self.N), dtype=np.uint64)
        self.lib.orc_coeffs_to_pt(self.h, _p(m, I64P), level, _p(out, U64P))
        return OPt(out, level, float(scale))

    def coeffs_to_pt_qp(self, m, level: int) -> np.ndarray:
        """NTT words of signed coefficients on data limbs 0..level then the K special limbs."""
        m = np.ascontiguousarray(m, dtype=np.int64)
        out = np.zeros((level + 1 + self.K, self.N), dtype=np.uint64)
        self.lib.orc_coeffs_to_pt_qp(self.h, _p(m, I64P), level, _p(out, U64P))
        return out

    def vec_mat_lazy_acc(self, ct: OCt, diags_qp: np.ndarray, step: int = 1) -> np.ndarray:
        """sum_k D_k (.) rot(ct, k step) with one ModDown (see ckks_oracle.cpp orc_vec_mat_lazy);
        diags_qp: [n][level+1+K][N]. Returns [2][level+1][N] (not rescaled)."""
        d = _u64(diags_qp)
        w = _u64(ct.words)
        out = np.zeros((2, ct.level + 1, self.N), dtype=np.uint64)
        if self.lib.orc_vec_mat_lazy_step(self.h, _p(w, U64P), ct.level, _p(d, U64P), d.shape[0], step,
                                          _p(out, U64P)) != 0:
            raise KeyError("missing Galois key")
        return out

    def encode(self, z, scale: float, level: int) -> OPt:
        _, m = self.encode_coeffs(z, scale)
        return self.coeffs_to_pt(m, level, scale)

    def decode(self, pt: OPt, n: int | None = None, want_coeffs: bool = False):
        n = self.slots if n is None else n
        w = _u64(pt.words)
        z = np.zeros(max(n, 1), dtype=np.float64)
        co = np.zeros(self.N, dtype=np.float64) if want_coeffs else None
        self.lib.orc_decode(self.h, _p(w, U64P), pt.level, float(pt.scale), n, _p(z, DP),
                            _p(co, DP) if co is not None else None)
        z = z[:n]
        return (z, co) if want_coeffs else z

    # ------------------------------------------------------ encryption ---
    def encrypt(self, pt: OPt, stream_id: int) -> OCt:
        out = np.zeros((2, pt.level + 1, self.N), dtype=np.uint64)
        w = _u64(pt.words)
        self.lib.orc_encrypt(self.h, _p(w, U64P), pt.level, stream_id, _p(out, U64P))
        return OCt(out, pt.level, pt.scale)

    def encrypt_symmetric(self, pt: OPt, stream_id: int, a_seed: int) -> OCt:
        """c1 = a = Uniform(a_seed, (SYM_A, stream_id, i)), c0 = -a s + e + m."""
        out = np.zeros((2, pt.level + 1, self.N), dtype=np.uint64)
        w = _u64(pt.words)
        self.lib.orc_encrypt_symmetric(self.h, _p(w, U64P), pt.level, stream_id, a_seed, _p(out, U64P))
        return OCt(out, pt.level, pt.scale)

    def decrypt(self, ct: OCt) -> OPt:
        out = np.zeros((ct.level + 1, self.N), dtype=np.uint64)
        w = _u64(ct.words)
        self.lib.orc_decrypt(self.h, _p(w, U64P), ct.size, ct.level, _p(out, U64P))
        return OPt(out, ct.level, ct.scale)

    # ------------------------------------------------------- arithmetic ---
    def _pw(self, op, a: np.ndarray, b: np.ndarray | None, level: int) -> np.ndarray:
        a = _u64(a)
        b = _u64(b) if b is not None else a
        pa = a.shape[0]
        pb = b.shape[0] if b.ndim == 3 else 1
        out = np.zeros_like(a)
        self.lib.orc_pointwise(self.h, op, _p(a, U64P), _p(b, U64P), pa, pb, level, _p(out, U64P))
        return out

    @staticmethod
    def _check(a: OCt, b) -> None:
        if a.level != b.level:
            raise ValueError("level mismatch")
        if a.scale != b.scale:
            raise ValueError("scale mismatch")

    def add(self, a: OCt, b: OCt) -> OCt:
        self._check(a, b)
        if a.size != b.size:
            raise ValueError("size mismatch")
        return OCt(self._pw(0, a.words, b.words, a.level), a.level, a.scale)

    def sub(self, a: OCt, b: OCt) -> OCt:
        self._check(a, b)
        return OCt(self._pw(1, a.words, b.words, a.level), a.level, a.scale)

    def negate(self, a: OCt) -> OCt:
        return OCt(self._pw(2, a.words, None, a.level), a.level, a.scale)

    def add_plain(self, a: OCt, p: OPt) -> OCt:
        self._check(a, p)
        out = a.words.copy()
        out[0] = self._pw(0, a.words[:1], p.words[None], a.level)[0]
        return OCt(out, a.level, a.scale)

    def mul_plain(self, a: OCt, p: OPt) -> OCt:
        if a.level != p.level:
            raise ValueError("level mismatch")
        out = self._pw(3, a.words, p.words[None], a.level)
        return OCt(out, a.level, a.scale * p.scale)

    def tensor(self, a: OCt, b: OCt) -> OCt:
        if a.level != b.level:
            raise ValueError("level mismatch")
        out = np.zeros((3, a.level + 1, self.N), dtype=np.uint64)
        x, y = _u64(a.words), _u64(b.words)
        self.lib.orc_tensor(self.h, _p(x, U64P), _p(y, U64P), a.level, _p(out, U64P))
        return OCt(out, a.level, a.scale * b.scale)

    def keyswitch(self, d: np.ndarray, level: int, step: int | None) -> np.ndarray:
        d = _u64(d)
        u = np.zeros((2, level + 1, self.N), dtype=np.uint64)
        rc = self.lib.orc_keyswitch(self.h, _p(d, U64P), level, 0 if step is None else 1,
                                    0 if step is None else step, _p(u, U64P))
        if rc != 0:
            raise KeyError(step)
        return u

    def relinearize(self, a: OCt) -> OCt:
        assert a.size == 3
        out = np.zeros((2, a.level + 1, self.N), dtype=np.uint64)
        w = _u64(a.words)
        self.lib.orc_relinearize(self.h, _p(w, U64P), a.level, _p(out, U64P))
        return OCt(out, a.level, a.scale)

    def rotate(self, a: OCt, step: int) -> OCt:
        if step % self.slots == 0 and step not in self.steps:
            return OCt(a.words.copy(), a.level, a.scale)
        out = np.zeros((2, a.level + 1, self.N), dtype=np.uint64)
        w = _u64(a.words)
        if self.lib.orc_rotate(self.h, _p(w, U64P), a.level, step, _p(out, U64P)) != 0:
            raise KeyError(f"missing Galois key for step {step}")
        return OCt(out, a.level, a.scale)

    def rescale(self, a: OCt) -> OCt:
        if a.level < 1:
            raise ValueError("level exhausted")
        out = np.zeros((a.size, a.level, self.N), dtype=np.uint64)
        w = _u64(a.words)
        self.lib.orc_rescale(self.h, _p(w, U64P), a.size, a.level, _p(out, U64P))
        return OCt(out, a.level - 1, a.scale / self.q[a.level])

    def square(self, a: OCt) -> OCt:
        """C14: tensor -> relinearize -> rescale."""
        return self.rescale(self.relinearize(self.tensor(a, a)))

    def divround(self, keep, drop, x_keep: np.ndarray, x_drop: np.ndarray) -> np.ndarray:
        k = (ctypes.c_int * len(keep))(*keep)
        d = (ctypes.c_int * len(drop))(*drop)
        xk, xd = _u64(x_keep), _u64(x_drop)
        out = np.zeros((len(keep), self.N), dtype=np.uint64)
        self.lib.orc_divround(self.h, k, len(keep), d, len(drop), _p(xk, U64P), _p(xd, U64P),
                              _p(out, U64P))
        return out


def philox4x32_10(ctr, key) -> np.ndarray:
    c = (ctypes.c_uint32 * 4)(*[int(x) & 0xffffffff for x in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(x) & 0xffffffff for x in key])
    o = (ctypes.c_uint32 * 4)()
    lib().orc_philox(c, k, o)
    return np.array(list(o), dtype=np.uint32)

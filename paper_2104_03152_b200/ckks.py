"""Thin Python binding of the C-ABI in include/he_ckks.h (argument marshalling only).

Every function here is the C function of the same name: it converts numpy
arrays / torch tensors to pointers, calls libhe_ckks.so and raises HEError on a
non-zero status.  No arithmetic of the method happens in Python, and there is no
CPU fallback: if the shared library or a CUDA device is missing, the calls fail.

Small handle classes (Context, Plaintext, Ciphertext) own the C handles and free
them on garbage collection.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# HE_CKKS_LIB: load another in-tree build of the same library (A/B experiments only)
LIB_PATH = os.environ.get("HE_CKKS_LIB") or os.path.join(_HERE, "libhe_ckks.so")

STATUS = {
    0: "OK", 1: "INVALID_PARAMS", 2: "PARAM_MISMATCH", 3: "DOMAIN_MISMATCH", 4: "LEVEL_MISMATCH",
    5: "SCALE_MISMATCH", 6: "LEVEL_EXHAUSTED", 7: "SCALE_OVERFLOW", 8: "MISSING_KEY",
    9: "MISSING_GALOIS_KEY", 10: "INVALID_ROTATION", 11: "TOO_MANY_VALUES", 12: "SHAPE_MISMATCH",
    13: "LAYOUT_MISMATCH", 14: "REPLICATION_EXHAUSTED", 15: "CUDA_ERROR", 16: "OUT_OF_MEMORY",
    17: "INVALID_ARGUMENT",
}


class HEError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.name = STATUS.get(code, str(code))


class he_params(C.Structure):
    _fields_ = [("log2N", C.c_int), ("n_primes", C.c_int), ("bits", C.POINTER(C.c_int)),
                ("n_special", C.c_int), ("scale_log2", C.c_double), ("dnum", C.c_int)]


VP = C.c_void_p
VPP = C.POINTER(C.c_void_p)
U64P = C.POINTER(C.c_uint64)
I64P = C.POINTER(C.c_int64)
DP = C.POINTER(C.c_double)
SZ = C.c_size_t

# name -> argtypes (restype he_status unless listed in _RESTYPES)
_SIGS = {
    "he_context_create": [C.POINTER(he_params), C.c_uint64, VPP],
    "he_context_free": [VP],
    "he_context_info": [VP, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)],
    "he_context_primes": [VP, U64P, U64P],
    "he_context_cdt": [VP, U64P],
    "he_set_stream": [VP, VP],
    "he_sync": [VP],
    "he_keygen": [VP, C.POINTER(C.c_int32), SZ],
    "he_drop_secret_key": [VP],
    "he_make_public": [VP, VPP],
    "he_set_allocator": [VP, VP, VP, VP],
    "he_pt_to_int_coeffs": [VP, VP, I64P],
    "he_add_inplace": [VP, VP, VP],
    "he_sub_inplace": [VP, VP, VP],
    "he_add_plain_inplace": [VP, VP, VP],
    "he_mul_plain_inplace": [VP, VP, VP],
    "he_rescale_inplace": [VP, VP],
    "he_rotate_inplace": [VP, VP, C.c_int32],
    "he_square_inplace": [VP, VP],
    "he_encode": [VP, DP, SZ, SZ, C.c_double, C.c_int, VPP],
    "he_encode_device": [VP, VP, SZ, SZ, C.c_double, C.c_int, VPP],
    "he_encode_unrounded": [VP, DP, SZ, SZ, C.c_double, DP],
    "he_decode": [VP, VP, DP, SZ],
    "he_decode_device": [VP, VP, VP, SZ],
    "he_decode_async": [VP, VP, VP, SZ],
    "he_encrypt": [VP, VP, C.c_uint64, VPP],
    "he_encode_encrypt": [VP, DP, SZ, SZ, C.c_double, C.c_int, C.c_uint64, VPP],
    "he_encode_encrypt_device": [VP, VP, SZ, SZ, C.c_double, C.c_int, C.c_uint64, VPP],
    "he_encrypt_symmetric": [VP, VP, C.c_uint64, C.c_uint64, VPP],
    "he_decrypt": [VP, VP, VPP],
    "he_add": [VP, VP, VP, VPP],
    "he_sub": [VP, VP, VP, VPP],
    "he_negate": [VP, VP, VPP],
    "he_add_plain": [VP, VP, VP, VPP],
    "he_mul_plain": [VP, VP, VP, VPP],
    "he_mul": [VP, VP, VP, VPP],
    "he_square": [VP, VP, VPP],
    "he_relinearize": [VP, VP, VPP],
    "he_rescale": [VP, VP, VPP],
    "he_rotate": [VP, VP, C.c_int32, VPP],
    "he_im2col_encode": [DP, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, SZ, DP, C.POINTER(C.c_int),
                         C.POINTER(C.c_int)],
    "he_mod_switch_to": [VP, VP, C.c_int, VPP],
    "he_dot": [VP, VP, VP, C.c_int, VPP],
    "he_dot_plain": [VP, VP, DP, SZ, C.c_int, VPP],
    "he_power": [VP, VP, C.c_int, VPP],
    "he_polyval": [VP, VP, DP, C.c_int, VPP],
    "he_im2col_encode_batch": [DP, SZ, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, SZ, DP],
    "he_im2col_conv": [VP, VP, DP, C.c_int, C.c_int, C.c_int, DP, C.c_int, C.c_int, C.c_int, VPP],
    "he_vec_mat": [VP, VP, DP, C.c_int, C.c_int, DP, C.c_int, C.c_int, VPP],
    "he_vec_mat_pt": [VP, VP, VP, VP, VPP],
    "he_im2col_conv_pt": [VP, VP, VP, VP, VP, C.c_int, VPP],
    "he_im2col_conv_hoisted_pt": [VP, VP, VP, VP, VP, C.c_int, C.c_int, VPP],
    "he_im2col_conv_bsgs_pt": [VP, VP, VP, VP, C.c_int, C.c_int, VPP],
    "he_im2col_conv_bsgs_encode": [VP, DP, C.c_int, C.c_int, C.c_int, DP, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.c_double, VPP, VPP],
    "he_vec_mat_encode": [VP, DP, C.c_int, C.c_int, DP, C.c_int, C.c_int, C.c_int, C.c_double, VPP, VPP],
    "he_im2col_conv_encode": [VP, DP, C.c_int, C.c_int, C.c_int, DP, C.c_int, C.c_int, C.c_int, C.c_int,
                              C.c_double, VPP, VPP, VPP],
    "he_free_plaintext": [VP],
    "he_free_ciphertext": [VP],
    "he_ct_info": [VP, C.POINTER(SZ), C.POINTER(C.c_int), C.POINTER(C.c_int), DP],
    "he_pt_info": [VP, C.POINTER(SZ), C.POINTER(C.c_int), DP],
    "he_ct_device_ptr": [VP, C.POINTER(U64P)],
    "he_pt_device_ptr": [VP, C.POINTER(U64P)],
    "he_ct_export_words": [VP, VP, VP, C.c_int],
    "he_ct_import_words": [VP, VP, C.c_int, SZ, C.c_int, C.c_int, C.c_double, VPP],
    "he_pt_export_words": [VP, VP, VP, C.c_int],
    "he_pt_import_words": [VP, VP, C.c_int, SZ, C.c_int, C.c_double, VPP],
    "he_pt_from_int_coeffs": [VP, I64P, SZ, C.c_double, C.c_int, VPP],
    "he_pt_from_int_coeffs_qp": [VP, I64P, SZ, C.c_double, C.c_int, VPP],
    "he_pt_limbs": [VP, C.POINTER(C.c_int)],
    "he_vec_mat_encode_bsgs": [VP, DP, C.c_int, C.c_int, DP, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                               VPP, VPP],
    "he_vec_mat_bsgs_pt": [VP, VP, VP, C.c_int, VP, VPP],
    "he_vec_mat_bsgs_fold_pt": [VP, VP, VP, C.c_int, C.c_int, C.c_int, VP, VPP],
    "he_vec_mat_encode_bsgs_fold": [VP, DP, C.c_int, C.c_int, DP, C.c_int, C.c_int, C.c_double, C.c_int,
                                    VPP, VPP],
    "he_vec_mat_encode_lazy": [VP, DP, C.c_int, C.c_int, DP, C.c_int, C.c_int, C.c_int, C.c_double, VPP, VPP],
    "he_key_export": [VP, C.c_int, C.c_int32, U64P],
    "he_key_words": [VP, C.c_int],
    "he_key_bytes": [VP],
    "he_ct_serialized_size": [VP, VP, C.POINTER(SZ)],
    "he_ct_serialize": [VP, VP, VP, C.c_int],
    "he_ct_serialized_size_seeded": [VP, VP, C.POINTER(SZ)],
    "he_ct_serialize_seeded": [VP, VP, VP, C.c_int],
    "he_ct_deserialize": [VP, VP, C.c_int, SZ, VPP],
    "he_ntt_forward": [VP, VP, SZ, C.c_int],
    "he_ntt_inverse": [VP, VP, SZ, C.c_int],
    "he_modmul": [VP, VP, VP, VP, SZ, C.c_int],
    "he_ntt_mul_intt": [VP, VP, VP, VP, SZ, C.c_int],
    "he_launch_count": [VP],
    "he_graph_begin": [VP],
    "he_graph_end": [VP, VPP],
    "he_graph_launch": [VP],
    "he_graph_kernels": [VP],
    "he_graph_free": [VP],
    "he_profile_enable": [VP, C.c_int],
    "he_profile_read": [VP, C.c_char_p, SZ],
    "he_last_error": [],
}
_RESTYPES = {"he_key_words": C.c_size_t, "he_key_bytes": C.c_size_t, "he_launch_count": C.c_uint64, "he_graph_kernels": C.c_uint64, "he_last_error": C.c_char_p}

_lib = None


def lib():
    """Load libhe_ckks.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2104_03152_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = _RESTYPES.get(name, C.c_int)
        _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


def _check(rc: int):
    if rc != 0:
        raise HEError(rc, lib().he_last_error().decode())


def _ptr(a):
    """Raw data pointer of a numpy array or torch tensor."""
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


def _is_dev(a) -> int:
    return int(hasattr(a, "is_cuda") and a.is_cuda)


# ---------------------------------------------------------------- handles ---
class Graph:
    """A recorded call sequence (he_graph_*): launch() enqueues one replay on the context stream."""

    def __init__(self, ctx, h):
        self.ctx, self.h = ctx, h

    def launch(self) -> None:
        _check(lib().he_graph_launch(self.h))

    @property
    def kernels(self) -> int:
        return int(lib().he_graph_kernels(self.h))

    def free(self) -> None:
        if self.h:
            _check(lib().he_graph_free(self.h))
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Plaintext:
    def __init__(self, ctx: "Context", h):
        self.ctx, self.h = ctx, h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.he_free_plaintext(self.h)
            self.h = None

    def info(self):
        B, lvl, sc = SZ(), C.c_int(), C.c_double()
        _check(lib().he_pt_info(self.h, C.byref(B), C.byref(lvl), C.byref(sc)))
        return B.value, lvl.value, sc.value

    @property
    def B(self): return self.info()[0]

    @property
    def level(self): return self.info()[1]

    @property
    def scale(self): return self.info()[2]

    @property
    def limbs(self) -> int:
        n = C.c_int()
        _check(lib().he_pt_limbs(self.h, C.byref(n)))
        return n.value

    def words(self) -> np.ndarray:
        B = self.info()[0]
        out = np.zeros((B, self.limbs, self.ctx.N), dtype=np.uint64)
        _check(lib().he_pt_export_words(self.ctx.h, self.h, _ptr(out), 0))
        return out


class Ciphertext:
    def __init__(self, ctx: "Context", h):
        self.ctx, self.h = ctx, h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.he_free_ciphertext(self.h)
            self.h = None

    def info(self):
        B, size, lvl, sc = SZ(), C.c_int(), C.c_int(), C.c_double()
        _check(lib().he_ct_info(self.h, C.byref(B), C.byref(size), C.byref(lvl), C.byref(sc)))
        return B.value, size.value, lvl.value, sc.value

    @property
    def B(self): return self.info()[0]

    @property
    def size(self): return self.info()[1]

    @property
    def level(self): return self.info()[2]

    @property
    def scale(self): return self.info()[3]

    def words(self) -> np.ndarray:
        B, size, lvl, _ = self.info()
        out = np.zeros((B, size, lvl + 1, self.ctx.N), dtype=np.uint64)
        _check(lib().he_ct_export_words(self.ctx.h, self.h, _ptr(out), 0))
        return out

    def device_ptr(self) -> int:
        p = U64P()
        _check(lib().he_ct_device_ptr(self.h, C.byref(p)))
        return C.cast(p, C.c_void_p).value or 0


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)


class Context:
    """he_context_create + the calls that take a context, under the C names."""

    def __init__(self, logN: int, bits, n_special: int, seed: int, scale_log2: float = 0.0, _handle=None):
        if _handle is None:
            bits = [int(b) for b in bits]
            arr = (C.c_int * len(bits))(*bits)
            p = he_params(logN, len(bits), arr, n_special, scale_log2, 0)
            h = C.c_void_p()
            _check(lib().he_context_create(C.byref(p), seed, C.byref(h)))
        else:
            h = _handle
        self.h = h
        lg, L, K = C.c_int(), C.c_int(), C.c_int()
        _check(lib().he_context_info(h, C.byref(lg), C.byref(L), C.byref(K)))
        self.logN, self.L, self.K = lg.value, L.value, K.value
        self.N = 1 << self.logN
        pr = np.zeros(self.L + self.K, dtype=np.uint64)
        ps = np.zeros(self.L + self.K, dtype=np.uint64)
        _check(lib().he_context_primes(h, pr.ctypes.data_as(U64P), ps.ctypes.data_as(U64P)))
        self.primes, self.psis = pr, ps
        self.q = [int(x) for x in pr]
        self._stream = None
        try:
            import torch
            self._device = torch.cuda.current_device() if torch.cuda.is_available() else None
        except Exception:
            self._device = None

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.he_sync(self.h)
            _lib.he_context_free(self.h)
            self.h = None

    @property
    def slots(self) -> int:
        return self.N // 2

    # -- context ------------------------------------------------------------
    def he_context_cdt(self) -> np.ndarray:
        out = np.zeros(20, dtype=np.uint64)
        _check(lib().he_context_cdt(self.h, out.ctypes.data_as(U64P)))
        return out

    def he_set_stream(self, stream) -> None:
        """stream: a torch.cuda.Stream (or raw cudaStream_t int)."""
        s = getattr(stream, "cuda_stream", stream)
        _check(lib().he_set_stream(self.h, C.c_void_p(int(s) if s else 0)))
        # kept so device inputs of asynchronous calls can be tied to this stream (record_stream)
        self._stream = stream if hasattr(stream, "cuda_stream") else None

    def _dev_input(self, t, what: str):
        """A device float64 input read asynchronously on the context stream: checked for dtype and
        device, made contiguous, and recorded on the context stream so torch's caching allocator does
        not hand its memory to other work before the library's kernels have read it."""
        import torch
        if t.dtype != torch.float64:
            raise HEError(17, f"{what}: device input must be float64, got {t.dtype}")
        if self._device is not None and t.device.index != self._device:
            raise HEError(17, f"{what}: tensor on cuda:{t.device.index}, context on cuda:{self._device}")
        t = t.contiguous()
        st = getattr(self, "_stream", None)
        if st is not None and st.cuda_stream != torch.cuda.current_stream(t.device).cuda_stream:
            t.record_stream(st)
        return t

    def _dev_output(self, out, shape, what: str):
        import torch
        if out.dtype != torch.float64 or tuple(out.shape) != tuple(shape) or not out.is_contiguous():
            raise HEError(17, f"{what}: out must be a contiguous float64 tensor of shape {tuple(shape)}, "
                              f"got {out.dtype} {tuple(out.shape)}")
        if self._device is not None and out.device.index != self._device:
            raise HEError(17, f"{what}: out on cuda:{out.device.index}, context on cuda:{self._device}")

    def he_sync(self) -> None:
        _check(lib().he_sync(self.h))

    def he_launch_count(self) -> int:
        return int(lib().he_launch_count(self.h))

    def he_graph_begin(self) -> None:
        """Record the following calls on this context into a CUDA graph (he_graph_end)."""
        _check(lib().he_graph_begin(self.h))

    def he_graph_end(self) -> "Graph":
        h = C.c_void_p()
        _check(lib().he_graph_end(self.h, C.byref(h)))
        return Graph(self, h)

    def he_profile_enable(self, on: bool = True) -> None:
        _check(lib().he_profile_enable(self.h, int(bool(on))))

    def he_profile_read(self) -> dict:
        """{kernel tag: [launches, total_ms, alg_bytes, blocks]} since the last read."""
        import json
        buf = C.create_string_buffer(1 << 16)
        _check(lib().he_profile_read(self.h, buf, len(buf)))
        return json.loads(buf.value.decode())

    def he_keygen(self, steps=()) -> None:
        steps = [int(s) for s in steps]
        arr = (C.c_int32 * max(1, len(steps)))(*steps)
        _check(lib().he_keygen(self.h, arr, len(steps)))

    def he_drop_secret_key(self) -> None:
        _check(lib().he_drop_secret_key(self.h))

    def he_make_public(self) -> "Context":
        """A new context with copies of the public / relinearisation / Galois keys and no secret key."""
        h = C.c_void_p()
        _check(lib().he_make_public(self.h, C.byref(h)))
        pub = Context(0, (), 0, 0, _handle=h)
        pub._stream = self._stream
        return pub

    def he_set_allocator(self, alloc=None, free=None) -> None:
        """Install a device allocator: alloc(bytes, stream_ptr) -> device pointer (int),
        free(ptr, bytes, stream_ptr).  he_set_allocator_torch() installs torch's caching allocator.
        With no arguments the internal pool is restored."""
        if alloc is None:
            self._alloc_cbs = None
            _check(lib().he_set_allocator(self.h, None, None, None))
            return

        def a(nbytes, stream, user):
            try:
                return int(alloc(int(nbytes), int(stream or 0)))
            except Exception:
                return 0

        def f(ptr, nbytes, stream, user):
            try:
                free(int(ptr), int(nbytes), int(stream or 0))
            except Exception:
                pass
        cbs = (ALLOC_FN(a), FREE_FN(f))
        _check(lib().he_set_allocator(self.h, C.cast(cbs[0], C.c_void_p), C.cast(cbs[1], C.c_void_p), None))
        self._alloc_cbs = cbs   # the C side holds raw function pointers: keep the thunks alive

    def he_set_allocator_torch(self) -> None:
        """Device memory from torch's caching allocator (stream-ordered on the context stream)."""
        import torch
        dev = self._device if self._device is not None else torch.cuda.current_device()

        def alloc(nbytes, stream):
            return torch.cuda.caching_allocator_alloc(nbytes, dev, stream if stream else None)

        def free(ptr, nbytes, stream):
            torch.cuda.caching_allocator_delete(ptr)
        self.he_set_allocator(alloc, free)

    def he_key_bytes(self) -> int:
        """Device bytes held by the public, relinearisation and Galois keys (keys at rest)."""
        return int(lib().he_key_bytes(self.h))

    def he_key_export(self, kind: int, step: int = 0) -> np.ndarray:
        n = int(lib().he_key_words(self.h, kind))
        out = np.zeros(n, dtype=np.uint64)
        _check(lib().he_key_export(self.h, kind, step, out.ctypes.data_as(U64P)))
        N, L, NP = self.N, self.L, self.L + self.K
        shape = {0: (NP, N), 1: (2, L, N), 2: (L, 2, NP, N), 3: (L, 2, NP, N)}[kind]
        return out.reshape(shape)

    # -- encode / decode ------------------------------------------------------
    def he_encode(self, z, scale: float, level: int) -> Plaintext:
        """z: [B][n] (or [n]) float64 host array, or a CUDA float64 tensor."""
        h = C.c_void_p()
        if _is_dev(z):
            z2 = self._dev_input(z if z.dim() == 2 else z.reshape(1, -1), "he_encode")
            _check(lib().he_encode_device(self.h, _ptr(z2), z2.shape[1], z2.shape[0], float(scale), level,
                                          C.byref(h)))
        else:
            z2 = np.ascontiguousarray(np.atleast_2d(np.asarray(z, dtype=np.float64)))
            _check(lib().he_encode(self.h, z2.ctypes.data_as(DP), z2.shape[1], z2.shape[0], float(scale),
                                   level, C.byref(h)))
        return Plaintext(self, h)

    def he_encode_unrounded(self, z, scale: float):
        """[B][N] float64: the coefficient values he_encode rounds (C7 parity hook)."""
        z2 = np.ascontiguousarray(np.atleast_2d(np.asarray(z, dtype=np.float64)))
        res = np.zeros((z2.shape[0], self.N), dtype=np.float64)
        _check(lib().he_encode_unrounded(self.h, z2.ctypes.data_as(DP), z2.shape[1], z2.shape[0], float(scale),
                                         res.ctypes.data_as(DP)))
        return res

    def he_decode(self, pt: Plaintext, n: int | None = None, out=None):
        n = self.slots if n is None else n
        B = pt.B
        if out is not None and _is_dev(out):
            self._dev_output(out, (B, n), "he_decode")
            _check(lib().he_decode_device(self.h, pt.h, _ptr(out), n))
            return out
        if out is not None:
            raise HEError(17, "he_decode: out must be a CUDA tensor (host results are returned)")
        res = np.zeros((B, n), dtype=np.float64)
        _check(lib().he_decode(self.h, pt.h, res.ctypes.data_as(DP), n))
        return res

    def he_decode_async(self, pt: Plaintext, out, n: int) -> None:
        """Enqueue decode + D2H into host `out` [B][n] float64 (a pinned torch tensor or numpy
        array); valid after he_sync or an event recorded on the context stream."""
        B = pt.B
        if _is_dev(out) or tuple(out.shape) != (B, n) or str(out.dtype) not in ("torch.float64", "float64"):
            raise HEError(17, f"he_decode_async: out must be a host float64 [{B}][{n}] buffer")
        _check(lib().he_decode_async(self.h, pt.h, _ptr(out), n))

    def he_pt_from_int_coeffs(self, m, scale: float, level: int) -> Plaintext:
        m2 = np.ascontiguousarray(np.atleast_2d(np.asarray(m, dtype=np.int64)))
        h = C.c_void_p()
        _check(lib().he_pt_from_int_coeffs(self.h, m2.ctypes.data_as(I64P), m2.shape[0], float(scale), level,
                                           C.byref(h)))
        return Plaintext(self, h)

    def he_pt_from_int_coeffs_qp(self, m, scale: float, level: int) -> Plaintext:
        m2 = np.ascontiguousarray(np.atleast_2d(np.asarray(m, dtype=np.int64)))
        h = C.c_void_p()
        _check(lib().he_pt_from_int_coeffs_qp(self.h, m2.ctypes.data_as(I64P), m2.shape[0], float(scale), level,
                                              C.byref(h)))
        return Plaintext(self, h)

    def he_pt_export_words(self, pt: Plaintext, out) -> None:
        """Plaintext words [B][limbs][N] into `out` (a device int64/uint64 tensor or a host uint64 array)."""
        if out.dtype not in (np.uint64,) and str(out.dtype) not in ("torch.int64", "torch.uint64"):
            raise HEError(17, "he_pt_export_words: out must hold 64-bit words")
        if int(np.prod(out.shape)) != pt.B * pt.limbs * self.N:
            raise HEError(17, "he_pt_export_words: out has the wrong number of words")
        _check(lib().he_pt_export_words(self.h, pt.h, _ptr(out), _is_dev(out)))

    def he_ct_export_words(self, ct: Ciphertext, out) -> None:
        """Ciphertext words [B][size][level+1][N] into `out` (device int64/uint64 tensor or host uint64 array)."""
        if int(np.prod(out.shape)) != ct.B * ct.size * (ct.level + 1) * self.N:
            raise HEError(17, "he_ct_export_words: out has the wrong number of words")
        _check(lib().he_ct_export_words(self.h, ct.h, _ptr(out), _is_dev(out)))

    def he_pt_to_int_coeffs(self, pt: Plaintext) -> np.ndarray:
        """Signed integer coefficients m[B][N] of a plaintext (INTT, CRT, centred)."""
        out = np.zeros((pt.B, self.N), dtype=np.int64)
        _check(lib().he_pt_to_int_coeffs(self.h, pt.h, out.ctypes.data_as(I64P)))
        return out

    def he_pt_import_words(self, w, level: int, scale: float) -> Plaintext:
        h = C.c_void_p()
        if _is_dev(w):
            B = w.shape[0]
            _check(lib().he_pt_import_words(self.h, _ptr(w), 1, B, level, float(scale), C.byref(h)))
        else:
            w2 = np.ascontiguousarray(w, dtype=np.uint64).reshape(-1, level + 1, self.N)
            _check(lib().he_pt_import_words(self.h, _ptr(w2), 0, w2.shape[0], level, float(scale), C.byref(h)))
        return Plaintext(self, h)

    def he_ct_import_words(self, w, level: int, scale: float, size: int = 2) -> Ciphertext:
        h = C.c_void_p()
        if _is_dev(w):
            B = w.shape[0]
            _check(lib().he_ct_import_words(self.h, _ptr(w), 1, B, size, level, float(scale), C.byref(h)))
        else:
            w2 = np.ascontiguousarray(w, dtype=np.uint64).reshape(-1, size, level + 1, self.N)
            _check(lib().he_ct_import_words(self.h, _ptr(w2), 0, w2.shape[0], size, level, float(scale),
                                            C.byref(h)))
        return Ciphertext(self, h)

    # -- encrypt / decrypt ------------------------------------------------------
    def he_encrypt(self, pt: Plaintext, stream_id: int = 0) -> Ciphertext:
        h = C.c_void_p()
        _check(lib().he_encrypt(self.h, pt.h, stream_id, C.byref(h)))
        return Ciphertext(self, h)

    def he_encode_encrypt(self, z, scale: float, level: int, stream_id: int = 0) -> Ciphertext:
        """he_encode + he_encrypt in one call (same words); z as in he_encode (host array or CUDA tensor)."""
        h = C.c_void_p()
        if _is_dev(z):
            z2 = self._dev_input(z if z.dim() == 2 else z.reshape(1, -1), "he_encode_encrypt")
            _check(lib().he_encode_encrypt_device(self.h, _ptr(z2), z2.shape[1], z2.shape[0], float(scale), level,
                                                  stream_id, C.byref(h)))
        else:
            z2 = np.ascontiguousarray(np.atleast_2d(np.asarray(z, dtype=np.float64)))
            _check(lib().he_encode_encrypt(self.h, z2.ctypes.data_as(DP), z2.shape[1], z2.shape[0], float(scale),
                                           level, stream_id, C.byref(h)))
        return Ciphertext(self, h)

    def he_encrypt_symmetric(self, pt: Plaintext, stream_id: int, a_seed: int) -> Ciphertext:
        """Secret-key encryption with c1 drawn from the public seed a_seed (seeded wire form)."""
        h = C.c_void_p()
        _check(lib().he_encrypt_symmetric(self.h, pt.h, stream_id, a_seed, C.byref(h)))
        return Ciphertext(self, h)

    def he_decrypt(self, ct: Ciphertext) -> Plaintext:
        h = C.c_void_p()
        _check(lib().he_decrypt(self.h, ct.h, C.byref(h)))
        return Plaintext(self, h)

    # -- arithmetic -------------------------------------------------------------
    def _ct2(self, fn, *args) -> Ciphertext:
        h = C.c_void_p()
        _check(fn(self.h, *args, C.byref(h)))
        return Ciphertext(self, h)

    def he_add(self, a, b): return self._ct2(lib().he_add, a.h, b.h)
    def he_sub(self, a, b): return self._ct2(lib().he_sub, a.h, b.h)
    def he_negate(self, a): return self._ct2(lib().he_negate, a.h)
    def he_add_plain(self, a, p): return self._ct2(lib().he_add_plain, a.h, p.h)
    def he_mul_plain(self, a, p): return self._ct2(lib().he_mul_plain, a.h, p.h)
    def he_mul(self, a, b): return self._ct2(lib().he_mul, a.h, b.h)
    def he_square(self, a): return self._ct2(lib().he_square, a.h)
    def he_relinearize(self, a): return self._ct2(lib().he_relinearize, a.h)
    def he_rescale(self, a): return self._ct2(lib().he_rescale, a.h)
    def he_rotate(self, a, k: int): return self._ct2(lib().he_rotate, a.h, int(k))

    # in-place forms: a <- op(a, ...) (the handle is kept; returns a)
    def _ip(self, fn, a, *args):
        _check(fn(self.h, a.h, *args))
        return a

    def he_add_inplace(self, a, b): return self._ip(lib().he_add_inplace, a, b.h)
    def he_sub_inplace(self, a, b): return self._ip(lib().he_sub_inplace, a, b.h)
    def he_add_plain_inplace(self, a, p): return self._ip(lib().he_add_plain_inplace, a, p.h)
    def he_mul_plain_inplace(self, a, p): return self._ip(lib().he_mul_plain_inplace, a, p.h)
    def he_rescale_inplace(self, a): return self._ip(lib().he_rescale_inplace, a)
    def he_rotate_inplace(self, a, k: int): return self._ip(lib().he_rotate_inplace, a, int(k))
    def he_square_inplace(self, a): return self._ip(lib().he_square_inplace, a)

    def he_mod_switch_to(self, a, level: int): return self._ct2(lib().he_mod_switch_to, a.h, int(level))
    def he_dot(self, a, b, n: int): return self._ct2(lib().he_dot, a.h, b.h, int(n))
    def he_power(self, a, p: int): return self._ct2(lib().he_power, a.h, int(p))

    def he_dot_plain(self, a, z, n: int):
        z = np.ascontiguousarray(z, dtype=np.float64)
        return self._ct2(lib().he_dot_plain, a.h, z.ctypes.data_as(DP), z.size, int(n))

    def he_polyval(self, a, coeffs):
        cf = np.ascontiguousarray(coeffs, dtype=np.float64)
        return self._ct2(lib().he_polyval, a.h, cf.ctypes.data_as(DP), cf.size)

    def he_vec_mat(self, ct, W, bias=None, replicate_out=False, pt_scale_shift=0) -> Ciphertext:
        W = np.ascontiguousarray(W, dtype=np.float64)
        n, m = W.shape
        b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float64)
        return self._ct2(lib().he_vec_mat, ct.h, W.ctypes.data_as(DP), n, m,
                         None if b is None else b.ctypes.data_as(DP), int(bool(replicate_out)),
                         int(pt_scale_shift))

    def he_vec_mat_encode(self, W, bias, replicate_out, pt_scale_shift, level, in_scale, lazy=False, bsgs_g=0,
                          fold=False):
        """fold=True (replicated output, m | n, bsgs_g | m): he_vec_mat_encode_bsgs_fold."""
        W = np.ascontiguousarray(W, dtype=np.float64)
        n, m = W.shape
        b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float64)
        d, bp = C.c_void_p(), C.c_void_p()
        if fold:
            assert replicate_out and bsgs_g
            _check(lib().he_vec_mat_encode_bsgs_fold(self.h, W.ctypes.data_as(DP), n, m,
                                                     None if b is None else b.ctypes.data_as(DP),
                                                     int(pt_scale_shift), level, float(in_scale), int(bsgs_g),
                                                     C.byref(d), C.byref(bp)))
            return Plaintext(self, d), (Plaintext(self, bp) if bp.value else None)
        if bsgs_g:
            _check(lib().he_vec_mat_encode_bsgs(self.h, W.ctypes.data_as(DP), n, m,
                                                None if b is None else b.ctypes.data_as(DP), int(bool(replicate_out)),
                                                int(pt_scale_shift), level, float(in_scale), int(bsgs_g),
                                                C.byref(d), C.byref(bp)))
            return Plaintext(self, d), (Plaintext(self, bp) if bp.value else None)
        fn = lib().he_vec_mat_encode_lazy if lazy else lib().he_vec_mat_encode
        _check(fn(self.h, W.ctypes.data_as(DP), n, m,
                                       None if b is None else b.ctypes.data_as(DP), int(bool(replicate_out)),
                                       int(pt_scale_shift), level, float(in_scale), C.byref(d), C.byref(bp)))
        return Plaintext(self, d), (Plaintext(self, bp) if bp.value else None)

    def he_im2col_conv_encode(self, kernels, bias, chunk, kernel_shift, mask_shift, level, in_scale):
        k = np.ascontiguousarray(kernels, dtype=np.float64)
        Cn, kh, kw = k.shape[0], k.shape[-2], k.shape[-1]
        b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float64)
        kp, mp, bp = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _check(lib().he_im2col_conv_encode(self.h, k.ctypes.data_as(DP), Cn, kh, kw,
                                           None if b is None else b.ctypes.data_as(DP), int(chunk),
                                           int(kernel_shift), int(mask_shift), level, float(in_scale),
                                           C.byref(kp), C.byref(mp), C.byref(bp)))
        return Plaintext(self, kp), Plaintext(self, mp), (Plaintext(self, bp) if bp.value else None)

    def he_vec_mat_pt(self, ct, diags: Plaintext, bias: Plaintext | None = None) -> Ciphertext:
        return self._ct2(lib().he_vec_mat_pt, ct.h, diags.h, None if bias is None else bias.h)

    def he_vec_mat_bsgs_fold_pt(self, ct, diags: Plaintext, g: int, n: int, m: int,
                                bias: Plaintext | None = None) -> Ciphertext:
        return self._ct2(lib().he_vec_mat_bsgs_fold_pt, ct.h, diags.h, int(g), int(n), int(m),
                         None if bias is None else bias.h)

    def he_vec_mat_bsgs_pt(self, ct, diags: Plaintext, g: int, bias: Plaintext | None = None) -> Ciphertext:
        return self._ct2(lib().he_vec_mat_bsgs_pt, ct.h, diags.h, int(g), None if bias is None else bias.h)

    def he_im2col_conv(self, ct, kernels, bias=None, chunk=64, kernel_shift=0, mask_shift=0) -> Ciphertext:
        """kernels: [C][kh][kw] (or [C][1][kh][kw]) float64."""
        k = np.ascontiguousarray(kernels, dtype=np.float64)
        Cn, kh, kw = k.shape[0], k.shape[-2], k.shape[-1]
        b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float64)
        return self._ct2(lib().he_im2col_conv, ct.h, k.ctypes.data_as(DP), Cn, kh, kw,
                         None if b is None else b.ctypes.data_as(DP), int(chunk), int(kernel_shift),
                         int(mask_shift))

    def he_im2col_conv_hoisted_pt(self, ct, kernels: Plaintext, masks: Plaintext, bias: Plaintext | None,
                                  chunk: int, n1: int) -> Ciphertext:
        return self._ct2(lib().he_im2col_conv_hoisted_pt, ct.h, kernels.h, masks.h,
                         None if bias is None else bias.h, int(chunk), int(n1))

    def he_im2col_conv_bsgs_encode(self, kernels, bias, chunk, g, pt_shift, level, in_scale):
        """kernels [C][kh][kw] float64 -> (g QP diagonals D_b, bias plaintext or None)."""
        k = np.ascontiguousarray(kernels, dtype=np.float64)
        Cn, kh, kw = k.shape[0], k.shape[-2], k.shape[-1]
        b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float64)
        dp, bp = C.c_void_p(), C.c_void_p()
        _check(lib().he_im2col_conv_bsgs_encode(self.h, k.ctypes.data_as(DP), Cn, kh, kw,
                                                None if b is None else b.ctypes.data_as(DP), int(chunk), int(g),
                                                int(pt_shift), level, float(in_scale), C.byref(dp), C.byref(bp)))
        return Plaintext(self, dp), (Plaintext(self, bp) if bp.value else None)

    def he_im2col_conv_bsgs_pt(self, ct, diags: Plaintext, bias: Plaintext | None, chunk: int, g: int) -> Ciphertext:
        return self._ct2(lib().he_im2col_conv_bsgs_pt, ct.h, diags.h, None if bias is None else bias.h,
                         int(chunk), int(g))

    def he_im2col_conv_pt(self, ct, kernels: Plaintext, masks: Plaintext, bias: Plaintext | None,
                          chunk: int) -> Ciphertext:
        return self._ct2(lib().he_im2col_conv_pt, ct.h, kernels.h, masks.h, None if bias is None else bias.h,
                         int(chunk))

    # -- wire format -------------------------------------------------------------
    def he_ct_serialize(self, ct: Ciphertext) -> bytes:
        n = SZ()
        _check(lib().he_ct_serialized_size(self.h, ct.h, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        _check(lib().he_ct_serialize(self.h, ct.h, buf, 0))
        return buf.raw

    def he_ct_serialize_seeded(self, ct: Ciphertext) -> bytes:
        n = SZ()
        _check(lib().he_ct_serialized_size_seeded(self.h, ct.h, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        _check(lib().he_ct_serialize_seeded(self.h, ct.h, buf, 0))
        return buf.raw

    def he_ct_deserialize(self, data: bytes) -> Ciphertext:
        h = C.c_void_p()
        _check(lib().he_ct_deserialize(self.h, data, 0, len(data), C.byref(h)))
        return Ciphertext(self, h)

    # -- ring primitives (device tensors [B][nl][N] uint64 / int64) --------------
    def he_ntt_forward(self, d, B: int, nl: int) -> None:
        _check(lib().he_ntt_forward(self.h, _ptr(d), B, nl))

    def he_ntt_inverse(self, d, B: int, nl: int) -> None:
        _check(lib().he_ntt_inverse(self.h, _ptr(d), B, nl))

    def he_modmul(self, a, b, out, B: int, nl: int) -> None:
        _check(lib().he_modmul(self.h, _ptr(a), _ptr(b), _ptr(out), B, nl))

    def he_ntt_mul_intt(self, a, b, out, B: int, nl: int) -> None:
        _check(lib().he_ntt_mul_intt(self.h, _ptr(a), _ptr(b), _ptr(out), B, nl))


def he_im2col_encode_batch(imgs, kh: int, kw: int, stride: int, n_slots: int, out=None):
    """imgs [B][H][W] float64 -> slots [B][n_slots] (C18), one C call for the batch."""
    imgs = np.ascontiguousarray(imgs, dtype=np.float64)
    B, H, W = imgs.shape
    if out is None:
        out = np.zeros((B, n_slots), dtype=np.float64)
    elif (not isinstance(out, np.ndarray) or out.dtype != np.float64 or out.shape != (B, n_slots)
          or not out.flags.c_contiguous):
        raise HEError(17, f"he_im2col_encode_batch: out must be a C-contiguous float64 array of shape {(B, n_slots)}")
    _check(lib().he_im2col_encode_batch(imgs.ctypes.data_as(DP), B, H, W, kh, kw, stride, n_slots,
                                        out.ctypes.data_as(DP)))
    return out


def he_im2col_encode(img, kh: int, kw: int, stride: int, n_slots: int):
    """Client-side im2col + vertical scan (C18). Returns (slots, windows, chunk)."""
    img = np.ascontiguousarray(img, dtype=np.float64)
    H, W = img.shape
    out = np.zeros(n_slots, dtype=np.float64)
    w, ch = C.c_int(), C.c_int()
    _check(lib().he_im2col_encode(img.ctypes.data_as(DP), H, W, kh, kw, stride, n_slots,
                                  out.ctypes.data_as(DP), C.byref(w), C.byref(ch)))
    return out, w.value, ch.value

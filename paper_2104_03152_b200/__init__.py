"""B200-native CKKS hot path of TenSEAL's encrypted inference (arXiv 2104.03152).

The product is the C-ABI shared library ``libhe_ckks.so`` (include/he_ckks.h)
built from ``csrc/`` for sm_100a; ``ckks`` is its thin Python binding and
``cnn`` drives the paper's encrypted CNN through it.  This package never
imports ``oracle/`` (test infrastructure).
"""
from .ckks import (Ciphertext, Context, HEError, Plaintext, he_im2col_encode, he_im2col_encode_batch,  # noqa: F401
                   lib, LIB_PATH)

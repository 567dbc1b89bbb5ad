"""CPU-side checks of the C-ABI boundary (no GPU needed):
* libhe_ckks.so loads and exports every function include/he_ckks.h declares;
* the Python binding declares exactly those functions;
* without a GPU, context creation fails loudly (HE_CUDA_ERROR, no CPU fallback);
* host-only entry points (he_im2col_encode) follow C18 (compared with the oracle's layout);
* the product package never imports oracle/.
"""
import ast
import ctypes
import os
import re

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "he_ckks.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(he_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libso():
    from paper_2104_03152_b200.build import build
    return ctypes.CDLL(build())


def test_header_symbols_exported(libso):
    names = declared()
    assert len(names) > 40
    for n in names:
        assert hasattr(libso, n), f"{n} declared in he_ckks.h but not exported"


def test_binding_matches_header():
    from paper_2104_03152_b200 import ckks
    assert sorted(ckks.exported_symbols()) == declared()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure path")
def test_no_gpu_fails_loudly():
    from paper_2104_03152_b200 import Context, HEError
    with pytest.raises(HEError) as e:
        Context(13, (60, 40, 40, 60), 1, 0)
    assert e.value.name == "CUDA_ERROR"


def test_invalid_params_rejected_before_device():
    from paper_2104_03152_b200 import Context, HEError
    for logN, bits, K in [(9, (40, 40), 1), (13, (61, 40), 1), (13, (40, 40, 40, 40), 3), (13, (40,), 1)]:
        with pytest.raises(HEError) as e:
            Context(logN, bits, K, 0)
        assert e.value.name == "INVALID_PARAMS"


def test_im2col_encode_matches_oracle_layout():
    from oracle import circuits as OC
    from paper_2104_03152_b200 import he_im2col_encode
    img = np.random.default_rng(0).normal(size=(28, 28))
    got, windows, chunk = he_im2col_encode(img, 7, 7, 3, 4096)
    assert (windows, chunk) == (64, 64)
    assert np.array_equal(got, OC.im2col_slots(img, 7, 7, 3, 4096))
    from paper_2104_03152_b200 import HEError
    with pytest.raises(HEError) as e:
        he_im2col_encode(img, 7, 7, 3, 1024)
    assert e.value.name == "LAYOUT_MISMATCH"


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2104_03152_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            p = os.path.join(dirpath, f)
            if f.endswith(".py"):
                tree = ast.parse(open(p).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert not any(a.name.split(".")[0] == "oracle" for a in node.names), p
                    if isinstance(node, ast.ImportFrom):
                        assert not (node.module or "").startswith("oracle"), p
            if f.endswith((".cu", ".cuh", ".cpp", ".h")):
                assert "oracle" not in "".join(re.findall(r'#include\s*[<"][^>"]*[>"]', open(p).read())), p

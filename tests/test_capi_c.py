"""The C-ABI from plain C: tests/capi_smoke.c is compiled against
include/he_ckks.h and linked with libhe_ckks.so; on a GPU box it runs the boundary end to end
(keygen, encode, encrypt, rotate, in-place square / add_plain / mul_plain / rescale / rotate,
asynchronous decode, he_make_public, he_pt_to_int_coeffs, a caller-installed allocator)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = "/usr/local/cuda"


def _build(tmp_path):
    exe = str(tmp_path / "capi_smoke")
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    "-I", f"{CUDA}/include", os.path.join(ROOT, "tests", "capi_smoke.c"),
                    "-L", os.path.join(ROOT, "paper_2104_03152_b200"), "-lhe_ckks",
                    "-L", f"{CUDA}/lib64", "-lcudart", "-lm", "-o", exe], check=True)
    return exe


def test_capi_smoke_compiles_against_header(tmp_path):
    from paper_2104_03152_b200.build import build
    build()
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_capi_smoke_runs(tmp_path):
    exe = _build(tmp_path)
    env = dict(os.environ, LD_LIBRARY_PATH=os.path.join(ROOT, "paper_2104_03152_b200") + ":" + f"{CUDA}/lib64")
    r = subprocess.run([exe], capture_output=True, text=True, env=env, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "capi_smoke ok" in r.stdout

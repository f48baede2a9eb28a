"""The C ABI from plain C (tests/host/capi_roundtrip.c, no Python or torch in the loop):
include/ntt128.h compiles as C11 and the program links against the in-tree
libntt128.so (CPU); on a GPU it runs a forward + inverse and BLAS round trip through the
exported functions and checks the closed form y_0 = sum x_i (Eq. ntt)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2509_12494_b200")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def compile_demo(tmp_path):
    from paper_2509_12494_b200 import build
    build.build()
    exe = str(tmp_path / "capi_roundtrip")
    cmd = ["gcc", "-std=c11", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(CUDA, "include"), os.path.join(ROOT, "tests", "host", "capi_roundtrip.c"), "-o", exe,
           "-L", LIBDIR, "-lntt128", "-L", os.path.join(CUDA, "lib64"), "-lcudart", f"-Wl,-rpath,{LIBDIR}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_header_is_c11_and_links(tmp_path):
    compile_demo(tmp_path)


@pytest.mark.gpu
def test_plain_c_roundtrip(tmp_path, params):
    exe = compile_demo(tmp_path)
    e = params["cfg1"]
    M = (1 << 64) - 1
    args = [format(e["q"] & M, "x"), format(e["q"] >> 64, "x"), format(e["omega"] & M, "x"), format(e["omega"] >> 64, "x")]
    r = subprocess.run([exe] + args, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "capi ok" in r.stdout

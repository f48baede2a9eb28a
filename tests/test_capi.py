"""C-ABI contract checks that need no GPU: the in-tree library loads, exports every
function include/ntt128.h declares, and rejects bad arguments before touching CUDA."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def N():
    from paper_2509_12494_b200 import build
    build.build()
    from paper_2509_12494_b200 import ntt128
    return ntt128


def declared_functions():
    src = open(os.path.join(ROOT, "include", "ntt128.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b((?:ntt128|vec128|ntt256|vec256)_\w+)\s*\(", src)))


def test_exports_every_declared_symbol(N):
    names = declared_functions()
    assert len(names) == 36, names
    lib = ctypes.CDLL(N.LIB_PATH)
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(N.EXPORTED)


def test_status_strings(N):
    for code, name in enumerate(["OK", "ERR_INVALID_ARG", "ERR_MODULUS", "ERR_NOT_PRIME", "ERR_NO_ROOT", "ERR_BAD_ROOT",
                                 "ERR_ALIGNMENT", "ERR_INPUT_RANGE", "ERR_OOM", "ERR_CUDA", "ERR_UNSUPPORTED"]):
        assert N.status_string(code) == "NTT128_" + name


def create(N, log2n, batch, qs, roots, flags=0):
    h = ctypes.c_void_p()
    return N._L.ntt128_plan_create(ctypes.byref(h), log2n, batch, N._pairs(qs), N._pairs(roots), len(qs), flags, 0)


def test_plan_create_validation_host_only(N, params):
    """every rejection below happens in host code before any CUDA call"""
    e = params["cfg1"]
    q, w, psi = e["q"], e["omega"], e["psi"]
    assert create(N, 0, 1, [q], [w]) == 1
    assert create(N, 27, 1, [q], [w]) == 1
    assert create(N, 10, 0, [q], [w]) == 1
    assert create(N, 10, 3, [q, q], [w, w]) == 1            # n_moduli not 1 or batch
    assert create(N, 10, 1, [q], [w], flags=0x8) == 1       # unknown flag bit
    assert create(N, 10, 1, [q + 1], [w]) == 2              # even modulus
    assert create(N, 10, 1, [1], [w]) == 2
    assert create(N, 10, 1, [q + 2 * 2048], [w]) == 3       # composite
    assert create(N, 12, 1, [q], [w]) == 4                  # 2^12 does not divide q-1
    assert create(N, 11, 1, [q], [w], flags=1) == 4         # negacyclic needs 2N | q-1
    assert create(N, 10, 1, [q], [q]) == 5                  # root >= q
    assert create(N, 10, 1, [q], [w * w % q]) == 5          # order N/2
    assert create(N, 10, 1, [q], [w], flags=1) == 5         # omega is not of order 2N
    assert create(N, 10, 1, [17], [3]) == 4                 # 1024 does not divide 16
    assert create(N, 3, 1, [17], [4]) == 5                  # 4 has order 4 in Z_17, not 8


def test_known_small_roots(N):
    # Z_17: 2 has order 8 (2^4 = 16 = -1), 3 is a generator (order 16)
    assert pow(2, 4, 17) == 16 and pow(3, 8, 17) == 16


def test_fourstep_validation_host_only(N, params):
    import ctypes as C
    from paper_2509_12494_b200 import fourstep  # noqa: F401  (declares argtypes)
    e = params["cfg5"]
    q, w = e["q"], e["omega"]
    h = C.c_void_p()
    f = N._L.ntt128_fourstep_create
    assert f(C.byref(h), 0, 13, N._pairs([q]), N._pairs([w]), 0, 1, 0) == 1      # log2n1 out of range
    assert f(C.byref(h), 13, 14, N._pairs([q]), N._pairs([w]), 0, 1, 0) == 1     # log2n1 + log2n2 > 26
    assert f(C.byref(h), 9, 0, N._pairs([q]), N._pairs([w]), 0, 1, 0) == 1       # log2n2 out of range
    assert f(C.byref(h), 9, 17, N._pairs([q]), N._pairs([w]), 0, 16, 0) == 1     # world > 8
    assert f(C.byref(h), 13, 13, N._pairs([q]), N._pairs([w]), 0, 3, 0) == 1     # world not a power of two
    assert f(C.byref(h), 13, 13, N._pairs([q]), N._pairs([w]), 2, 2, 0) == 1     # rank >= world
    assert f(C.byref(h), 2, 2, N._pairs([q]), N._pairs([w]), 0, 8, 0) == 1      # world > n1
    assert f(C.byref(h), 3, 9, N._pairs([q]), N._pairs([w]), 0, 8, 0) == 1      # blocks of width n1 / G = 1
    assert f(C.byref(h), 13, 13, N._pairs([q + 1]), N._pairs([w]), 0, 1, 0) == 2  # even modulus
    assert f(C.byref(h), 13, 13, N._pairs([q]), N._pairs([w * w % q]), 0, 1, 0) == 5  # order N/2


def test_vec_validation_host_only(N, params):
    q = params["cfg2"]["q"]
    L = N._L
    assert L.vec128_add(16, 32, 48, 10, N._pairs([q + 1]), 0, None) == 2     # even q
    assert L.vec128_add(16, 32, 48, 10, N._pairs([q]), 0x4, None) == 1       # bad flags
    assert L.vec128_add(8, 32, 48, 10, N._pairs([q]), 0, None) == 6          # misaligned
    assert L.vec128_add(0, 0, 0, 10, N._pairs([q]), 0, None) == 1            # null pointers
    assert L.vec128_add(0, 0, 0, 0, N._pairs([q]), 0, None) == 0             # n = 0 no-op
    assert L.vec128_axpy(16, None, 32, 10, N._pairs([q]), 0, None) == 1      # null scalar

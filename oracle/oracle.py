"""ctypes binding of the plain C oracle (oracle/oracle128.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product path
(paper_2509_12494_b200/).  Shares no code with the CUDA path.

Residue arrays are numpy uint64 [..., 2] = [lo, hi] (same memory image as the
product's tensors).  Scalars are Python ints.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle128.c")
_LIB = os.path.join(_HERE, "liboracle128.so")
_lib = None

U64P = ctypes.POINTER(ctypes.c_uint64)


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, OpenMP).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-Wall", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i64 = ctypes.c_int64
        for name in ("o_mul_full", "o_rem_u256", "o_addmod", "o_submod", "o_mulmod", "o_powmod", "o_invmod"):
            getattr(L, name).restype = None
        L.o_is_prime.restype = ctypes.c_int
        L.o_find_prime.restype = ctypes.c_int
        L.o_find_prime.argtypes = [ctypes.c_int, U64P, ctypes.c_int, U64P]
        for name in ("o_vadd", "o_vsub", "o_vmul"):
            getattr(L, name).argtypes = [U64P, U64P, U64P, i64, U64P]
            getattr(L, name).restype = None
        L.o_axpy.argtypes = [U64P, U64P, U64P, i64, U64P]
        L.o_axpy.restype = None
        for name in ("o_ntt_batch", "o_intt_batch"):
            getattr(L, name).argtypes = [U64P, U64P, i64, i64, U64P, U64P, i64, ctypes.c_int]
            getattr(L, name).restype = None
        L.o_ntt_large.argtypes = [U64P, U64P, i64, U64P, U64P, ctypes.c_int]
        L.o_ntt_large.restype = None
        L.o_ntt_eval.argtypes = [U64P, i64, U64P, U64P, i64, U64P]
        L.o_ntt_eval.restype = None
        L.o_poly_mul_schoolbook.argtypes = [U64P, U64P, U64P, i64, U64P]
        L.o_poly_mul_schoolbook.restype = None
        L.o_conv.argtypes = [U64P, U64P, U64P, i64, U64P, ctypes.c_int]
        L.o_conv.restype = None
        L.o_negacyclic_dft.argtypes = [U64P, U64P, i64, U64P, U64P]
        L.o_negacyclic_dft.restype = None
        L.o_negacyclic_batch.argtypes = [U64P, U64P, i64, i64, U64P, U64P, i64, ctypes.c_int]
        L.o_negacyclic_batch.restype = None
        L.o_negacyclic_polymul_batch.argtypes = [U64P, U64P, U64P, i64, i64, U64P, U64P, i64]
        L.o_negacyclic_polymul_batch.restype = None
        L.o_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


# ----------------------------------------------------------------------------- helpers
def _pair(v: int) -> np.ndarray:
    assert 0 <= v < (1 << 128)
    return np.array([v & 0xFFFFFFFFFFFFFFFF, v >> 64], dtype=np.uint64)


def _pairs(vals) -> np.ndarray:
    return np.ascontiguousarray(np.stack([_pair(int(v)) for v in vals]))


def _p(a: np.ndarray):
    assert a.dtype == np.uint64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(U64P)


def _int(p: np.ndarray) -> int:
    return int(p[0]) | (int(p[1]) << 64)


def _c(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint64)


# ----------------------------------------------------------------------------- scalars
def mul_full(a: int, b: int) -> int:
    out = np.zeros(4, dtype=np.uint64)
    lib().o_mul_full(_p(_pair(a)), _p(_pair(b)), _p(out))
    return int(out[0]) | (int(out[1]) << 64) | (int(out[2]) << 128) | (int(out[3]) << 192)


def rem_u256(x: int, q: int) -> int:
    x4 = np.array([(x >> (64 * i)) & 0xFFFFFFFFFFFFFFFF for i in range(4)], dtype=np.uint64)
    out = np.zeros(2, dtype=np.uint64)
    lib().o_rem_u256(_p(x4), _p(_pair(q)), _p(out))
    return _int(out)


def _binop(name, a, b, q):
    out = np.zeros(2, dtype=np.uint64)
    getattr(lib(), name)(_p(_pair(a)), _p(_pair(b)), _p(_pair(q)), _p(out))
    return _int(out)


def addmod(a, b, q): return _binop("o_addmod", a, b, q)
def submod(a, b, q): return _binop("o_submod", a, b, q)
def mulmod(a, b, q): return _binop("o_mulmod", a, b, q)
def powmod(a, e, q): return _binop("o_powmod", a, e, q)


def invmod(a: int, q: int) -> int:
    out = np.zeros(2, dtype=np.uint64)
    lib().o_invmod(_p(_pair(a)), _p(_pair(q)), _p(out))
    return _int(out)


def is_prime(n: int) -> bool:
    return bool(lib().o_is_prime(_p(_pair(n))))


def find_prime(bits: int, m: int, skip: int = 0) -> int:
    out = np.zeros(2, dtype=np.uint64)
    rc = lib().o_find_prime(bits, _p(_pair(m)), skip, _p(out))
    if rc != 0:
        raise ValueError(f"no prime < 2^{bits} with p = 1 mod {m} (skip {skip})")
    return _int(out)


def num_threads() -> int:
    return int(lib().o_num_threads())


# ----------------------------------------------------------------------------- BLAS
def _blas(name, x, y, q):
    x, y = _c(x), _c(y)
    z = np.empty_like(x)
    getattr(lib(), name)(_p(z), _p(x), _p(y), x.size // 2, _p(_pair(q)))
    return z


def vadd(x, y, q): return _blas("o_vadd", x, y, q)
def vsub(x, y, q): return _blas("o_vsub", x, y, q)
def vmul(x, y, q): return _blas("o_vmul", x, y, q)


def axpy(a: int, x, y, q):
    """returns a*x + y mod q (the oracle does not modify the caller's y)"""
    x = _c(x)
    out = _c(y).copy()
    lib().o_axpy(_p(out), _p(_pair(a)), _p(x), x.size // 2, _p(_pair(q)))
    return out


# ----------------------------------------------------------------------------- NTT
def _batch_args(x, qs, roots):
    x = _c(x)
    n = x.shape[-2]
    batch = x.size // (2 * n)
    qs = list(qs) if isinstance(qs, (list, tuple)) else [qs]
    roots = list(roots) if isinstance(roots, (list, tuple)) else [roots]
    assert len(qs) == len(roots)
    return x, n, batch, _pairs(qs), _pairs(roots), len(qs)


def dft(x, q, w):
    """Eq. ntt by definition, O(n^2).  x: [..., n, 2]; q, w: int or per-poly lists."""
    x, n, batch, qa, wa, nq = _batch_args(x, q, w)
    y = np.empty_like(x)
    lib().o_ntt_batch(_p(y), _p(x), batch, n, _p(wa), _p(qa), nq, 0)
    return y


def ntt(x, q, w):
    """radix-2 Cooley-Tukey, natural order in and out."""
    x, n, batch, qa, wa, nq = _batch_args(x, q, w)
    y = np.empty_like(x)
    lib().o_ntt_batch(_p(y), _p(x), batch, n, _p(wa), _p(qa), nq, 1)
    return y


def idft(y, q, w):
    y, n, batch, qa, wa, nq = _batch_args(y, q, w)
    x = np.empty_like(y)
    lib().o_intt_batch(_p(x), _p(y), batch, n, _p(wa), _p(qa), nq, 0)
    return x


def intt(y, q, w):
    y, n, batch, qa, wa, nq = _batch_args(y, q, w)
    x = np.empty_like(y)
    lib().o_intt_batch(_p(x), _p(y), batch, n, _p(wa), _p(qa), nq, 1)
    return x


def ntt_large(x, q: int, w: int, inverse: bool = False):
    x = _c(x)
    y = np.empty_like(x)
    lib().o_ntt_large(_p(y), _p(x), x.size // 2, _p(_pair(w)), _p(_pair(q)), int(inverse))
    return y


def ntt_eval(x, q: int, w: int, k: int) -> int:
    """y_k of Eq. ntt by direct O(n) evaluation (threads over chunks of j)."""
    x = _c(x)
    out = np.zeros(2, dtype=np.uint64)
    lib().o_ntt_eval(_p(x), x.size // 2, _p(_pair(w)), _p(_pair(q)), k, _p(out))
    return _int(out)


# ----------------------------------------------------------------------------- polynomials
def poly_mul_schoolbook(a, b, q: int):
    a, b = _c(a), _c(b)
    n = a.shape[-2]
    c = np.empty((2 * n - 1, 2), dtype=np.uint64)
    lib().o_poly_mul_schoolbook(_p(c), _p(a), _p(b), n, _p(_pair(q)))
    return c


def conv_cyclic(a, b, q: int):
    a, b = _c(a), _c(b)
    c = np.empty_like(a)
    lib().o_conv(_p(c), _p(a), _p(b), a.shape[-2], _p(_pair(q)), 0)
    return c


def conv_negacyclic(a, b, q: int):
    a, b = _c(a), _c(b)
    c = np.empty_like(a)
    lib().o_conv(_p(c), _p(a), _p(b), a.shape[-2], _p(_pair(q)), 1)
    return c


def negacyclic_dft(x, q: int, psi: int):
    x = _c(x)
    y = np.empty_like(x)
    lib().o_negacyclic_dft(_p(y), _p(x), x.shape[-2], _p(_pair(psi)), _p(_pair(q)))
    return y


def negacyclic_ntt(x, q, psi, inverse: bool = False):
    x, n, batch, qa, pa, nq = _batch_args(x, q, psi)
    y = np.empty_like(x)
    lib().o_negacyclic_batch(_p(y), _p(x), batch, n, _p(pa), _p(qa), nq, int(inverse))
    return y


def negacyclic_polymul(a, b, q, psi):
    a, n, batch, qa, pa, nq = _batch_args(a, q, psi)
    b = _c(b)
    c = np.empty_like(a)
    lib().o_negacyclic_polymul_batch(_p(c), _p(a), _p(b), batch, n, _p(pa), _p(qa), nq)
    return c

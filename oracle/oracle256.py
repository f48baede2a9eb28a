"""ctypes binding of the 256-bit plain C oracle (oracle/oracle256.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
oracle legs, never by the product path.  Shares no code with the CUDA path.

Residue arrays are numpy uint64 [..., 4] (four little-endian limbs); scalars are Python ints.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle256.c")
_LIB = os.path.join(_HERE, "liboracle256.so")
_lib = None


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
        for name in ("o4_mul_full", "o4_addmod", "o4_submod", "o4_mulmod", "o4_powmod", "o4_vmul", "o4_ntt_batch"):
            getattr(L, name).restype = None
        L.o4_num_threads.restype = ctypes.c_int
        L.o4_is_prime.restype = ctypes.c_int
        L.o4_find_prime.restype = ctypes.c_int
        L.o4_find_prime.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p]
        _lib = L
    return _lib


def to_limbs(v: int) -> np.ndarray:
    return np.array([(v >> (64 * i)) & 0xFFFFFFFFFFFFFFFF for i in range(4)], dtype=np.uint64)


def from_limbs(a) -> int:
    return sum(int(x) << (64 * i) for i, x in enumerate(a))


def to_array(vals) -> np.ndarray:
    vals = list(vals)
    out = np.empty((len(vals), 4), dtype=np.uint64)
    for i, v in enumerate(vals):
        out[i] = to_limbs(v)
    return out


def to_ints(a: np.ndarray) -> list[int]:
    return [from_limbs(r) for r in a.reshape(-1, 4)]


def _p(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _scalar(name, *args):
    out = np.zeros(8 if name == "o4_mul_full" else 4, dtype=np.uint64)
    arrs = [to_limbs(a) for a in args]
    getattr(lib(), name)(*[_p(a) for a in arrs], _p(out))
    return from_limbs(out)


def mul_full(a: int, b: int) -> int:
    return _scalar("o4_mul_full", a, b)


def addmod(a, b, q): return _scalar("o4_addmod", a, b, q)
def submod(a, b, q): return _scalar("o4_submod", a, b, q)
def mulmod(a, b, q): return _scalar("o4_mulmod", a, b, q)
def powmod(a, e, q): return _scalar("o4_powmod", a, e, q)


def is_prime(n: int) -> bool:
    return bool(lib().o4_is_prime(_p(to_limbs(n))))


def find_prime(bits: int, m: int, skip: int = 0) -> int:
    """the skip-th largest prime q < 2^bits with q = 1 mod m (m a power of two)"""
    out = np.zeros(4, dtype=np.uint64)
    if not lib().o4_find_prime(bits, m, skip, _p(out)):
        raise RuntimeError("no prime found")
    return from_limbs(out)


def num_threads() -> int:
    return lib().o4_num_threads()


def vmul(x: np.ndarray, y: np.ndarray, q: int) -> np.ndarray:
    x, y = np.ascontiguousarray(x, dtype=np.uint64), np.ascontiguousarray(y, dtype=np.uint64)
    z = np.empty_like(x)
    lib().o4_vmul(_p(z), _p(x), _p(y), ctypes.c_int64(x.size // 4), _p(to_limbs(q)))
    return z


def ntt(x: np.ndarray, q, w, inverse: bool = False, small: bool = False) -> np.ndarray:
    """x [batch, n, 4] (or [n, 4]); q, w ints or per-polynomial lists"""
    x = np.ascontiguousarray(x, dtype=np.uint64)
    shape = x.shape
    x = x.reshape(-1, shape[-2], 4)
    batch, n = x.shape[0], x.shape[1]
    qs = q if isinstance(q, (list, tuple)) else [q]
    ws = w if isinstance(w, (list, tuple)) else [w]
    qa, wa = to_array(qs), to_array(ws)
    y = np.empty_like(x)
    lib().o4_ntt_batch(_p(y), _p(x), ctypes.c_int64(batch), ctypes.c_int64(n), _p(wa), _p(qa),
                       ctypes.c_int64(len(qs)), ctypes.c_int(int(inverse)), ctypes.c_int(int(small)))
    return y.reshape(shape)


def intt(y, q, w, small: bool = False):
    return ntt(y, q, w, inverse=True, small=small)

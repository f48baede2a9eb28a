"""CPU test of the product Barrett multiply (csrc/barrett128.cuh): the same
source the sm_100a vec128_mul kernel compiles, built for the host with g++ and checked
against Python integers on random and edge operands for several 128-bit moduli."""
import ctypes
import os
import random
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "host", "barrett_host.cpp")


@pytest.fixture(scope="module")
def lib(tmp_path_factory):
    so = str(tmp_path_factory.mktemp("barrett") / "libbarrett_host.so")
    subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-Wno-unknown-pragmas", "-o", so, SRC], check=True)
    L = ctypes.CDLL(so)
    L.barrett_mul_batch.argtypes = [ctypes.c_void_p] * 5 + [ctypes.c_long]
    return L


def words(vals):
    out = np.zeros((len(vals), 4), dtype=np.uint32)
    for i, v in enumerate(vals):
        for k in range(4):
            out[i, k] = (v >> (32 * k)) & 0xFFFFFFFF
    return out


def ints(w):
    return [sum(int(x) << (32 * k) for k, x in enumerate(row)) for row in w]


def run(L, a, b, q):
    mu = (1 << 256) // q - (1 << 128)
    A, Bw, Q, M = words(a), words(b), words([q]), words([mu])
    R = np.zeros_like(A)
    L.barrett_mul_batch(A.ctypes.data, Bw.ctypes.data, Q.ctypes.data, M.ctypes.data, R.ctypes.data, len(a))
    return ints(R)


MODULI = [
    (1 << 128) - 8257535,                           # cfg2 / cfg3 q0
    (1 << 128) - 2013265919,                        # cfg5
    (1 << 128) - 159,                               # largest prime below 2^128
    (1 << 127) + 29,                                # smallest prime above 2^127
    0x804671da650e225b9b75f6b15a9a0001,             # random 128-bit (params extra)
    0xBFFFFFFFFFFFFFFFFFFFFFFFFFFFFFF3,             # largest prime below 1.5 * 2^127
]


@pytest.mark.parametrize("q", MODULI)
def test_barrett_random_and_edges(lib, q):
    rng = random.Random(q & 0xFFFF)
    edge = [0, 1, 2, q - 1, q - 2, q // 2, (q + 1) // 2, (1 << 64) - 1, 1 << 64, (1 << 96) + 1, (1 << 127) - 1]
    edge = [e % q for e in edge]
    a, b = [], []
    for x in edge:
        for y in edge:
            a.append(x)
            b.append(y)
    for _ in range(20000):
        a.append(rng.randrange(q))
        b.append(rng.randrange(q))
    for _ in range(2000):                           # products just below multiples of q (q prime)
        x = rng.randrange(1, q)
        y = (rng.randrange(1, q) * pow(x, -1, q)) % q
        a.append(x)
        b.append((y - 1) % q)
    got = run(lib, a, b, q)
    assert got == [(x * y) % q for x, y in zip(a, b)]

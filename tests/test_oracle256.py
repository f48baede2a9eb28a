"""Pins of the 256-bit oracle (oracle/oracle256.c) against what the
mathematics fixes: Python integers for every scalar operation (random and edge operands),
sympy's BPSW for the prime search, Fermat's little theorem, the DFT by definition in pure
Python for N <= 16, closed forms (delta -> ones, ones -> [N, 0, ...], e_1 -> [w^k]),
radix-2 == definition, inverse(forward(x)) == x, and the generated roots' exact orders."""
import random

import numpy as np
import pytest
import sympy

from oracle import oracle256 as O4
import synth

MODULI = [(1 << 256) - 189, (1 << 255) - 19, (1 << 192) - 237, (1 << 130) + 51, 65537, 97]


def edges(q):
    v = [0, 1, 2, q - 1, q - 2, q // 2, (q + 1) // 2, (1 << 64) - 1, 1 << 64, (1 << 128) - 1, 1 << 128,
         (1 << 192) + 1, (1 << 255) - 1]
    return sorted({x % q for x in v})


@pytest.mark.parametrize("q", MODULI)
def test_scalar_ops_vs_python(q):
    rng = random.Random(q & 0xFFFF)
    pairs = [(a, b) for a in edges(q) for b in edges(q)] + [(rng.randrange(q), rng.randrange(q)) for _ in range(300)]
    for a, b in pairs:
        assert O4.mulmod(a, b, q) == a * b % q
        assert O4.addmod(a, b, q) == (a + b) % q
        assert O4.submod(a, b, q) == (a - b) % q
        assert O4.mul_full(a, b) == a * b
    for _ in range(20):
        a, e = rng.randrange(q), rng.randrange(1 << 256)
        assert O4.powmod(a, e, q) == pow(a, e, q)


def test_addmod_257th_bit():
    """a + b >= 2^256 (the sum needs a 257th bit) for q close to 2^256 (Eq. saddmod)"""
    q = (1 << 256) - 189
    for a in (q - 1, q - 2, (1 << 255) + 5):
        for b in (q - 1, q - 3, (1 << 255) + 7):
            assert O4.addmod(a, b, q) == (a + b) % q


def test_primes_vs_sympy():
    for bits, m in ((256, 1 << 21), (255, 1 << 21), (192, 1 << 21), (200, 1 << 10)):
        q = O4.find_prime(bits, m)
        assert q < (1 << bits) and (q - 1) % m == 0 and sympy.isprime(q)
        k = (q - 1) // m
        for kk in range(k + 1, k + 60):                          # nothing prime above it below 2^bits
            c = kk * m + 1
            if c >= (1 << bits):
                break
            assert not sympy.isprime(c)
    rng = random.Random(3)
    for _ in range(40):
        n = rng.randrange(1 << 255, 1 << 256) | 1
        assert O4.is_prime(n) == sympy.isprime(n)
    q = O4.find_prime(256, 1 << 21)
    for a in (2, 3, 12345678901234567890, q - 2):
        assert O4.powmod(a, q - 1, q) == 1                       # Fermat


def dft_py(x, q, w):
    n = len(x)
    return [sum(x[j] * pow(w, j * k, q) for j in range(n)) % q for k in range(n)]


@pytest.mark.parametrize("key", ["b256", "b255", "b192"])
def test_ntt_vs_definition(params, key):
    e = params["w256"][key]
    q, L = e["q"], e["logn"]
    for logn in (1, 2, 3, 4):
        w = pow(e["omega"], 1 << (L - logn), q)
        n = 1 << logn
        x = synth.uniform_residues_w(q, 2 * n, 50 + logn).reshape(2, n, 4)
        ref = [dft_py(O4.to_ints(x[b]), q, w) for b in range(2)]
        assert [O4.to_ints(r) for r in O4.ntt(x, q, w, small=True)] == ref      # O(N^2) definition
        assert [O4.to_ints(r) for r in O4.ntt(x, q, w)] == ref                  # radix-2
        assert np.array_equal(O4.intt(O4.ntt(x, q, w), q, w), x)


def test_ntt_closed_forms_and_radix2(params):
    e = params["w256"]["b254"]
    q, L = e["q"], e["logn"]
    logn = 8
    n = 1 << logn
    w = pow(e["omega"], 1 << (L - logn), q)
    delta = O4.to_array([1] + [0] * (n - 1))
    ones = O4.to_array([1] * n)
    e1 = O4.to_array([0, 1] + [0] * (n - 2))
    assert O4.to_ints(O4.ntt(delta, q, w)) == [1] * n
    assert O4.to_ints(O4.ntt(ones, q, w)) == [n] + [0] * (n - 1)
    assert O4.to_ints(O4.ntt(e1, q, w)) == [pow(w, k, q) for k in range(n)]
    x = synth.uniform_residues_w(q, n, 77)
    assert np.array_equal(O4.ntt(x, q, w), O4.ntt(x, q, w, small=True))
    y = O4.ntt(x, q, w)
    assert sum(O4.to_ints(y)) % q == n * O4.to_ints(x)[0] % q                 # sum_k y_k = N x_0
    assert np.array_equal(O4.intt(y, q, w), x)


def test_w256_roots_exact_order(params):
    for key, e in params["w256"].items():
        q, L = e["q"], e["logn"]
        assert sympy.isprime(q) and (q - 1) % (2 << L) == 0
        assert pow(e["psi"], 1 << L, q) == q - 1                  # psi of exact order 2^(L+1)
        assert e["omega"] == e["psi"] * e["psi"] % q
        assert pow(e["omega"], 1 << (L - 1), q) == q - 1          # omega of exact order 2^L


@pytest.mark.parametrize("q", MODULI)
def test_vmul_vs_python(q):
    """o4_vmul (the 256-bit element-wise product the GPU vec256_mul is compared with):
    every element against Python's a * b % q, on edge and random operands"""
    rng = random.Random(q & 0xFFF)
    ev = edges(q)
    xs = [a for a in ev for _ in ev] + [rng.randrange(q) for _ in range(2000)]
    ys = [b for _ in ev for b in ev] + [rng.randrange(q) for _ in range(2000)]
    z = O4.vmul(O4.to_array(xs), O4.to_array(ys), q)
    assert O4.to_ints(z) == [a * b % q for a, b in zip(xs, ys)]

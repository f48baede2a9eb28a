"""Pins of the oracle's primality test, prime search and the pinned parameters
(tests/golden/params.json) against sympy (BPSW) and Python's pow.

Rules: BASELINE.json configs; readings c10-c12.
"""
import json
import os
import random

import pytest
import sympy

from oracle import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
EX = json.load(open(os.path.join(HERE, "golden", "paper_examples.json")))


def test_is_prime_small_exhaustive():
    for n in range(0, 6000):
        assert O.is_prime(n) == sympy.isprime(n), n


def test_is_prime_pseudoprimes():
    # Carmichael numbers and strong pseudoprimes to small bases
    for n in (561, 1105, 1729, 2465, 2821, 6601, 8911, 2047, 3277, 4033, 4681, 8321, 3215031751,
              3825123056546413051, 318665857834031151167461, 3317044064679887385961981):
        assert O.is_prime(n) == sympy.isprime(n), n


def test_is_prime_random_128():
    rng = random.Random(11)
    for _ in range(300):
        n = rng.getrandbits(128) | 1
        assert O.is_prime(n) == sympy.isprime(n), hex(n)
    for _ in range(20):  # semiprimes of two 64-bit primes
        p = sympy.nextprime(rng.getrandbits(64))
        r = sympy.nextprime(rng.getrandbits(64))
        assert not O.is_prime(p * r)


def test_find_prime_is_largest(params):
    """q is prime and no q' = q + k M < 2^bits above it is prime (sympy)."""
    cases = [(128, 2 * 1024, params["cfg1"]["q"]), (128, 1 << 17, params["cfg2"]["q"]), (128, 1 << 27, params["cfg5"]["q"])]
    cases += [(128, 2 << int(k), v["q"]) for k, v in params["cfg4"].items()]
    for bits, m, q in cases:
        assert sympy.isprime(q)
        assert q % m == 1 and q < (1 << bits)
        c = q + m
        while c < (1 << bits):
            assert not sympy.isprime(c)
            c += m


def test_cfg3_rule(params):
    mods = params["cfg3"]["moduli"]
    assert len({m["q"] for m in mods}) == 64
    hist = {}
    for i, m in enumerate(mods):
        q = m["q"]
        b = 128 - (i % 5)
        assert q.bit_length() == b and q % (1 << 17) == 1 and sympy.isprime(q)
        hist[b] = hist.get(b, 0) + 1
    assert hist == {128: 13, 127: 13, 126: 13, 125: 13, 124: 12}
    # q_i is the floor(i/5)-th largest: the (i//5) primes above it of that width exist and are larger
    for i in range(5):
        q0, q1 = mods[i]["q"], mods[i + 5]["q"]
        assert q1 < q0
        c = q1 + (1 << 17)
        between = 0
        while c < q0:
            between += sympy.isprime(c)
            c += 1 << 17
        assert between == 0


def test_app_a_values(params):
    # SURVEY.md App. A (verified there with sympy BPSW)
    assert params["cfg1"]["q"] == 0xffffffffffffffffffffffffffff2801
    assert params["cfg2"]["q"] == 0xffffffffffffffffffffffffff820001
    assert params["cfg5"]["q"] == 0xffffffffffffffffffffffff88000001
    assert params["cfg3"]["moduli"][63]["q"] == 0x1ffffffffffffffffffffffffae20001


def _all_roots(params):
    yield params["cfg1"]
    yield params["cfg5"]
    yield from params["cfg3"]["moduli"]
    yield from params["cfg4"].values()
    yield from params["extra"].values()


def test_roots_exact_order(params):
    for e in _all_roots(params):
        q, n, psi, w = e["q"], 1 << e["logn"], e["psi"], e["omega"]
        assert pow(psi, n, q) == q - 1          # psi^N = -1: exact order 2N
        assert pow(w, n, q) == 1 and pow(w, n // 2, q) == q - 1 if n > 1 else True
        assert w == psi * psi % q


def test_spec_root_examples():
    e = EX["spec_root_5_4"]
    assert pow(e["omega"], e["n"], e["q"]) == 1 and pow(e["omega"], e["n"] // 2, e["q"]) != 1
    assert O.powmod(e["omega"], e["n"], e["q"]) == 1
    e = EX["spec_no_root_13_8"]
    from oracle.gen_params import find_root
    with pytest.raises(AssertionError):
        find_root(e["q"], e["n"], 0, 0)   # an element of order n needs n | q-1

"""Pins of the oracle's modular arithmetic (oracle/oracle128.c) against things other
than itself: Python arbitrary-precision integers, Fermat's little theorem, ring laws,
and SPEC's hand values (tests/golden/paper_examples.json).

Eq. 1-3, Eq. muls.
"""
import json
import os
import random

import pytest

from oracle import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
EX = json.load(open(os.path.join(HERE, "golden", "paper_examples.json")))
M128 = (1 << 128) - 1


def moduli(params):
    qs = [3, 17, 97, 7681, 65537, (1 << 61) - 1, M128]  # M128 is odd (not prime): arithmetic still defined
    qs += [params["cfg1"]["q"], params["cfg2"]["q"], params["cfg5"]["q"]]
    qs += [m["q"] for m in params["cfg3"]["moduli"][:5]]
    qs += [v["q"] for v in params["extra"].values()]
    return qs


def edge_values(q):
    """SURVEY.md §8(c) edge corpus e1 (restricted to < q)."""
    qh, ql = q >> 64, q & ((1 << 64) - 1)
    cand = [0, 1, 2, q - 1, q - 2, (q - 1) // 2, (q + 1) // 2, 2**32 - 1, 2**32, 2**32 + 1, 2**64 - 1, 2**64,
            2**64 + 1, 2**96, 2**127 - 1, 2**127, 2**127 + 1]
    for lo in (0, max(ql - 1, 0), ql, 2**64 - 1):
        cand.append((qh << 64) | lo)
    return sorted({c for c in cand if 0 <= c < q})


def pairs(q, rng, nrand=300):
    ev = edge_values(q)
    out = [(a, b) for a in ev for b in ev]
    out += [(rng.randrange(q), rng.randrange(q)) for _ in range(nrand)]
    # e2: sums landing on q-1, q, q+1, 2^128-1, 2^128, 2^128+1
    for t in (q - 1, q, q + 1, 2**128 - 1, 2**128, 2**128 + 1):
        for _ in range(5):
            b = rng.randrange(q)
            a = t - b
            if 0 <= a < q:
                out.append((a, b))
    # e3: both high words all-ones with a low-half carry (Listing 1 failure case)
    out.append((q - 1, q - 1))
    # e4: differences -1, 0, 1
    for _ in range(5):
        a = rng.randrange(1, q - 1)
        out += [(a, a + 1), (a, a), (a + 1, a)]
    return out


def test_spec_mulmod_example():
    e = EX["spec_mulmod_17"]
    assert O.mulmod(e["a"], e["b"], e["q"]) == e["expect"]


def test_mul_full_vs_bigint():
    rng = random.Random(1)
    vals = [0, 1, M128, M128 - 1, 2**64 - 1, 2**64, 2**127] + [rng.getrandbits(128) for _ in range(500)]
    for a in vals:
        for b in (vals[:7] + [rng.getrandbits(128)]):
            assert O.mul_full(a, b) == a * b


def test_rem_u256_vs_bigint():
    rng = random.Random(2)
    for q in (3, 17, 65537, M128, (1 << 127) + 1, rng.getrandbits(128) | 1):
        for _ in range(200):
            x = rng.getrandbits(256)
            assert O.rem_u256(x, q) == x % q
        assert O.rem_u256((1 << 256) - 1, q) == ((1 << 256) - 1) % q


def test_add_sub_mul_vs_bigint(params):
    rng = random.Random(3)
    for q in moduli(params):
        for a, b in pairs(q, rng, nrand=100 if q > 1 << 64 else 40):
            assert O.addmod(a, b, q) == (a + b) % q, (hex(q), a, b)
            assert O.submod(a, b, q) == (a - b) % q, (hex(q), a, b)
            assert O.mulmod(a, b, q) == (a * b) % q, (hex(q), a, b)


def test_mulmod_e5_products(params):
    """e5: products with a*b mod q in {0, 1, q-1} via (a, a^-1) and (a, -a^-1)."""
    rng = random.Random(4)
    for q in [params["cfg2"]["q"], params["extra"]["mid127"]["q"], params["extra"]["b124"]["q"], 65537]:
        for _ in range(20):
            a = rng.randrange(1, q)
            ai = pow(a, -1, q)
            assert O.mulmod(a, ai, q) == 1
            assert O.mulmod(a, q - ai, q) == q - 1
            assert O.mulmod(a, 0, q) == 0
            assert O.invmod(a, q) == ai


def test_fermat(params):
    rng = random.Random(5)
    for q in [m["q"] for m in params["cfg3"]["moduli"]][:8] + [params["cfg5"]["q"], 17, 65537]:
        for _ in range(3):
            a = rng.randrange(1, q)
            assert O.powmod(a, q - 1, q) == 1


def test_ring_laws(params):
    rng = random.Random(6)
    for q in (params["cfg2"]["q"], params["extra"]["b124"]["q"], 97):
        for _ in range(50):
            a, b, c = (rng.randrange(q) for _ in range(3))
            assert O.addmod(a, b, q) == O.addmod(b, a, q)
            assert O.mulmod(a, b, q) == O.mulmod(b, a, q)
            assert O.mulmod(O.mulmod(a, b, q), c, q) == O.mulmod(a, O.mulmod(b, c, q), q)
            assert O.mulmod(a, O.addmod(b, c, q), q) == O.addmod(O.mulmod(a, b, q), O.mulmod(a, c, q), q)
            assert O.submod(O.addmod(a, b, q), b, q) == a


def test_powmod_random_exponents_vs_python(params):
    """square-and-multiply against Python's pow on random 128-bit exponents (not only the
    Fermat / inverse exponents q - 1 and q - 2), edge exponents 0, 1, 2^127, 2^128 - 1"""
    rng = random.Random(11)
    qs = [params["cfg5"]["q"], params["cfg2"]["q"], params["extra"]["b124"]["q"], 97, 65537, (1 << 128) - 159]
    for q in qs:
        for e in [0, 1, 2, 1 << 64, 1 << 127, (1 << 128) - 1] + [rng.randrange(1 << 128) for _ in range(40)]:
            a = rng.randrange(q)
            assert O.powmod(a, e, q) == pow(a, e, q), (hex(q), e)

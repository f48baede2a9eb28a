"""Host check (no GPU) of the pseudo-Mersenne class arithmetic of csrc/psm128.cuh through
its word-level model (tools/model/psm_model.py): every add / sub / mul result is a 128-bit
representative of the exact value modulo q 2^s, psm_canon returns the exact residue, and every
carry the kernel code drops is asserted zero -- on edge values (around 0, C, q, Q, 2^128) in
all pairs and on random operands, for the SURVEY Appendix A primes (124..128 bits).  A
development model of the kernels, not the oracle."""
import importlib.util
import os
import random

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _load(rel, name):
    spec = importlib.util.spec_from_file_location(name, os.path.join(ROOT, rel))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


QS = [
    (1 << 128) - 55295, (1 << 128) - 8257535, (1 << 128) - 2013265919,     # Appendix A, 128-bit
    0x7fffffffffffffffffffffffff860001, 0x3ffffffffffffffffffffffffffc0001,  # cfg3 q_1, q_2
    0x1ffffffffffffffffffffffffffc0001, 0xfffffffffffffffffffffffffa60001,   # cfg3 q_3, q_4
    (1 << 128) - (1 << 32) + 2 + 1,                                        # C = 2^32 - 3 (arithmetic only)
    (1 << 128) - 1,                                                        # C = 1 (smallest; not prime: arithmetic only)
    (1 << 124) - (1 << 28) + 1,                                            # s = 4, c 2^s = 2^32 - 16
]


@pytest.mark.parametrize("q", QS)
def test_psm_edges_and_random(q):
    m = _load("tools/model/psm_model.py", "psm_model")
    ev = m.edge_values(q)
    for a in ev:
        for b in ev:
            m.check(q, a, b)
    rng = random.Random(q & 0xFFFF)
    for _ in range(1500):
        m.check(q, rng.randrange(1 << 128), rng.randrange(1 << 128))
    for _ in range(300):   # operands within a few C of 2^128: the double folds
        s, C = m.params(q)
        m.check(q, (1 << 128) - 1 - rng.randrange(2 * C), (1 << 128) - 1 - rng.randrange(2 * C))


def test_class_membership():
    m = _load("tools/model/psm_model.py", "psm_model")
    with pytest.raises(AssertionError):
        m.params(0x804671da650e225b9b75f6b15a9a0001)   # SURVEY Appendix A's random prime: not in the class
    with pytest.raises(AssertionError):
        m.params((1 << 128) - (1 << 32) - 1)           # C = 2^32 + 1
    with pytest.raises(AssertionError):
        m.params((1 << 128) - (1 << 32) + 1)           # C = 2^32 - 1: excluded (l4 + 1 must fit a word)

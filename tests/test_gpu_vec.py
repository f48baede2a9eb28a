"""GPU parity of the modular BLAS (vec128_add/sub/mul/axpy) against the oracle,
bit-exact, through the C ABI (BASELINE cfg 2)."""
import random

import numpy as np
import pytest

from oracle import oracle as O
import synth
from tests._util import edge_pairs, to_dev, to_host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def N():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2509_12494_b200 import ntt128
    return ntt128


def moduli(params):
    qs = [3, 17, 97, 65537, (1 << 61) - 1, (1 << 128) - 1, params["cfg1"]["q"], params["cfg2"]["q"], params["cfg5"]["q"]]
    qs += [v["q"] for v in params["extra"].values()]
    qs += [m["q"] for m in params["cfg3"]["moduli"][:5]]
    return qs


def check_all(N, x, y, q, a):
    dx, dy = to_dev(x), to_dev(y)
    assert np.array_equal(to_host(N.vadd(dx, dy, q)), O.vadd(x, y, q))
    assert np.array_equal(to_host(N.vsub(dx, dy, q)), O.vsub(x, y, q))
    assert np.array_equal(to_host(N.vmul(dx, dy, q)), O.vmul(x, y, q))
    ay = dy.clone()
    N.axpy(a, dx, ay, q)
    assert np.array_equal(to_host(ay), O.axpy(a, x, y, q))


def test_cfg2_full(N, params):
    """BASELINE cfg 2: n = 2^20, q = largest prime < 2^128 with q = 1 mod 2^17, a uniform"""
    q, n, a = params["cfg2"]["q"], params["cfg2"]["n"], params["cfg2"]["a"]
    x = synth.uniform_residues(q, n, synth.stream_seed(2, 0, 0))
    y = synth.uniform_residues(q, n, synth.stream_seed(2, 1, 0))
    check_all(N, x, y, q, a)


@pytest.mark.parametrize("n", [1, 2, 3, 7, 255, 1021, (1 << 20) - 3])
def test_ragged_lengths(N, params, n):
    q = params["cfg2"]["q"]
    x = synth.uniform_residues(q, n, 11 + n)
    y = synth.uniform_residues(q, n, 12 + n)
    check_all(N, x, y, q, random.Random(n).randrange(q))


def test_all_moduli_edge_corpus(N, params):
    rng = random.Random(5)
    for q in moduli(params):
        pairs = edge_pairs(q, rng)
        pairs += [(rng.randrange(q), rng.randrange(q)) for _ in range(2000)]
        x = synth.from_ints([p[0] for p in pairs])
        y = synth.from_ints([p[1] for p in pairs])
        for a in (0, 1, q - 1, rng.randrange(q)):
            check_all(N, x, y, q, a)


def test_in_place_aliasing(N, params):
    q = params["cfg2"]["q"]
    x = synth.uniform_residues(q, 4099, 21)
    y = synth.uniform_residues(q, 4099, 22)
    dx, dy = to_dev(x), to_dev(y)
    N.vadd(dx, dy, q, out=dx)
    assert np.array_equal(to_host(dx), O.vadd(x, y, q))
    dx = to_dev(x)
    N.vmul(dx, dy, q, out=dy)
    assert np.array_equal(to_host(dy), O.vmul(x, y, q))


def test_errors(N, params):
    import torch
    q = params["cfg2"]["q"]
    x = to_dev(synth.uniform_residues(q, 64, 1))
    bad = x.clone()
    bad[5, :] = -1                       # both limbs all ones: 2^128 - 1 >= q
    with pytest.raises(N.NTT128ArgError, match="INPUT_RANGE"):
        N.vadd(bad, x, q, check_input=True)
    with pytest.raises(N.NTT128ArgError, match="MODULUS"):
        N.vadd(x, x, q + 1)
    big = torch.zeros(65, 2, dtype=torch.int64, device="cuda")
    # misaligned device pointer -> NTT128_ERR_ALIGNMENT (6), nothing enqueued
    assert N._L.vec128_add(big.data_ptr() + 8, x.data_ptr(), x.data_ptr(), 8, N._pairs([q]), 0, None) == 6
    assert N._L.vec128_add(0, 0, 0, 0, N._pairs([q]), 0, None) == 0      # n == 0 is a no-op
    with pytest.raises(N.NTT128ArgError, match="INPUT_RANGE"):
        N.axpy(q, x, x.clone(), q)                                     # scalar a >= q


@pytest.mark.parametrize("q", [(1 << 127) + 29, (1 << 128) - 159, 0xBFFFFFFFFFFFFFFFFFFFFFFFFFFFFFF3])
def test_vmul_barrett_hard_cases(N, q):
    """vec128_mul on q > 2^127 runs the Barrett product (csrc/barrett128.cuh): operands whose
    product lies just below / at / above a multiple of q exercise every correction count"""
    import random
    rng = random.Random(q & 0xFFFFF)
    a, b = [], []
    for _ in range(3000):
        x = rng.randrange(1, q)
        t = rng.randrange(1, q)
        y = (t * pow(x, -1, q)) % q
        for d in (-1, 0, 1):
            a.append(x)
            b.append((y + d) % q)
    for _ in range(3000):
        a.append(rng.randrange(q))
        b.append(rng.randrange(q))
    x, y = synth.from_ints(a), synth.from_ints(b)
    got = synth.to_ints(to_host(N.vmul(to_dev(x), to_dev(y), q)))
    assert got == [(u * v) % q for u, v in zip(a, b)]
    assert np.array_equal(to_host(N.vmul(to_dev(x), to_dev(y), q)), O.vmul(x, y, q))

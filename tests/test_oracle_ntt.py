"""Pins of the oracle's transforms and polynomial products (oracle/oracle128.c):
the paper's worked example, pure-Python brute force DFTs (Eq. ntt by definition),
closed forms, the convolution theorem against schoolbook products, and round trips.

Eq. ntt; schoolbook product PAPER.md:266-271.
"""
import itertools
import json
import os
import random

import numpy as np
import pytest

from oracle import oracle as O
import synth

HERE = os.path.dirname(os.path.abspath(__file__))
EX = json.load(open(os.path.join(HERE, "golden", "paper_examples.json")))


def arr(vals):
    return synth.from_ints(vals)


def ints(a):
    return synth.to_ints(a)


def py_dft(x, w, q):
    n = len(x)
    return [sum(x[j] * pow(w, j * k, q) for j in range(n)) % q for k in range(n)]


def root(q, n, rng=None):
    """an element of exact order n (n a power of two) by brute search, pure Python"""
    assert (q - 1) % n == 0
    for g in range(2, q):
        w = pow(g, (q - 1) // n, q)
        if pow(w, n // 2, q) == q - 1 if n > 1 else w == 1:
            return w
    raise ValueError


def test_paper_evaluation_form_example():
    e = EX["paper_eval_form_5"]
    x = arr(e["coeffs"])
    assert ints(O.dft(x, e["q"], e["omega"])) == e["expect_ntt"]
    assert ints(O.ntt(x, e["q"], e["omega"])) == e["expect_ntt"]
    # the evaluation form is the multiset {f(1), f(2), f(3), f(4)}
    assert sorted(ints(O.dft(x, e["q"], e["omega"]))) == sorted(e["f_at"].values())


def test_exhaustive_q5_n4():
    """all 625 inputs, both primitive 4th roots (2 and 3) vs the definition"""
    xs = np.array(list(itertools.product(range(5), repeat=4)), dtype=np.uint64)
    X = np.zeros((625, 4, 2), dtype=np.uint64)
    X[:, :, 0] = xs
    for w in (2, 3):
        Y = O.dft(X, [5] * 625, [w] * 625)
        Z = O.ntt(X, [5] * 625, [w] * 625)
        for i in range(625):
            ref = py_dft([int(v) for v in xs[i]], w, 5)
            assert ints(Y[i]) == ref and ints(Z[i]) == ref


def test_dft_bruteforce_small(params):
    rng = random.Random(21)
    qs = [17, 97, 7681, 65537, params["cfg1"]["q"], params["extra"]["mid127"]["q"], params["extra"]["b124"]["q"]]
    for q in qs:
        for logn in range(1, 5):
            n = 1 << logn
            if (q - 1) % n:
                continue
            w = root(q, n) if q < 1 << 20 else pow(params["extra"]["b124"]["omega"] if q == params["extra"]["b124"]["q"] else
                                                     params["extra"]["mid127"]["omega"] if q == params["extra"]["mid127"]["q"] else
                                                     params["cfg1"]["omega"], (1 << 17 if q != params["cfg1"]["q"] else 1 << 10) // n, q)
            assert pow(w, n, q) == 1
            x = [rng.randrange(q) for _ in range(n)]
            ref = py_dft(x, w, q)
            assert ints(O.dft(arr(x), q, w)) == ref
            assert ints(O.ntt(arr(x), q, w)) == ref


def test_closed_forms(params):
    e = params["cfg1"]
    q, n, w = e["q"], 1 << e["logn"], e["omega"]
    one = [1] + [0] * (n - 1)
    assert ints(O.ntt(arr(one), q, w)) == [1] * n                      # delta -> all ones
    assert ints(O.ntt(arr([1] * n), q, w)) == [n] + [0] * (n - 1)      # ones -> [n,0..]
    e1 = [0, 1] + [0] * (n - 2)
    assert ints(O.ntt(arr(e1), q, w)) == [pow(w, k, q) for k in range(n)]
    rng = random.Random(22)
    x = [rng.randrange(q) for _ in range(n)]
    y = ints(O.ntt(arr(x), q, w))
    assert y[0] == sum(x) % q                                          # y_0 = sum x_j
    assert sum(y) % q == n * x[0] % q                                  # sum_k y_k = n x_0
    s = 5                                                              # shift theorem
    xs = [x[(j - s) % n] for j in range(n)]
    assert ints(O.ntt(arr(xs), q, w)) == [y[k] * pow(w, s * k, q) % q for k in range(n)]
    a, z = rng.randrange(q), [rng.randrange(q) for _ in range(n)]   # linearity
    yz = ints(O.ntt(arr(z), q, w))
    lin = ints(O.ntt(arr([(a * x[j] + z[j]) % q for j in range(n)]), q, w))
    assert lin == [(a * y[k] + yz[k]) % q for k in range(n)]


@pytest.mark.parametrize("logn", [1, 2, 3, 5, 8, 10, 12])
def test_ntt_equals_dft_and_roundtrip(params, logn):
    rng = np.random.default_rng(logn)
    for key in ("b124", "mid127", "rand128_0", "q65537"):
        e = params["extra"][key]
        q = e["q"]
        if e["logn"] + 1 < logn:
            continue
        w = pow(e["omega"], (1 << e["logn"]) >> logn, q) if logn <= e["logn"] else e["psi"]
        n = 1 << logn
        assert pow(w, n, q) == 1 and (n == 1 or pow(w, n // 2, q) == q - 1)
        x = synth.uniform_residues(q, 2 * n, int(rng.integers(1 << 40))).reshape(2, n, 2)
        y = O.ntt(x, [q, q], [w, w])
        if logn <= 10:
            assert np.array_equal(y, O.dft(x, [q, q], [w, w]))
        assert np.array_equal(O.intt(y, [q, q], [w, w]), x)
        if logn <= 8:
            assert np.array_equal(O.idft(y, [q, q], [w, w]), x)


def test_ntt_large_and_eval(params):
    e = params["cfg4"]["12"]
    q, n, w = e["q"], 1 << 12, e["omega"]
    x = synth.uniform_residues(q, n, 99)
    y = O.ntt(x, q, w)
    assert np.array_equal(O.ntt_large(x, q, w), y)
    assert np.array_equal(O.ntt_large(y, q, w, inverse=True), x)
    yi = synth.to_ints(y)
    for k in (0, 1, 7, 2048, 4095):
        assert O.ntt_eval(x, q, w, k) == yi[k]


def py_conv(a, b, q, sign):
    n = len(a)
    c = [0] * n
    for i in range(n):
        for j in range(n):
            k = i + j
            if k >= n:
                c[k - n] = (c[k - n] + sign * a[i] * b[j]) % q
            else:
                c[k] = (c[k] + a[i] * b[j]) % q
    return c


def test_schoolbook_and_conv_bruteforce():
    e = EX["spec_square_17"]
    assert ints(O.poly_mul_schoolbook(arr(e["a"]), arr(e["b"]), e["q"])) == e["expect"]
    rng = random.Random(23)
    for q in (17, 97, 65537, (1 << 127) + 45):
        for n in (1, 2, 3, 8, 16):
            a = [rng.randrange(q) for _ in range(n)]
            b = [rng.randrange(q) for _ in range(n)]
            full = [sum(a[i] * b[k - i] for i in range(n) if 0 <= k - i < n) % q for k in range(2 * n - 1)]
            assert ints(O.poly_mul_schoolbook(arr(a), arr(b), q)) == full
            assert ints(O.conv_cyclic(arr(a), arr(b), q)) == py_conv(a, b, q, 1)
            assert ints(O.conv_negacyclic(arr(a), arr(b), q)) == py_conv(a, b, q, -1)


def test_convolution_theorem(params):
    """NTT(a (*) b) = NTT(a) . NTT(b)"""
    for key, logn in (("b124", 3), ("q7681", 8), ("mid127", 10)):
        e = params["extra"][key]
        q, n = e["q"], 1 << logn
        w = pow(e["omega"], (1 << e["logn"]) >> logn, q)
        a = synth.uniform_residues(q, n, 1)
        b = synth.uniform_residues(q, n, 2)
        lhs = O.ntt(O.conv_cyclic(a, b, q), q, w)
        rhs = O.vmul(O.ntt(a, q, w), O.ntt(b, q, w), q)
        assert np.array_equal(lhs, rhs)


def test_negacyclic(params):
    for key, logn in (("q17", 3), ("q97", 4), ("b126", 6), ("rand128_1", 9)):
        e = params["extra"][key]
        q, n = e["q"], 1 << logn
        psi = pow(e["psi"], (1 << e["logn"]) >> logn, q)
        assert pow(psi, n, q) == q - 1
        x = synth.uniform_residues(q, n, 3)
        y = O.negacyclic_ntt(x, q, psi)
        assert np.array_equal(y, O.negacyclic_dft(x, q, psi))
        # definition in pure Python: evaluation at psi^(2k+1)
        if n <= 16:
            xi = synth.to_ints(x)
            ref = [sum(xi[j] * pow(psi, j * (2 * k + 1), q) for j in range(n)) % q for k in range(n)]
            assert synth.to_ints(y) == ref
        assert np.array_equal(O.negacyclic_ntt(y, q, psi, inverse=True), x)
        a, b = synth.uniform_residues(q, n, 4), synth.uniform_residues(q, n, 5)
        assert np.array_equal(O.negacyclic_polymul(a, b, q, psi), O.conv_negacyclic(a, b, q))
        # X * X^(n-1) = -1 in Z_q[X]/(X^n + 1)
        X1 = arr([0, 1] + [0] * (n - 2))
        Xn1 = arr([0] * (n - 1) + [1])
        assert synth.to_ints(O.negacyclic_polymul(X1, Xn1, q, psi)) == [q - 1] + [0] * (n - 1)


def test_blas(params):
    q = params["cfg2"]["q"]
    rng = random.Random(24)
    n = 1 << 11
    x = synth.uniform_residues(q, n, 7)
    y = synth.uniform_residues(q, n, 8)
    a = rng.randrange(q)
    xi, yi = synth.to_ints(x), synth.to_ints(y)
    assert synth.to_ints(O.vadd(x, y, q)) == [(u + v) % q for u, v in zip(xi, yi)]
    assert synth.to_ints(O.vsub(x, y, q)) == [(u - v) % q for u, v in zip(xi, yi)]
    assert synth.to_ints(O.vmul(x, y, q)) == [(u * v) % q for u, v in zip(xi, yi)]
    assert synth.to_ints(O.axpy(a, x, y, q)) == [(a * u + v) % q for u, v in zip(xi, yi)]
    # closed forms
    negx = arr([(q - v) % q for v in xi])
    assert synth.to_ints(O.vadd(x, negx, q)) == [0] * n
    assert synth.to_ints(O.vsub(x, x, q)) == [0] * n
    assert np.array_equal(O.vmul(x, arr([1] * n), q), x)
    assert np.array_equal(O.axpy(0, x, y, q), y)
    assert np.array_equal(O.axpy(1, x, arr([0] * n), q), x)


def test_butterfly_count_example():
    e = EX["spec_butterflies_1024"]
    n = e["n"]
    assert (n // 2) * (n.bit_length() - 1) == e["expect"]

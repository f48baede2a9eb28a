"""GPU parity of the permutation-free negacyclic path:
ntt128_forward_bitrev / ntt128_inverse_bitrev and the polymul built on them, bit-exact
against the oracle's natural-order negacyclic transform (permuted by n-bit reversal) and
its polynomial product.  Every modulus class (q < 2^126 Harvey, q < 2^127 half-lazy,
full width), every pass schedule (2, 3 and 4 passes of 5..8 bits), structured inputs."""
import numpy as np
import pytest

from oracle import oracle as O
import synth
from tests._util import to_dev, to_host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def N():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2509_12494_b200 import ntt128
    return ntt128


def brev_perm(logn):
    n = 1 << logn
    return np.array([int(format(i, f"0{logn}b")[::-1], 2) for i in range(n)], dtype=np.int64)


def psi_for(e, logn):
    return pow(e["psi"], 1 << (e["logn"] - logn), e["q"])


@pytest.mark.parametrize("logn", [10, 11, 12, 13, 14, 16, 17])
def test_forward_bitrev_all_classes(N, params, logn):
    for key in ("b124", "b126", "b127", "mid127", "rand128_1"):
        e = params["extra"][key]
        q, psi = e["q"], psi_for(e, logn)
        B, n = 2, 1 << logn
        x = synth.uniform_residues(q, n * B, 1100 + logn).reshape(B, n, 2)
        plan = N.Plan(logn, q, psi, batch=B, negacyclic=True)
        y = to_host(plan.forward_bitrev(to_dev(x)))
        ref = O.negacyclic_ntt(x, [q] * B, [psi] * B)[:, brev_perm(logn)]
        assert np.array_equal(y, ref), f"forward_bitrev mismatch {key} N=2^{logn}"
        assert np.array_equal(to_host(plan.inverse_bitrev(to_dev(y))), x), f"inverse_bitrev {key} N=2^{logn}"


@pytest.mark.parametrize("logn", [20, 25])
def test_bitrev_three_and_four_passes(N, params, logn):
    """2^20: three 7/7/6-bit passes; 2^25: four passes (7/6/6/6)"""
    e = params["cfg5"]
    q, psi = e["q"], pow(e["psi"], 1 << (e["logn"] - logn), e["q"])
    n = 1 << logn
    x = synth.uniform_residues(q, n, 1200 + logn).reshape(1, n, 2)
    plan = N.Plan(logn, q, psi, negacyclic=True)
    dy = plan.forward_bitrev(to_dev(x))
    if logn <= 20:
        ref = O.negacyclic_ntt(x, q, psi)[:, brev_perm(logn)]
        assert np.array_equal(to_host(dy), ref)
    else:   # sampled outputs by direct evaluation Y[i] = a(psi^(2 brev(i) + 1))
        y = to_host(dy)
        rng = np.random.default_rng(logn)
        for i in [0, 1, n - 1] + [int(v) for v in rng.integers(0, n, 3)]:
            k = int(format(i, f"0{logn}b")[::-1], 2)
            pt = pow(psi, 2 * k + 1, q)                       # a(pt) = sum_j a_j pt^j
            assert synth.to_ints(y[0, i:i + 1])[0] == O.ntt_eval(x[0], q, pt, 1)
    assert np.array_equal(to_host(plan.inverse_bitrev(dy)), x)


def test_bitrev_structured_and_in_place(N, params):
    e = params["extra"]["b125"]
    logn = 12
    q, psi = e["q"], psi_for(e, logn)
    n = 1 << logn
    rows = [[1] + [0] * (n - 1), [q - 1] * n, [0, q - 1] * (n // 2), [1] * n]
    x = np.stack([synth.from_ints(r) for r in rows])
    plan = N.Plan(logn, q, psi, batch=len(rows), negacyclic=True)
    d = to_dev(x)
    plan.forward_bitrev(d, out=d)
    ref = O.negacyclic_ntt(x, [q] * len(rows), [psi] * len(rows))[:, brev_perm(logn)]
    assert np.array_equal(to_host(d), ref)
    assert synth.to_ints(to_host(d)[0]) == [1] * n            # delta -> all ones in any order
    plan.inverse_bitrev(d, out=d)
    assert np.array_equal(to_host(d), x)


def test_bitrev_rns_polymul(N, params):
    """cfg3 moduli (all three classes), N = 2^16: the permutation-free polymul"""
    mods = params["cfg3"]["moduli"][:10]
    qs, psis = [m["q"] for m in mods], [m["psi"] for m in mods]
    n, B = 1 << 16, len(mods)
    a = np.stack([synth.uniform_residues(qs[i], n, synth.stream_seed(3, 0, 1300 + i)) for i in range(B)])
    b = np.stack([synth.uniform_residues(qs[i], n, synth.stream_seed(3, 1, 1300 + i)) for i in range(B)])
    plan = N.Plan(16, qs, psis, batch=B, negacyclic=True)
    c = to_host(plan.polymul(to_dev(a), to_dev(b)))
    assert np.array_equal(c, O.negacyclic_polymul(a, b, qs, psis))


def test_bitrev_polymul_vs_schoolbook(N, params):
    e = params["extra"]["b127"]
    for logn in (10, 11):
        q, psi = e["q"], psi_for(e, logn)
        n = 1 << logn
        a = synth.uniform_residues(q, n, 1400 + logn).reshape(1, n, 2)
        b = synth.uniform_residues(q, n, 1500 + logn).reshape(1, n, 2)
        plan = N.Plan(logn, q, psi, negacyclic=True)
        c = to_host(plan.polymul(to_dev(a), to_dev(b)))
        assert np.array_equal(c[0], O.conv_negacyclic(a[0], b[0], q))


def test_bitrev_unsupported(N, params):
    e = params["extra"]["rand128_0"]
    q = e["q"]
    small = N.Plan(9, q, psi_for(e, 9), negacyclic=True)
    x = to_dev(synth.uniform_residues(q, 512, 1).reshape(1, 512, 2))
    with pytest.raises(N.NTT128Error, match="UNSUPPORTED"):
        small.forward_bitrev(x)
    cyc = N.Plan(12, q, pow(e["psi"], 1 << (e["logn"] + 1 - 12), q))
    x = to_dev(synth.uniform_residues(q, 4096, 1).reshape(1, 4096, 2))
    with pytest.raises(N.NTT128Error, match="UNSUPPORTED"):
        cyc.forward_bitrev(x)

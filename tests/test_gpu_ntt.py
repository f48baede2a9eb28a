"""GPU parity of the NTT (forward, inverse, negacyclic, polymul) against the oracle,
bit-exact, through the C ABI.  Eq. ntt; BASELINE cfgs 1, 3, 4.

Sizes span single-pass (N <= 2^12), two-pass (2^13..2^18) and three-pass (>= 2^19)
schedules; moduli span every width regime (17 ... 2^128 - c); inputs include the
structured cases (delta, ones, all q-1, alternating) and uniform residues."""
import random

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


def sub_root(e, logn, negacyclic=False):
    """root of order 2^logn (cyclic) or psi of order 2^(logn+1) from a params entry"""
    q, L = e["q"], e["logn"]
    if negacyclic:
        assert logn <= L
        return pow(e["psi"], 1 << (L - logn), q)
    assert logn <= L + 1
    return pow(e["psi"], 1 << (L + 1 - logn), q)


def structured(q, n):
    return {
        "delta": [1] + [0] * (n - 1),
        "ones": [1] * n,
        "qm1": [q - 1] * n,
        "alt": [0, q - 1] * (n // 2) if n > 1 else [0],
        "geom": [pow(3, j, q) for j in range(n)],
    }


def run_cyclic(N, q, w, logn, batch, seed):
    n = 1 << logn
    x = synth.uniform_residues(q, n * batch, seed).reshape(batch, n, 2)
    plan = N.Plan(logn, q, w, batch=batch)
    dx = to_dev(x)
    dy = plan.forward(dx)
    y = to_host(dy)
    ref = O.ntt(x, [q] * batch, [w] * batch)
    assert np.array_equal(y, ref), f"forward mismatch N=2^{logn} q={hex(q)}"
    xr = to_host(plan.inverse(dy))
    assert np.array_equal(xr, x), f"inverse mismatch N=2^{logn}"
    return plan


@pytest.mark.parametrize("logn", list(range(1, 13)))
def test_single_pass_sizes(N, params, logn):
    for key in ("b124", "mid127", "rand128_0", "b127"):
        e = params["extra"][key]
        run_cyclic(N, e["q"], sub_root(e, logn), logn, 3, 100 + logn)


@pytest.mark.parametrize("logn", list(range(13, 19)))
def test_two_pass_sizes(N, params, logn):
    for key in ("mid127", "rand128_1"):
        e = params["extra"][key]
        run_cyclic(N, e["q"], sub_root(e, logn), logn, 2, 200 + logn)


@pytest.mark.parametrize("logn", [19, 20, 21, 22])
def test_three_pass_sizes(N, params, logn):
    """three-pass splits of the measured table (5+6+8, 6+6+8, 9+6+6, 6+8+8)"""
    e = params["cfg5"]
    run_cyclic(N, e["q"], sub_root(e, logn), logn, 1, 300 + logn)


def test_small_moduli(N, params):
    for key in ("q17", "q97", "q7681", "q65537"):
        e = params["extra"][key]
        for logn in range(1, e["logn"] + 2):
            if logn > 14:
                break
            run_cyclic(N, e["q"], sub_root(e, logn), logn, 2, 400 + logn)


def test_structured_inputs(N, params):
    for logn in (4, 10, 16):
        e = params["cfg4"]["16"]
        q, w = e["q"], sub_root(e, logn)
        n = 1 << logn
        S = structured(q, n)
        x = np.stack([synth.from_ints(v) for v in S.values()])
        plan = N.Plan(logn, q, w, batch=len(S))
        y = to_host(plan.forward(to_dev(x)))
        assert np.array_equal(y, O.ntt(x, [q] * len(S), [w] * len(S)))
        assert synth.to_ints(y[0]) == [1] * n                      # delta -> ones
        assert synth.to_ints(y[1]) == [n % q] + [0] * (n - 1)     # ones -> [n, 0...]
        assert np.array_equal(to_host(plan.inverse(to_dev(y))), x)


@pytest.mark.parametrize("key", ["b124", "b125", "b126", "b127", "cfg5"])
def test_pseudo_mersenne_class_structured(N, params, key):
    """multi-pass plain cyclic plans whose moduli are all 2^b - c with c 2^(128-b) < 2^32 run the
    pseudo-Mersenne class (csrc/psm128.cuh): structured inputs (q - 1 everywhere, alternating
    0 / q - 1, a geometric sequence) plus uniform ones, every bit length 124..128 and the
    largest fold constant of the parameter set (cfg5's C = 2013265919), vs the oracle"""
    e = params["cfg5"] if key == "cfg5" else params["extra"][key]
    q = e["q"]
    for logn in (13, 17):
        w, n = sub_root(e, logn), 1 << logn
        S = structured(q, n)
        x = np.stack([synth.from_ints(v) for v in S.values()] +
                     [synth.uniform_residues(q, n, 900 + logn).reshape(n, 2)])
        B = x.shape[0]
        plan = N.Plan(logn, q, w, batch=B)
        y = to_host(plan.forward(to_dev(x)))
        assert np.array_equal(y, O.ntt(x, [q] * B, [w] * B))
        assert np.array_equal(to_host(plan.inverse(to_dev(y))), x)


def test_arith_class_query(N, params):
    """ntt128_plan_arith_class: pseudo-Mersenne only when EVERY modulus of a cyclic plan is
    2^b - c with c 2^(128-b) < 2^32; one general prime puts the whole plan in the generic class
    (both plans give the oracle's result either way)"""
    a, b = params["cfg4"]["16"], params["extra"]["rand128_0"]
    logn, n = 13, 1 << 13
    wa, wb = sub_root(a, logn), sub_root(b, logn)
    assert N.Plan(logn, a["q"], wa, batch=2).arith_class() == "pseudo_mersenne"
    assert N.Plan(logn, b["q"], wb, batch=2).arith_class() == "montgomery"
    qs, ws = [a["q"], b["q"]], [wa, wb]
    plan = N.Plan(logn, qs, ws, batch=2)
    assert plan.arith_class() == "montgomery"
    x = np.stack([synth.uniform_residues(q, n, 950 + i).reshape(n, 2) for i, q in enumerate(qs)])
    y = to_host(plan.forward(to_dev(x)))
    assert np.array_equal(y, O.ntt(x, qs, ws))
    assert np.array_equal(to_host(plan.inverse(to_dev(y))), x)


def test_cfg1_full(N, params):
    """BASELINE cfg 1: N = 1024, one polynomial, forward + inverse, natural order"""
    e = params["cfg1"]
    q, w = e["q"], e["omega"]
    x = synth.uniform_residues(q, 1024, synth.stream_seed(1, 0, 0)).reshape(1, 1024, 2)
    plan = N.Plan(10, q, w)
    y = to_host(plan.forward(to_dev(x)))
    assert np.array_equal(y, O.dft(x, q, w))                    # O(N^2) definition
    assert np.array_equal(to_host(plan.inverse(to_dev(y))), x)


def test_cfg3_full_rns(N, params):
    """BASELINE cfg 3: N = 2^16, 64 polynomials, one distinct 124..128-bit prime each"""
    mods = params["cfg3"]["moduli"]
    qs, ws = [m["q"] for m in mods], [m["omega"] for m in mods]
    n, B = 1 << 16, 64
    x = np.stack([synth.uniform_residues(qs[i], n, synth.stream_seed(3, 0, i)) for i in range(B)])
    plan = N.Plan(16, qs, ws, batch=B)
    dy = plan.forward(to_dev(x))
    y = to_host(dy)
    assert np.array_equal(y, O.ntt(x, qs, ws))
    assert np.array_equal(to_host(plan.inverse(dy)), x)


def test_cfg3_negacyclic_polymul(N, params):
    """cfg 3 also: negacyclic a*b mod (X^N + 1, q_i) via NTT . pointwise . INTT (8 polys,
    every stage checked; all 64 in tests/test_gpu_large.py)"""
    mods = params["cfg3"]["moduli"][:8]
    qs, psis = [m["q"] for m in mods], [m["psi"] for m in mods]
    n, B = 1 << 16, len(mods)
    a = np.stack([synth.uniform_residues(qs[i], n, synth.stream_seed(3, 0, 100 + i)) for i in range(B)])
    b = np.stack([synth.uniform_residues(qs[i], n, synth.stream_seed(3, 1, 100 + i)) for i in range(B)])
    plan = N.Plan(16, qs, psis, batch=B, negacyclic=True)
    da, db = to_dev(a), to_dev(b)
    fa = to_host(plan.forward(da))
    assert np.array_equal(fa, O.negacyclic_ntt(a, qs, psis))
    assert np.array_equal(to_host(plan.inverse(to_dev(fa))), a)
    c = to_host(plan.polymul(da, db))
    assert np.array_equal(c, O.negacyclic_polymul(a, b, qs, psis))


@pytest.mark.parametrize("logn", [1, 3, 8, 12, 13, 17])
def test_negacyclic_vs_definition(N, params, logn):
    e = params["extra"]["rand128_0"]
    q, psi = e["q"], sub_root(e, logn, negacyclic=True)
    n = 1 << logn
    x = synth.uniform_residues(q, 2 * n, 500 + logn).reshape(2, n, 2)
    plan = N.Plan(logn, q, psi, batch=2, negacyclic=True)
    y = to_host(plan.forward(to_dev(x)))
    if logn <= 8:
        assert np.array_equal(y[0], O.negacyclic_dft(x[0], q, psi))
    assert np.array_equal(y, O.negacyclic_ntt(x, q, psi))
    assert np.array_equal(to_host(plan.inverse(to_dev(y))), x)
    a, b = x[0:1], synth.uniform_residues(q, n, 600 + logn).reshape(1, n, 2)
    p1 = N.Plan(logn, q, psi, batch=1, negacyclic=True)
    c = to_host(p1.polymul(to_dev(a), to_dev(b)))
    if logn <= 12:
        assert np.array_equal(c[0], O.conv_negacyclic(a[0], b[0], q))
    assert np.array_equal(c, O.negacyclic_polymul(a, b, q, psi))


@pytest.mark.parametrize("logn", [2, 9, 14])
def test_cyclic_polymul(N, params, logn):
    e = params["extra"]["mid127"]
    q, w = e["q"], sub_root(e, logn)
    n = 1 << logn
    a = synth.uniform_residues(q, n, 700 + logn).reshape(1, n, 2)
    b = synth.uniform_residues(q, n, 800 + logn).reshape(1, n, 2)
    plan = N.Plan(logn, q, w)
    c = to_host(plan.polymul(to_dev(a), to_dev(b)))
    ref = O.conv_cyclic(a[0], b[0], q) if logn <= 12 else O.intt(O.vmul(O.ntt(a, q, w), O.ntt(b, q, w), q), q, w)[0]
    assert np.array_equal(c[0], ref)


def test_in_place(N, params):
    e = params["extra"]["b126"]
    for logn in (10, 16):
        q, w = e["q"], sub_root(e, logn)
        x = synth.uniform_residues(q, 2 << logn, 900 + logn).reshape(2, 1 << logn, 2)
        plan = N.Plan(logn, q, w, batch=2)
        d = to_dev(x)
        plan.forward(d, out=d)
        assert np.array_equal(to_host(d), O.ntt(x, [q, q], [w, w]))
        plan.inverse(d, out=d)
        assert np.array_equal(to_host(d), x)


def test_plan_errors(N, params):
    e = params["cfg1"]
    q, w = e["q"], e["omega"]
    with pytest.raises(N.NTT128ArgError, match="INVALID_ARG"):
        N.Plan(0, q, w)
    with pytest.raises(N.NTT128ArgError, match="INVALID_ARG"):
        N.Plan(27, q, w)
    with pytest.raises(N.NTT128ArgError, match="MODULUS"):
        N.Plan(10, q + 1, w)
    with pytest.raises(N.NTT128ArgError, match="NOT_PRIME"):
        N.Plan(10, q + 2 * 2048, w)
    with pytest.raises(N.NTT128ArgError, match="NO_ROOT"):
        N.Plan(12, q, w)                     # 2^12 does not divide q - 1 (v2(q-1) = 11)
    with pytest.raises(N.NTT128ArgError, match="BAD_ROOT"):
        N.Plan(10, q, w * w % q)              # order N/2
    with pytest.raises(N.NTT128ArgError, match="BAD_ROOT"):
        N.Plan(10, q, w, negacyclic=True)     # omega has order N, not 2N
    plan = N.Plan(10, q, w, check_input=True)
    x = synth.uniform_residues(q, 1024, 1).reshape(1, 1024, 2)
    x[0, 7] = [0xFFFFFFFFFFFFFFFF, 0xFFFFFFFFFFFFFFFF]
    with pytest.raises(N.NTT128ArgError, match="INPUT_RANGE"):
        plan.forward(to_dev(x))


@pytest.mark.parametrize("logn", [3, 6, 8, 10, 11, 14])
def test_rns_many_primes_small_sizes(N, params, logn):
    """one distinct prime per polynomial at sizes whose CTAs hold several polynomials
    (single pass, C > 1) -- every polynomial must use its own modulus and twiddles"""
    mods = params["cfg3"]["moduli"][:16]
    qs = [m["q"] for m in mods]
    ws = [sub_root(m, logn) for m in mods]
    psis = [sub_root(m, logn, negacyclic=True) for m in mods]
    n, B = 1 << logn, len(mods)
    x = np.stack([synth.uniform_residues(qs[i], n, 1000 * logn + i) for i in range(B)])
    plan = N.Plan(logn, qs, ws, batch=B)
    y = to_host(plan.forward(to_dev(x)))
    assert np.array_equal(y, O.ntt(x, qs, ws))
    assert np.array_equal(to_host(plan.inverse(to_dev(y))), x)
    pn = N.Plan(logn, qs, psis, batch=B, negacyclic=True)
    yn = to_host(pn.forward(to_dev(x)))
    assert np.array_equal(yn, O.negacyclic_ntt(x, qs, psis))
    b = np.stack([synth.uniform_residues(qs[i], n, 2000 * logn + i) for i in range(B)])
    c = to_host(pn.polymul(to_dev(x), to_dev(b)))
    assert np.array_equal(c, O.negacyclic_polymul(x, b, qs, psis))


@pytest.mark.parametrize("logn,B", [(13, 80), (16, 136), (11, 72)])
def test_rns_more_primes_than_one_launch(N, params, logn, B):
    """more RNS polynomials than one launch's kernel-parameter moduli table (NTT_QMAX = 64):
    multi-pass passes run as chunks of 64 polynomials, each with its own slice
    of data, counters, twiddle tables and moduli; the moduli cycle through the 64 cfg3 primes
    in a shifted order so every chunk mixes all three classes.  Cyclic forward / inverse,
    negacyclic (natural and bit-reversed pipelines) and polymul against the oracle on
    polynomials of every chunk, round trips on all."""
    mods = params["cfg3"]["moduli"]
    idx = [(7 * i + 3) % 64 for i in range(B)]
    qs = [mods[k]["q"] for k in idx]
    ws = [sub_root(mods[k], logn) for k in idx]
    psis = [sub_root(mods[k], logn, negacyclic=True) for k in idx]
    n = 1 << logn
    x = np.stack([synth.uniform_residues(qs[i], n, 3000 * logn + i) for i in range(B)])
    sel = sorted({0, 1, 63, 64, 65, B - 1} | ({127, 128} if B > 128 else set()))
    plan = N.Plan(logn, qs, ws, batch=B)
    y = to_host(plan.forward(to_dev(x)))
    assert np.array_equal(y[sel], O.ntt(x[sel], [qs[i] for i in sel], [ws[i] for i in sel]))
    assert np.array_equal(to_host(plan.inverse(to_dev(y))), x)
    pn = N.Plan(logn, qs, psis, batch=B, negacyclic=True)
    yn = to_host(pn.forward(to_dev(x)))
    assert np.array_equal(yn[sel], O.negacyclic_ntt(x[sel], [qs[i] for i in sel], [psis[i] for i in sel]))
    assert np.array_equal(to_host(pn.inverse(to_dev(yn))), x)
    b = np.stack([synth.uniform_residues(qs[i], n, 4000 * logn + i) for i in range(B)])
    c = to_host(pn.polymul(to_dev(x), to_dev(b)))
    assert np.array_equal(c[sel], O.negacyclic_polymul(x[sel], b[sel], [qs[i] for i in sel], [psis[i] for i in sel]))


@pytest.mark.parametrize("logn", [8, 9, 10, 11])
def test_cluster_latency_path(N, params, logn):
    """up to 512 polynomials at N = 2^8 .. 2^11 run on 8-CTA clusters (distributed shared
    memory exchange between the in-CTA stages and the last three): one to 17 polynomials
    with distinct primes of all classes, in place, and 600 polynomials past the threshold
    (the batched single pass) against 512 at it"""
    e = params["extra"]["rand128_0"]
    q, w = e["q"], sub_root(e, logn)
    n = 1 << logn
    xb = synth.uniform_residues(q, n * 600, 4000 + logn).reshape(600, n, 2)
    ref = O.ntt(xb, [q] * 600, [w] * 600)
    for B in (512, 600):
        plan = N.Plan(logn, q, w, batch=B)
        y = to_host(plan.forward(to_dev(xb[:B])))
        assert np.array_equal(y, ref[:B]), f"B={B}"
        assert np.array_equal(to_host(plan.inverse(to_dev(y))), xb[:B]), f"B={B}"
    mods = params["cfg3"]["moduli"][:17]
    for B in (1, 5, 16, 17):
        qs = [m["q"] for m in mods[:B]]
        ws = [sub_root(m, logn) for m in mods[:B]]
        n = 1 << logn
        x = np.stack([synth.uniform_residues(qs[i], n, 3000 * logn + 10 * B + i) for i in range(B)])
        plan = N.Plan(logn, qs, ws, batch=B)
        d = to_dev(x)
        y = to_host(plan.forward(d))
        assert np.array_equal(y, O.ntt(x, qs, ws)), f"B={B}"
        plan.forward(d, out=d)
        assert np.array_equal(to_host(d), y)
        plan.inverse(d, out=d)
        assert np.array_equal(to_host(d), x), f"B={B}"

"""GPU tests of chained calls (NTT128_FLAG_CHAIN, include/ntt128.h; DESIGN.md §6 "Chained
calls"): a transform's first pass waits per polynomial on the previous call's last-pass
counters instead of on the whole previous grid.

A wrong rule would let a first pass read a polynomial before the previous call wrote it, or
overwrite one a previous call still reads.  Every scenario runs many calls back to back with
no host synchronisation (so the launches really overlap) and compares every result bit-exactly
with the oracle, or with the same call sequence on a plan without the flag: chains of
dependent forward / inverse calls on 2-, 3- and 4-pass plans, the benchmark's rotating buffer
sets, in-place calls, buffers that partially overlap the previous call's (must fall back to
the whole-grid wait), BLAS calls between transforms (library work in between: no chaining
across it), two chained plans interleaved on one stream, polymul through both pipelines, and
stream capture."""
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


def _mods(params, B, logn):
    """first B cfg3 moduli (q = 1 mod 2^17) with roots of order 2^logn (logn <= 16) or the cfg4
    prime of that size repeated (logn = 17..19)"""
    if logn <= 16:
        mods = params["cfg3"]["moduli"][:B]
        return [m["q"] for m in mods], [pow(m["omega"], 1 << (16 - logn), m["q"]) for m in mods]
    e = params["cfg4"][str(logn)] if str(logn) in params["cfg4"] else None
    if e is None:
        e5 = params["cfg5"]
        q, w = e5["q"], pow(e5["omega"], 1 << (26 - logn), e5["q"])
    else:
        q, w = e["q"], e["omega"]
    return [q] * B, [w] * B


def _inputs(qs, n, tag):
    return np.stack([synth.uniform_residues(q, n, synth.stream_seed(7, tag, i)) for i, q in enumerate(qs)])


@pytest.mark.parametrize("logn,B", [(14, 16), (16, 8), (19, 2), (23, 1)])
def test_chained_dependent_calls(N, params, logn, B):
    """forward -> inverse -> forward ... each reading the previous call's output (2, 3 and 4
    passes); every spectrum equals the oracle's, the last inverse equals the input"""
    import torch
    qs, ws = _mods(params, B, logn)
    n = 1 << logn
    x = _inputs(qs, n, logn)
    ref = O.ntt(x, qs, ws) if logn <= 19 else None
    plan = N.Plan(logn, qs, ws, batch=B, chain=True)
    cur = to_dev(x)
    spectra = []
    for _ in range(8 if logn <= 19 else 3):
        y = plan.forward(cur)
        spectra.append(y)
        cur = plan.inverse(y)
    torch.cuda.synchronize()
    if ref is not None:
        for y in spectra:
            assert np.array_equal(to_host(y), ref)
    else:   # N = 2^23: spectra agree with an unchained plan's
        ref_t = N.Plan(logn, qs, ws, batch=B).forward(to_dev(x))
        for y in spectra:
            assert torch.equal(y, ref_t)
    assert np.array_equal(to_host(cur), x)


def test_chained_rotating_sets(N, params):
    """the benchmark's step (forward X[k] -> Y[k], inverse Y[k] -> Z[k], k rotating over 4
    buffer sets), 24 steps without a sync"""
    import torch
    qs, ws = _mods(params, 16, 16)
    n, B = 1 << 16, 16
    xs = [_inputs(qs, n, 100 + k) for k in range(4)]
    refs = [O.ntt(x, qs, ws) for x in xs]
    plan = N.Plan(16, qs, ws, batch=B, chain=True)
    X = [to_dev(x) for x in xs]
    Y = [torch.empty_like(t) for t in X]
    Z = [torch.empty_like(t) for t in X]
    snaps = []
    for i in range(24):
        k = i % 4
        plan.forward(X[k], out=Y[k])
        plan.inverse(Y[k], out=Z[k])
        if i >= 20:
            snaps.append((k, Y[k].clone(), Z[k].clone()))
    torch.cuda.synchronize()
    for k, y, z in snaps:
        assert np.array_equal(to_host(y), refs[k])
        assert np.array_equal(to_host(z), xs[k])


def test_chained_in_place(N, params):
    """in-place forward / inverse (a stream-ordered copy into scratch, then the passes)"""
    import torch
    qs, ws = _mods(params, 8, 16)
    x = _inputs(qs, 1 << 16, 200)
    ref = O.ntt(x, qs, ws)
    plan = N.Plan(16, qs, ws, batch=8, chain=True)
    t = to_dev(x)
    snaps = []
    for _ in range(6):
        plan.forward(t, out=t)
        snaps.append(t.clone())
        plan.inverse(t, out=t)
    torch.cuda.synchronize()
    for y in snaps:
        assert np.array_equal(to_host(y), ref)
    assert np.array_equal(to_host(t), x)


def test_chained_partial_overlap_falls_back(N, params):
    """the second call's input starts one polynomial into the first call's output: the
    per-polynomial order would pair the wrong slices, so the call must wait for the grid"""
    import torch
    qs, ws = _mods(params, 1, 16)
    n, B = 1 << 16, 8
    qs, ws = qs * B, ws * B
    x = _inputs(qs, n, 300)
    plan = N.Plan(16, qs[0], ws[0], batch=B, chain=True)
    big = torch.zeros((B + 1, n, 2), dtype=torch.int64, device="cuda")
    src = to_dev(x)
    outs = []
    for _ in range(4):
        plan.forward(src, out=big[:B])                        # writes polynomials 0..B-1 of big
        z = plan.inverse(big[1:])                             # reads polynomials 1..B of big
        outs.append(z)
    torch.cuda.synchronize()
    bh = np.zeros(((B + 1), n, 2), dtype=np.uint64)
    bh[:B] = O.ntt(x, qs, ws)
    ref = O.intt(bh[1:], qs, ws)
    for z in outs:
        assert np.array_equal(to_host(z).reshape(B, n, 2), ref)


def test_chained_blas_between(N, params):
    """library BLAS calls between chained transforms (they read the spectrum and write the
    next transform's input): the transform after them must not chain across them"""
    import torch
    qs, ws = _mods(params, 1, 16)
    q, w = qs[0], ws[0]
    n, B = 1 << 16, 8
    x = np.stack([synth.uniform_residues(q, n, synth.stream_seed(7, 400, i)) for i in range(B)])
    c = np.stack([synth.uniform_residues(q, n, synth.stream_seed(7, 401, i)) for i in range(B)])
    res = {}
    for chain in (False, True):
        plan = N.Plan(16, q, w, batch=B, chain=chain)
        cur, dc = to_dev(x), to_dev(c)
        outs = []
        for _ in range(5):
            y = plan.forward(cur)
            prod = N.vmul(y, dc, q)            # reads y, writes prod
            cur = plan.inverse(prod)           # reads prod
            outs.append(cur)
        torch.cuda.synchronize()
        res[chain] = [to_host(t) for t in outs]
    for a, b in zip(res[False], res[True]):
        assert np.array_equal(a, b)
    # one step against the oracle: inverse(forward(x) * c) is the cyclic product x * intt(c)
    y = O.ntt(x, [q] * B, [w] * B)
    prod = O.vmul(y.reshape(-1, 2), c.reshape(-1, 2), q).reshape(B, n, 2)
    assert np.array_equal(res[True][0], O.intt(prod, [q] * B, [w] * B))


def test_two_chained_plans_interleaved(N, params):
    """plans A and B (same shape, separate counters) alternate on one stream, each reading the
    other's output: a call after the other plan's call must wait for that grid"""
    import torch
    qs, ws = _mods(params, 8, 14)
    x = _inputs(qs, 1 << 14, 500)
    ref = O.ntt(x, qs, ws)
    A = N.Plan(14, qs, ws, batch=8, chain=True)
    Bp = N.Plan(14, qs, ws, batch=8, chain=True)
    cur = to_dev(x)
    spectra = []
    for i in range(8):
        p1, p2 = (A, Bp) if i % 2 == 0 else (Bp, A)
        y = p1.forward(cur)
        spectra.append(y)
        cur = p2.inverse(y)
    torch.cuda.synchronize()
    for y in spectra:
        assert np.array_equal(to_host(y), ref)
    assert np.array_equal(to_host(cur), x)


@pytest.mark.parametrize("logn", [9, 14, 16])
def test_chained_polymul(N, params, logn):
    """negacyclic polymul (2^9: natural-order path; 2^14, 2^16: the bit-reversed pipeline),
    c aliasing a, repeated: a <- a * b; against the unchained plan and the oracle"""
    import torch
    B = 4
    mods = params["cfg3"]["moduli"][:B]
    qs = [m["q"] for m in mods]
    psis = [pow(m["psi"], 1 << (16 - logn), m["q"]) for m in mods]
    n = 1 << logn
    a = _inputs(qs, n, 600 + logn)
    b = _inputs(qs, n, 700 + logn)
    res = {}
    for chain in (False, True):
        plan = N.Plan(logn, qs, psis, batch=B, negacyclic=True, chain=chain)
        da, db = to_dev(a), to_dev(b)
        snaps = []
        for _ in range(4):
            plan.polymul(da, db, out=da)
            snaps.append(da.clone())
        torch.cuda.synchronize()
        res[chain] = [to_host(t) for t in snaps]
    for u, v in zip(res[False], res[True]):
        assert np.array_equal(u, v)
    if logn <= 9:
        ref = np.stack([O.conv_negacyclic(a[i], b[i], qs[i]) for i in range(B)])
        assert np.array_equal(res[True][0], ref)


def test_chained_plan_under_capture(N, params):
    """a chained plan captured into a CUDA graph (counters are bypassed there) and replayed"""
    import torch
    qs, ws = _mods(params, 8, 16)
    x = _inputs(qs, 1 << 16, 800)
    ref = O.ntt(x, qs, ws)
    plan = N.Plan(16, qs, ws, batch=8, chain=True)
    dx = to_dev(x)
    dy, dz = torch.empty_like(dx), torch.empty_like(dx)
    plan.forward(dx, out=dy)
    plan.inverse(dy, out=dz)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            plan.forward(dx, out=dy)
            plan.inverse(dy, out=dz)
    dy.zero_()
    dz.zero_()
    g.replay()
    plan.forward(dz, out=dy)    # a direct chained call after a replay
    torch.cuda.synchronize()
    assert np.array_equal(to_host(dy), ref)
    assert np.array_equal(to_host(dz), x)

"""GPU tests of the pass-overlap machinery of multi-pass transforms:
programmatic dependent launch plus per-stream, per-polynomial completion counters.

A wrong counter target or a missing acquire/release would let a later pass read a
polynomial before the previous pass wrote it; these tests run many transforms back to
back without host synchronisation (so launches really overlap), on two streams that
share one plan, and under CUDA-graph capture (where the counters are bypassed), and
compare every result bit-exactly with the oracle / the round trip."""
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


def _cfg3_subset(params, B, logn=16):
    """first B cfg3 moduli with roots of order 2^logn (omega is of order 2^16)"""
    mods = params["cfg3"]["moduli"][:B]
    return [m["q"] for m in mods], [pow(m["omega"], 1 << (16 - logn), m["q"]) for m in mods]


def test_back_to_back_chain(N, params):
    """32 forward/inverse transforms chained on one stream with no host sync: each
    forward reads the previous inverse's output; all intermediate spectra checked"""
    import torch
    qs, ws = _cfg3_subset(params, 16, 14)
    n, B = 1 << 14, 16
    x = np.stack([synth.uniform_residues(qs[i], n, synth.stream_seed(3, 0, 500 + i)) for i in range(B)])
    ref = O.ntt(x, qs, ws)
    plan = N.Plan(14, qs, ws, batch=B)
    cur = to_dev(x)
    spectra = []
    for _ in range(16):
        y = plan.forward(cur)
        spectra.append(y)
        cur = plan.inverse(y)
    torch.cuda.synchronize()
    for y in spectra:
        assert np.array_equal(to_host(y), ref)
    assert np.array_equal(to_host(cur), x)


def test_two_streams_share_plan(N, params):
    """one plan, two streams with independent work in flight at once"""
    import torch
    qs, ws = _cfg3_subset(params, 8)
    n, B = 1 << 16, 8
    xa = np.stack([synth.uniform_residues(qs[i], n, synth.stream_seed(3, 0, 600 + i)) for i in range(B)])
    xb = np.stack([synth.uniform_residues(qs[i], n, synth.stream_seed(3, 1, 600 + i)) for i in range(B)])
    plan = N.Plan(16, qs, ws, batch=B)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    da, db = to_dev(xa), to_dev(xb)
    torch.cuda.synchronize()
    outs = {"a": [], "b": []}
    for _ in range(6):
        with torch.cuda.stream(s1):
            ya = plan.forward(da)
            outs["a"].append(ya)
            da = plan.inverse(ya)
        with torch.cuda.stream(s2):
            yb = plan.forward(db)
            outs["b"].append(yb)
            db = plan.inverse(yb)
    torch.cuda.synchronize()
    ra, rb = O.ntt(xa, qs, ws), O.ntt(xb, qs, ws)
    for y in outs["a"]:
        assert np.array_equal(to_host(y), ra)
    for y in outs["b"]:
        assert np.array_equal(to_host(y), rb)
    assert np.array_equal(to_host(da), xa) and np.array_equal(to_host(db), xb)


def test_graph_capture_replay(N, params):
    """transforms captured in a CUDA graph (counters bypassed) replay correctly many times"""
    import torch
    qs, ws = _cfg3_subset(params, 4, 15)
    n, B = 1 << 15, 4
    x = np.stack([synth.uniform_residues(qs[i], n, synth.stream_seed(3, 0, 700 + i)) for i in range(B)])
    plan = N.Plan(15, qs, ws, batch=B)
    dx = to_dev(x)
    dy, dz = torch.empty_like(dx), torch.empty_like(dx)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        plan.forward(dx, out=dy)          # warm the stream's state outside the capture
        plan.inverse(dy, out=dz)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.forward(dx, out=dy)
        plan.inverse(dy, out=dz)
    ref = O.ntt(x, qs, ws)
    for _ in range(5):
        dy.zero_()
        dz.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(to_host(dy), ref)
        assert np.array_equal(to_host(dz), x)


def test_three_pass_chain(N, params):
    """three-pass plan (N = 2^20): counters between passes 1->2 and 2->3"""
    import torch
    e = params["cfg5"]
    q, L = e["q"], e["logn"]
    w = pow(e["psi"], 1 << (L + 1 - 20), q)
    n, B = 1 << 20, 2
    x = synth.uniform_residues(q, n * B, synth.stream_seed(5, 0, 800)).reshape(B, n, 2)
    plan = N.Plan(20, q, w, batch=B)
    cur = to_dev(x)
    ys = []
    for _ in range(4):
        y = plan.forward(cur)
        ys.append(y)
        cur = plan.inverse(y)
    torch.cuda.synchronize()
    ref = O.ntt(x, [q] * B, [w] * B)
    for y in ys:
        assert np.array_equal(to_host(y), ref)
    assert np.array_equal(to_host(cur), x)


def test_graph_capture_in_place_and_polymul(N, params):
    """in-place multi-pass transforms and polymul captured in a CUDA graph: their scratch is
    a graph-owned stream-ordered allocation (no per-stream cache lookup under capture)"""
    import torch
    mods = params["cfg3"]["moduli"][:4]
    qs, psis = [m["q"] for m in mods], [m["psi"] for m in mods]
    ws = [pow(m["omega"], 2, m["q"]) for m in mods]          # order 2^15
    n, B = 1 << 15, 4
    x = np.stack([synth.uniform_residues(qs[i], n, synth.stream_seed(3, 0, 800 + i)) for i in range(B)])
    b = np.stack([synth.uniform_residues(qs[i], n, synth.stream_seed(3, 1, 800 + i)) for i in range(B)])
    plan = N.Plan(15, qs, ws, batch=B)
    pn = N.Plan(15, qs, [pow(p, 2, q) for p, q in zip(psis, qs)], batch=B, negacyclic=True)
    d, da, db, dc = to_dev(x), to_dev(x), to_dev(b), torch.empty_like(to_dev(x))
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.forward(d, out=d)
        pn.polymul(da, db, out=dc)
    ref = O.ntt(x, qs, ws)
    refc = O.negacyclic_polymul(x, b, qs, [pow(p, 2, q) for p, q in zip(psis, qs)])
    for _ in range(3):
        d.copy_(to_dev(x))
        dc.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(to_host(d), ref)
        assert np.array_equal(to_host(dc), refc)

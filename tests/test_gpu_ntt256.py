"""GPU parity of the wider-modulus path (ntt256_*, vec256_mul) against
the 256-bit oracle (oracle/oracle256.c), bit-exact: single-pass sizes, two- and three-pass
schedules, 256/255/254/192/190-bit primes (moduli < 2^192 run the 6-word arithmetic; plans whose
moduli are all < R/4 -- b254 on 8 words, b190 on 6 -- run the lazy class, values in [0, 4q)
between stages), several moduli per batch, structured inputs, in place, and the plan's
argument checks."""
import numpy as np
import pytest

from oracle import oracle256 as O4
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def N():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2509_12494_b200 import ntt128
    return ntt128


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint64)


def root(e, logn):
    return pow(e["omega"], 1 << (e["logn"] - logn), e["q"])


def run(N, qs, ws, logn, x):
    B = x.shape[0]
    plan = N.Plan256(logn, qs if len(qs) > 1 else qs[0], ws if len(ws) > 1 else ws[0], batch=B)
    dy = plan.forward(dev(x))
    y = host(dy)
    ref = O4.ntt(x, qs, ws, small=logn <= 6)
    assert np.array_equal(y, ref), f"forward mismatch N=2^{logn}"
    assert np.array_equal(host(plan.inverse(dy)), x), f"inverse mismatch N=2^{logn}"


@pytest.mark.parametrize("logn", [1, 2, 3, 5, 8, 9, 11, 13, 16])
def test_ntt256_sizes(N, params, logn):
    for key in ("b256", "b192", "b254", "b190"):
        e = params["w256"][key]
        x = synth.uniform_residues_w(e["q"], 2 << logn, 2000 + logn).reshape(2, 1 << logn, 4)
        run(N, [e["q"]], [root(e, logn)], logn, x)


@pytest.mark.parametrize("key", ["b255", "b192", "b254", "b190"])
def test_ntt256_three_pass(N, params, key):
    """three passes (6 + 6 + 6); b192 (q < 2^192) runs the 6-word kernels, b254 / b190 the
    lazy class (two passes on [0, 4q) values before the canonicalising last pass)"""
    e = params["w256"][key]
    logn = 18
    x = synth.uniform_residues_w(e["q"], 1 << logn, 2100).reshape(1, 1 << logn, 4)
    run(N, [e["q"]], [root(e, logn)], logn, x)


@pytest.mark.parametrize("key", ["b192", "b190", "b254"])
def test_ntt192_structured_and_in_place(N, params, key):
    """6-word plans (b192 canonical, b190 lazy) and the 8-word lazy class (b254): delta ->
    ones, all q-1 (the largest values every stage can see), in place"""
    import torch
    e = params["w256"][key]
    q, logn = e["q"], 11
    n = 1 << logn
    x = np.stack([O4.to_array([1] + [0] * (n - 1)), O4.to_array([q - 1] * n),
                  synth.uniform_residues_w(q, n, 2500)])
    run(N, [q], [root(e, logn)], logn, x)
    plan = N.Plan256(logn, q, root(e, logn), batch=3)
    d = dev(x)
    plan.forward(d, out=d)
    assert O4.to_ints(host(d)[0]) == [1] * n
    assert np.array_equal(host(d), O4.ntt(x, q, root(e, logn)))
    plan.inverse(d, out=d)
    assert torch.equal(d, dev(x))


def test_ntt256_many_moduli_and_structured(N, params):
    keys = ["b256", "b255", "b254", "b192"]
    logn = 10
    qs = [params["w256"][k]["q"] for k in keys]
    ws = [root(params["w256"][k], logn) for k in keys]
    n = 1 << logn
    rows = [synth.uniform_residues_w(qs[0], n, 2200), O4.to_array([1] + [0] * (n - 1)),
            O4.to_array([qs[2] - 1] * n), synth.uniform_residues_w(qs[3], n, 2201)]
    x = np.stack(rows)
    run(N, qs, ws, logn, x)
    plan = N.Plan256(logn, qs, ws, batch=4)
    y = host(plan.forward(dev(x)))
    assert O4.to_ints(y[1]) == [1] * n                       # delta -> ones


@pytest.mark.parametrize("logn", [9, 12, 17])
def test_ntt256_lazy_many_moduli(N, params, logn):
    """a lazy 8-word plan with several moduli (b254, b192, b190 < 2^254: moduli from the device
    table, not the kernel parameter), 1-3 passes, all-(q-1) and uniform rows"""
    keys = ["b254", "b192", "b190"]
    qs = [params["w256"][k]["q"] for k in keys]
    ws = [root(params["w256"][k], logn) for k in keys]
    n = 1 << logn
    x = np.stack([O4.to_array([qs[0] - 1] * n), synth.uniform_residues_w(qs[1], n, 2600 + logn),
                  synth.uniform_residues_w(qs[2], n, 2700 + logn)])
    run(N, qs, ws, logn, x)


def test_ntt256_in_place(N, params):
    import torch
    e = params["w256"]["b254"]
    logn = 12
    x = synth.uniform_residues_w(e["q"], 1 << logn, 2300).reshape(1, 1 << logn, 4)
    plan = N.Plan256(logn, e["q"], root(e, logn))
    d = dev(x)
    plan.forward(d, out=d)
    assert np.array_equal(host(d), O4.ntt(x, e["q"], root(e, logn)))
    plan.inverse(d, out=d)
    assert torch.equal(d, dev(x))


def test_vmul256(N, params):
    for key in ("b256", "b192"):
        q = params["w256"][key]["q"]
        x = synth.uniform_residues_w(q, 5000, 2400)
        y = synth.uniform_residues_w(q, 5000, 2401)
        edge = O4.to_array([0, 1, q - 1, q - 2, (q + 1) // 2, (1 << 128) - 1, 1 << 128])
        x = np.concatenate([x, np.repeat(edge, len(edge), axis=0)])
        y = np.concatenate([y, np.tile(edge, (len(edge), 1))])
        got = host(N.vmul256(dev(x), dev(y), q))
        assert np.array_equal(got, O4.vmul(x, y, q))
        assert O4.to_ints(got[:50]) == [a * b % q for a, b in zip(O4.to_ints(x[:50]), O4.to_ints(y[:50]))]


def test_plan256_errors(N, params):
    e = params["w256"]["b256"]
    q = e["q"]
    with pytest.raises(N.NTT128ArgError, match="INVALID_ARG"):
        N.Plan256(25, q, root(e, 20))
    with pytest.raises(N.NTT128ArgError, match="MODULUS"):
        N.Plan256(4, q + 1, root(e, 4))
    with pytest.raises(N.NTT128ArgError, match="NOT_PRIME"):
        N.Plan256(4, q - 2, root(e, 4))
    with pytest.raises(N.NTT128ArgError, match="BAD_ROOT"):
        N.Plan256(4, q, root(e, 3))                            # order 8, not 16

"""Element-wise parity at the largest sizes and at the benchmarked batches (the paper's
criterion is bitwise-identical results; SURVEY.md §8(c) "Parity procedure"):

* BASELINE cfg 5, N = 2^26: the FULL output of the three-pass plan, of the four-step at
  G = 1 and of the four-step over 8 virtual ranks (both transports, and the natural block
  layout at G = 1 and 8) against the oracle's
  textbook radix-2 `ntt_large`, itself pinned at sampled outputs by direct O(N)
  evaluation of Eq. ntt, which shares no structure with any radix
  algorithm; exact round trips;
* cyclic N = 2^23, 2^24 (8+8+8) and 2^25 (9+8+8): full outputs;
* BASELINE cfg 4: every size N = 2^10 .. 2^17 at the batch the bench times (B = 2^26 / N,
  1 GiB): 8 seeded polynomials spread over the batch against the oracle, the whole batch
  round-tripped on the device;
* BASELINE cfg 3 negacyclic polymul on all 64 polynomials (64 distinct primes).
"""
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


@pytest.fixture(scope="module")
def cfg5(params):
    """cfg 5 input and its oracle spectrum, computed once for the module (~2 min of host work)"""
    e = params["cfg5"]
    q, w = e["q"], e["omega"]
    n = 1 << 26
    x = synth.uniform_residues(q, n, synth.stream_seed(5, 0, 900))
    y = O.ntt_large(x, q, w)
    # pin the oracle's radix-2 output at this size by the definition (~8 s of host work per point)
    rng = np.random.default_rng(26)
    ks = [0, 1, n - 1, int(rng.integers(0, n))]
    for k in ks:
        assert synth.to_ints(y[k:k + 1])[0] == O.ntt_eval(x, q, w, k), f"oracle ntt_large vs Eq. ntt at k={k}"
    return q, w, x, y


def test_cfg5_three_pass_full(N, cfg5):
    import torch
    q, w, x, y = cfg5
    plan = N.Plan(26, q, w)
    dx = to_dev(x.reshape(1, -1, 2))
    dy = plan.forward(dx)
    assert np.array_equal(to_host(dy).reshape(-1, 2), y), "three-pass N=2^26 forward != oracle"
    assert torch.equal(plan.inverse(dy), dx), "three-pass N=2^26 round trip"


def test_cfg5_fourstep_g1_full(N, cfg5):
    import torch
    from paper_2509_12494_b200 import fourstep as FS
    q, w, x, y = cfg5
    l1, l2 = FS.split(26)
    n1, n2 = 1 << l1, 1 << l2
    for transport in ("nccl", "p2p"):
        fs = FS.FourStep(26, q, w, transport=transport)
        cols = to_dev(FS.to_columns(x, n1, n2, 0, 1))
        rows = fs.forward(cols)
        assert np.array_equal(FS.from_rows([to_host(rows)], n1, n2), y), f"four-step G=1 ({transport}) != oracle"
        assert torch.equal(fs.inverse(rows), cols), f"four-step G=1 ({transport}) round trip"
        del fs, cols, rows
        torch.cuda.empty_cache()


@pytest.mark.parametrize("peers", [False, True])
def test_cfg5_fourstep_virtual_g8_full(N, cfg5, peers):
    import torch
    from paper_2509_12494_b200 import fourstep as FS
    from tests.test_gpu_fourstep import virtual_run, virtual_run_peers
    q, w, x, y = cfg5
    yv, xr = (virtual_run_peers if peers else virtual_run)(FS, 26, q, w, x, 8)
    assert np.array_equal(yv, y), f"four-step virtual G=8 (peers={peers}) != oracle"
    assert np.array_equal(xr, x), f"four-step virtual G=8 (peers={peers}) round trip"
    torch.cuda.empty_cache()


@pytest.mark.parametrize("world", [1, 8])
def test_cfg5_fourstep_natural_layout_full(N, cfg5, world):
    """natural block layout: rank g's slices of x in, of y out"""
    import torch
    from paper_2509_12494_b200 import fourstep as FS
    from tests.test_gpu_fourstep import virtual_run_natural
    q, w, x, y = cfg5
    yv, xr = virtual_run_natural(FS, 26, q, w, x, world)
    assert np.array_equal(yv, y), f"four-step natural layout, virtual G={world} != oracle"
    assert np.array_equal(xr, x), f"four-step natural layout, virtual G={world} round trip"
    torch.cuda.empty_cache()


@pytest.mark.parametrize("logn", [23, 24, 25])
def test_cyclic_large_full(N, params, logn):
    """three-pass splits 9+6+8 (2^23), 8+8+8 (2^24), 9+8+8 (2^25): full outputs"""
    import torch
    e = params["cfg5"]
    q = e["q"]
    w = pow(e["omega"], 1 << (26 - logn), q)
    n = 1 << logn
    x = synth.uniform_residues(q, n, 3000 + logn)
    plan = N.Plan(logn, q, w)
    dx = to_dev(x.reshape(1, n, 2))
    dy = plan.forward(dx)
    assert np.array_equal(to_host(dy).reshape(-1, 2), O.ntt_large(x, q, w)), f"N=2^{logn} forward != oracle"
    assert torch.equal(plan.inverse(dy), dx), f"N=2^{logn} round trip"


@pytest.mark.parametrize("logn", list(range(10, 18)))
def test_cfg4_benchmarked_batch(N, params, logn):
    """the exact launch configuration bench.py times for cfg 4: B = 2^26 / N polynomials"""
    import torch
    e = params["cfg4"][str(logn)]
    q, w = e["q"], e["omega"]
    n = 1 << logn
    B = (1 << 26) // n
    x = synth.uniform_residues(q, 1 << 26, synth.stream_seed(4, 0, logn)).reshape(B, n, 2)
    plan = N.Plan(logn, q, w, batch=B)
    dx = to_dev(x)
    dy = plan.forward(dx)
    rng = np.random.default_rng(logn)
    idx = sorted({0, B - 1, B // 2} | {int(v) for v in rng.integers(0, B, 5)})
    sel = torch.tensor(idx, device=dy.device)
    got = to_host(dy.index_select(0, sel))
    ref = O.ntt(np.ascontiguousarray(x[idx]), [q] * len(idx), [w] * len(idx))
    assert np.array_equal(got, ref), f"cfg4 N=2^{logn} x {B}: sampled polynomials {idx} != oracle"
    assert torch.equal(plan.inverse(dy), dx), f"cfg4 N=2^{logn} x {B}: round trip"
    del plan, dx, dy
    torch.cuda.empty_cache()


def test_cfg3_polymul_all_64(N, params):
    """BASELINE cfg 3 negacyclic polymul: every one of the 64 polynomials (own prime each)"""
    mods = params["cfg3"]["moduli"]
    qs, psis = [m["q"] for m in mods], [m["psi"] for m in mods]
    n, B = 1 << 16, 64
    a = np.stack([synth.uniform_residues(qs[i], n, synth.stream_seed(3, 0, i)) for i in range(B)])
    b = np.stack([synth.uniform_residues(qs[i], n, synth.stream_seed(3, 1, i)) for i in range(B)])
    plan = N.Plan(16, qs, psis, batch=B, negacyclic=True)
    c = to_host(plan.polymul(to_dev(a), to_dev(b)))
    assert np.array_equal(c, O.negacyclic_polymul(a, b, qs, psis))


def test_small_q_add_sub_exhaustive(N, params):
    """vec128_add / vec128_sub over ALL q^2 pairs (a, b) for q = 65537 (SURVEY.md §8(c)
    pin table: 'exhaustive over all (a, b) for small q ... on GPU'), against Eq. saddmod /
    ssubmod written out on int64 tensors: (a + b) mod q and (a - b) mod q"""
    import torch
    q = 65537
    total = q * q
    chunk = 1 << 25
    for i0 in range(0, total, chunk):
        m = min(chunk, total - i0)
        i = torch.arange(i0, i0 + m, device="cuda", dtype=torch.int64)
        a, b = i // q, i % q
        x = torch.stack([a, torch.zeros_like(a)], 1)
        y = torch.stack([b, torch.zeros_like(b)], 1)
        s = N.vadd(x, y, q)
        d = N.vsub(x, y, q)
        assert torch.equal(s[:, 0], (a + b) % q) and not s[:, 1].any(), f"vec128_add, pairs [{i0}, {i0 + m})"
        assert torch.equal(d[:, 0], (a - b) % q) and not d[:, 1].any(), f"vec128_sub, pairs [{i0}, {i0 + m})"

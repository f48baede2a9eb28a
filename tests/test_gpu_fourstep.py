"""GPU parity of the four-step transform (ntt128_fourstep_*, cfg 5) against the oracle:
G = 1, and G = 2/4/8 emulated on one GPU (the ranks run one after another; the
all-to-all is done by block copies between their buffers)."""
import numpy as np
import pytest

from oracle import oracle as O
import synth
from tests._util import to_dev, to_host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def FS():
    import torch
    assert torch.cuda.is_available()
    from paper_2509_12494_b200 import fourstep
    return fourstep


def virtual_run(FS, log2n, q, w, x, world):
    import torch
    l1, l2 = FS.split(log2n)
    n1, n2 = 1 << l1, 1 << l2
    locs = [FS.FourStepLocal(log2n, q, w, r, world) for r in range(world)]
    R1, R2 = n1 // world, n2 // world
    sends = []
    for r, L in enumerate(locs):
        s = torch.empty((world, R1, R2, 2), dtype=torch.int64, device="cuda")
        L.forward_a(to_dev(FS.to_columns(x, n1, n2, r, world)), s)
        sends.append(s)
    rows = []
    for h, L in enumerate(locs):
        recv = torch.stack([sends[g][h] for g in range(world)]).contiguous()
        out = torch.empty((R2, n1, 2), dtype=torch.int64, device="cuda")
        rows.append(L.forward_c(recv, out))
    y = FS.from_rows([to_host(t) for t in rows], n1, n2)
    # inverse back to the column layout
    sends = []
    for r, L in enumerate(locs):
        s = torch.empty((world, R2, R1, 2), dtype=torch.int64, device="cuda")
        L.inverse_a(rows[r], s)
        sends.append(s)
    cols = []
    for g, L in enumerate(locs):
        recv = torch.stack([sends[h][g] for h in range(world)]).contiguous()
        out = torch.empty((R1, n2, 2), dtype=torch.int64, device="cuda")
        cols.append(to_host(L.inverse_c(recv, out)))
    return y, FS.from_columns(cols, n1, n2)


def virtual_run_peers(FS, log2n, q, w, x, world):
    """fused exchange (ntt128_fourstep_*_a_peers): virtual rank g's pack kernel stores its
    blocks straight into every virtual rank's receive buffer (all on this GPU); the ranks
    run one after another, so no kernel waits on another"""
    import torch
    l1, l2 = FS.split(log2n)
    n1, n2 = 1 << l1, 1 << l2
    locs = [FS.FourStepLocal(log2n, q, w, r, world) for r in range(world)]
    R1, R2 = n1 // world, n2 // world
    recvs = [torch.full((world, R1, R2, 2), -1, dtype=torch.int64, device="cuda") for _ in range(world)]
    ptrs = [t.data_ptr() for t in recvs]
    for r, L in enumerate(locs):
        L.forward_a_peers(to_dev(FS.to_columns(x, n1, n2, r, world)), ptrs)
    rows = []
    for h, L in enumerate(locs):
        rows.append(L.forward_c(recvs[h], torch.empty((R2, n1, 2), dtype=torch.int64, device="cuda")))
    y = FS.from_rows([to_host(t) for t in rows], n1, n2)
    recvs = [torch.full((world, R2, R1, 2), -1, dtype=torch.int64, device="cuda") for _ in range(world)]
    ptrs = [t.data_ptr() for t in recvs]
    for r, L in enumerate(locs):
        L.inverse_a_peers(rows[r], ptrs)
    cols = [to_host(L.inverse_c(recvs[g], torch.empty((R1, n2, 2), dtype=torch.int64, device="cuda")))
            for g, L in enumerate(locs)]
    return y, FS.from_columns(cols, n1, n2)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("log2n", [8, 14, 20])
def test_fourstep_fused_exchange_virtual_ranks(FS, params, log2n, world):
    e = params["extra"]["b126"] if log2n <= 17 else params["cfg5"]   # b126: a q < 2^126 (lazy class)
    q = e["q"]
    w = pow(e["psi"], 1 << (e["logn"] + 1 - log2n), q)
    x = synth.uniform_residues(q, 1 << log2n, 400 + log2n + world)
    y, xr = virtual_run_peers(FS, log2n, q, w, x, world)
    assert np.array_equal(y, O.ntt(x, q, w))
    assert np.array_equal(xr, x)


def test_fourstep_p2p_transport_single_rank(FS, params):
    """FourStep(transport="p2p") at world 1 (the rank's own buffer is its only peer)"""
    e = params["cfg5"]
    q, log2n = e["q"], 16
    w = pow(e["omega"], 1 << (26 - log2n), q)
    x = synth.uniform_residues(q, 1 << log2n, 77)
    l1, l2 = FS.split(log2n)
    fs = FS.FourStep(log2n, q, w, transport="p2p")
    rows = fs.forward(to_dev(FS.to_columns(x, 1 << l1, 1 << l2, 0, 1)))
    assert np.array_equal(FS.from_rows([to_host(rows)], 1 << l1, 1 << l2), O.ntt(x, q, w))
    cols = fs.inverse(rows)
    assert np.array_equal(FS.from_columns([to_host(cols)], 1 << l1, 1 << l2), x)


@pytest.mark.parametrize("log2n", [2, 5, 10, 16, 20])
def test_fourstep_g1(FS, params, log2n):
    e = params["cfg5"]
    q = e["q"]
    w = pow(e["omega"], 1 << (26 - log2n), q)
    x = synth.uniform_residues(q, 1 << log2n, 31 + log2n)
    y, xr = virtual_run(FS, log2n, q, w, x, 1)
    assert np.array_equal(y, O.ntt(x, q, w))
    assert np.array_equal(xr, x)


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("log2n", [8, 14])
def test_fourstep_virtual_ranks(FS, params, log2n, world):
    e = params["extra"]["mid127"]
    q = e["q"]
    w = pow(e["psi"], 1 << (e["logn"] + 1 - log2n), q)
    x = synth.uniform_residues(q, 1 << log2n, 300 + log2n + world)
    y, xr = virtual_run(FS, log2n, q, w, x, world)
    assert np.array_equal(y, O.ntt(x, q, w))
    assert np.array_equal(xr, x)


def virtual_run_natural(FS, log2n, q, w, x, world):
    """natural block layout (include/ntt128.h): virtual rank g holds x[g N/G, (g+1) N/G);
    the three all-to-alls per direction are block copies between the ranks' buffers"""
    import torch
    n = 1 << log2n
    locs = [FS.FourStepLocal(log2n, q, w, r, world) for r in range(world)]
    R1, R2 = locs[0].R1, locs[0].R2

    def run(cur, names, blocks):
        for name, shp in zip(names[:3], blocks):
            sends = []
            for r, L in enumerate(locs):
                s = torch.full((world, *shp, 2), -1, dtype=torch.int64, device="cuda")
                getattr(L, name)(cur[r], s)
                sends.append(s)
            cur = [torch.stack([sends[g][h] for g in range(world)]).contiguous() for h in range(world)]
        outs = []
        for r, L in enumerate(locs):
            o = torch.full((n // world, 2), -1, dtype=torch.int64, device="cuda")
            getattr(L, names[3])(cur[r], o)
            outs.append(o)
        return outs

    xs = [to_dev(x[r * n // world:(r + 1) * n // world]) for r in range(world)]
    ys = run(xs, ("forward_pack", "forward_a_nat", "forward_c_nat", "forward_unpack"), ((R2, R1), (R1, R2), (R2, R1)))
    y = np.concatenate([to_host(t) for t in ys])
    xb = run(ys, ("inverse_pack", "inverse_a_nat", "inverse_c_nat", "inverse_unpack"), ((R1, R2), (R2, R1), (R1, R2)))
    return y, np.concatenate([to_host(t) for t in xb])


_ORACLE = {}


def _oracle_ntt(log2n, key, q, w):
    """the oracle's transform of the seed-(500 + log2n) input, computed once per (size, prime)
    for all world sizes (2^22 takes the oracle ~45 s)"""
    if (log2n, key) not in _ORACLE:
        _ORACLE[(log2n, key)] = O.ntt(synth.uniform_residues(q, 1 << log2n, 500 + log2n), q, w)
    return _ORACLE[(log2n, key)]


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("log2n", [8, 13, 17, 22])
def test_fourstep_natural_layout_virtual_ranks(FS, params, log2n, world):
    """natural block layout: concatenated forward slices = the oracle's NTT, exact round trip
    (FULL-class cfg5 prime; a lazy-class prime up to its 2^17 roots; 2^22 = 2^9 x 2^13 has
    multi-pass passes A and C)"""
    for key in (("cfg5", "b126") if log2n <= 17 else ("cfg5",)):
        e = params["cfg5"] if key == "cfg5" else params["extra"]["b126"]
        q = e["q"]
        if key == "cfg5":
            w = pow(e["omega"], 1 << (26 - log2n), q)
        else:
            w = pow(e["psi"], 1 << (e["logn"] + 1 - log2n), q)
        x = synth.uniform_residues(q, 1 << log2n, 500 + log2n)
        y, xr = virtual_run_natural(FS, log2n, q, w, x, world)
        assert np.array_equal(y, _oracle_ntt(log2n, key, q, w)), key
        assert np.array_equal(xr, x), key


def test_fourstep_natural_layout_class(FS, params):
    """FourStep(layout="natural") at world 1: the slice is the whole vector"""
    e = params["cfg5"]
    q, log2n = e["q"], 16
    w = pow(e["omega"], 1 << (26 - log2n), q)
    x = synth.uniform_residues(q, 1 << log2n, 78)
    fs = FS.FourStep(log2n, q, w, layout="natural")
    y = fs.forward(to_dev(x))
    assert np.array_equal(to_host(y), O.ntt(x, q, w))
    assert np.array_equal(to_host(fs.inverse(y)), x)


def test_fourstep_natural_layout_errors(FS, params):
    import torch
    from paper_2509_12494_b200 import ntt128 as N
    e = params["cfg5"]
    q = e["q"]
    w = pow(e["omega"], 1 << 16, q)
    L = FS.FourStepLocal(10, q, w, 0, 2)
    a = torch.zeros((512, 2), dtype=torch.int64, device="cuda")
    with pytest.raises(N.NTT128ArgError):
        L.forward_pack(a, a)          # in-place pack is refused
    with pytest.raises(N.NTT128ArgError):
        L.inverse_unpack(a, a)


def test_fourstep_p2p_symmetric_memory_one_rank(FS, params):
    """the p2p transport's symmetric-memory path (allocation, rendezvous, peer pointers,
    device barriers) on a one-rank NCCL process group: the code a multi-GPU run takes,
    with no rank waiting on another"""
    import socket
    import torch
    import torch.distributed as dist
    if dist.is_initialized():
        pytest.skip("a process group already exists in this process")
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    store = dist.TCPStore("127.0.0.1", port, 1, True)
    dist.init_process_group("nccl", store=store, rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        e = params["cfg5"]
        q, log2n = e["q"], 14
        w = pow(e["omega"], 1 << (26 - log2n), q)
        x = synth.uniform_residues(q, 1 << log2n, 79)
        l1, l2 = FS.split(log2n)
        fs = FS.FourStep(log2n, q, w, transport="p2p", symmetric=True)
        assert fs._hdl is not None and len(fs._peers) == 1
        rows = fs.forward(to_dev(FS.to_columns(x, 1 << l1, 1 << l2, 0, 1)))
        assert np.array_equal(FS.from_rows([to_host(rows)], 1 << l1, 1 << l2), O.ntt(x, q, w))
        cols = fs.inverse(rows)
        assert np.array_equal(FS.from_columns([to_host(cols)], 1 << l1, 1 << l2), x)
        del fs
    finally:
        dist.destroy_process_group()

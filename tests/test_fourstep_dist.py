"""CPU (gloo, world_size 2) test of the distributed four-step's host logic: layouts,
packing order and the all-to-all schedule of paper_2509_12494_b200/fourstep.py, with
an oracle-backed local backend standing in for the rank's kernels (test
infrastructure only).  The composition must equal the oracle's N-point NTT."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
import synth
from paper_2509_12494_b200.fourstep import FourStep, from_columns, from_rows, split, to_columns, to_rows


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64))


def _n(t):
    return t.numpy().view(np.uint64)


class OracleLocal:
    """the semantics of ntt128_fourstep_{forward,inverse}_{a,c} (include/ntt128.h), on the CPU oracle"""

    def __init__(self, log2n, q, w, rank, world):
        self.l1, self.l2 = split(log2n)
        self.n1, self.n2 = 1 << self.l1, 1 << self.l2
        self.N = self.n1 * self.n2
        self.q, self.w, self.rank, self.world = q, w, rank, world
        self.R1, self.R2 = self.n1 // world, self.n2 // world

    def _blocks(self, z, R, C):
        """z[R][C] -> send[G][R][C/G]: block h holds the columns [h C/G, (h+1) C/G)"""
        return np.ascontiguousarray(z.reshape(R, self.world, C // self.world, 2).transpose(1, 0, 2, 3))

    def _twiddle(self, m, row0, w):
        """m[r][c] * w^((row0 + r) c): the four-step twiddle, applied in pass C"""
        R, C = m.shape[0], m.shape[1]
        tw = np.stack([synth.from_ints([pow(w, ((row0 + r) * c) % self.N, self.q) for c in range(C)]) for r in range(R)])
        return O.vmul(np.ascontiguousarray(m).reshape(-1, 2), tw.reshape(-1, 2), self.q).reshape(R, C, 2)

    def forward_a(self, cols, send):
        z = O.ntt(_n(cols), self.q, pow(self.w, self.n1, self.q))          # [R1][n2]
        send.copy_(_t(self._blocks(z, self.R1, self.n2)))

    def forward_c(self, recv, rows):
        m = _n(recv).reshape(self.n1, self.R2, 2).transpose(1, 0, 2)       # [R2][n1]: row cc = k2 = rank R2 + cc
        m = self._twiddle(m, self.rank * self.R2, self.w)
        rows.copy_(_t(O.ntt(m, self.q, pow(self.w, self.n2, self.q))))
        return rows

    def inverse_a(self, rows, send):
        z = O.ntt(_n(rows), self.q, pow(self.w, -self.n2, self.q))        # [R2][n1], unscaled
        send.copy_(_t(self._blocks(z, self.R2, self.n1)))

    def inverse_c(self, recv, cols):
        m = _n(recv).reshape(self.n2, self.R1, 2).transpose(1, 0, 2)       # [R1][n2]: row m = j1 = rank R1 + m
        m = self._twiddle(m, self.rank * self.R1, pow(self.w, -1, self.q))
        m = O.vmul(m.reshape(-1, 2), synth.from_ints([pow(self.N, -1, self.q)] * (m.size // 2)), self.q).reshape(m.shape)
        cols.copy_(_t(O.ntt(m, self.q, pow(self.w, -self.n1, self.q))))   # N^-1 applied with the twiddle
        return cols


    # natural block layout (include/ntt128.h "Natural block layout"): data movement around the
    # same passes, written here with numpy transposes
    def _tr(self, t, R, C):
        """[R][C] (flat t) -> [C][R]"""
        return np.ascontiguousarray(_n(t).reshape(R, C, 2).transpose(1, 0, 2))

    def forward_pack(self, nat, send):
        send.copy_(_t(self._blocks(_n(nat).reshape(self.R2, self.n1, 2), self.R2, self.n1)))

    def forward_a_nat(self, recv, send):
        self.forward_a(_t(self._tr(recv, self.n2, self.R1)), send)

    def forward_c_nat(self, recv, send):
        rows = self.forward_c(recv, torch.empty((self.R2, self.n1, 2), dtype=torch.int64))
        send.copy_(_t(self._blocks(_n(rows), self.R2, self.n1)))

    def forward_unpack(self, recv, nat):
        nat.copy_(_t(self._tr(recv, self.n2, self.R1).reshape(-1, 2)))

    def inverse_pack(self, nat, send):
        send.copy_(_t(self._blocks(_n(nat).reshape(self.R1, self.n2, 2), self.R1, self.n2)))

    def inverse_a_nat(self, recv, send):
        self.inverse_a(_t(self._tr(recv, self.n1, self.R2)), send)

    def inverse_c_nat(self, recv, send):
        cols = self.inverse_c(recv, torch.empty((self.R1, self.n2, 2), dtype=torch.int64))
        send.copy_(_t(self._blocks(_n(cols), self.R1, self.n2)))

    def inverse_unpack(self, recv, nat):
        nat.copy_(_t(self._tr(recv, self.n1, self.R2).reshape(-1, 2)))


def _worker(rank, world, port, log2n, q, w, x, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    l1, l2 = split(log2n)
    n1, n2 = 1 << l1, 1 << l2
    fs = FourStep(log2n, q, w, rank, world, local=OracleLocal(log2n, q, w, rank, world))
    rows = fs.forward(_t(to_columns(x, n1, n2, rank, world)))
    cols = fs.inverse(rows)
    out[rank] = (_n(rows).copy(), _n(cols).copy())
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("log2n,world", [(6, 2), (9, 2)])
def test_fourstep_gloo_world2(params, log2n, world):
    e = params["extra"]["rand128_0"]
    q = e["q"]
    w = pow(e["psi"], 1 << (e["logn"] + 1 - log2n), q)
    n1, n2 = (1 << split(log2n)[0]), (1 << split(log2n)[1])
    x = synth.uniform_residues(q, 1 << log2n, 77 + log2n)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), log2n, q, w, x, out), nprocs=world)
    y = from_rows([out[r][0] for r in range(world)], n1, n2)
    assert np.array_equal(y, O.ntt(x, q, w))
    xr = from_columns([out[r][1] for r in range(world)], n1, n2)
    assert np.array_equal(xr, x)


def _worker_natural(rank, world, port, log2n, q, w, x, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 1 << log2n
    fs = FourStep(log2n, q, w, rank, world, local=OracleLocal(log2n, q, w, rank, world), layout="natural")
    ys = fs.forward(_t(x[rank * n // world:(rank + 1) * n // world]))
    xs = fs.inverse(ys)
    out[rank] = (_n(ys).copy(), _n(xs).copy())
    dist.destroy_process_group()


@pytest.mark.parametrize("log2n,world", [(6, 2), (9, 2), (8, 4)])
def test_fourstep_natural_layout_gloo(params, log2n, world):
    """natural block layout: rank g's forward output is y[g N/G, (g+1) N/G) of the oracle's
    N-point NTT, and the inverse returns each rank its own slice of x"""
    e = params["extra"]["rand128_0"]
    q = e["q"]
    w = pow(e["psi"], 1 << (e["logn"] + 1 - log2n), q)
    x = synth.uniform_residues(q, 1 << log2n, 91 + log2n)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_natural, args=(world, _free_port(), log2n, q, w, x, out), nprocs=world)
    y = np.concatenate([out[r][0] for r in range(world)])
    assert np.array_equal(y, O.ntt(x, q, w))
    assert np.array_equal(np.concatenate([out[r][1] for r in range(world)]), x)


def test_natural_layout_requires_all_to_all():
    with pytest.raises(ValueError):
        FourStep(6, 97, 1, local=object(), transport="p2p", layout="natural")
    with pytest.raises(ValueError):
        FourStep(6, 97, 1, local=object(), layout="rowmajor")


def test_layout_maps_roundtrip():
    x = synth.from_ints(range(64))
    for world in (1, 2, 4):
        parts = [to_columns(x, 8, 8, r, world) for r in range(world)]
        assert np.array_equal(from_columns(parts, 8, 8), x)
        parts = [to_rows(x, 8, 8, r, world) for r in range(world)]
        assert np.array_equal(from_rows(parts, 8, 8), x)
    # X_g[r][j2] = x[(g R1 + r) + n1 j2]
    c = to_columns(x, 8, 8, 1, 2)
    assert synth.to_ints(c[2, 3:4]) == [(1 * 4 + 2) + 8 * 3]

"""Distributed four-step NTT of one huge polynomial over G ranks (one process per GPU).

Binding of the ntt128_fourstep_* C ABI (include/ntt128.h, "Distributed four-step") plus
the host-side exchange: each rank runs its local pass A in the library (its last pass
stores every output into the block of its destination rank), the blocks move with ONE
all-to-all of equal splits (torch.distributed, NCCL over NVLink/NVSwitch on GPUs) -- or,
with transport="p2p", pass A stores them straight into the peers' receive buffers -- then
the local pass C (whose first pass gathers the received columns and applies the
four-step twiddle as it loads).  No arithmetic happens here.

Layouts (N = n1 n2, R1 = n1/G, R2 = n2/G, rank g):
  columns  X_g[r][j2] = x[(g R1 + r) + n1 j2]     (forward input, inverse output)
  rows     Y_g[r][k1] = y[(g R2 + r) + n2 k1]     (forward output, inverse input)
`to_columns` / `from_columns` / `to_rows` / `from_rows` are the pure index maps between
these and natural order (host logic; numpy, no arithmetic).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import ntt128 as _n

_L = _n._L
_vp = ctypes.c_void_p
_L.ntt128_fourstep_create.argtypes = [ctypes.POINTER(_vp), ctypes.c_uint32, ctypes.c_uint32, _n._u64p, _n._u64p,
                                      ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int]
_L.ntt128_fourstep_create.restype = ctypes.c_int
for _name in ("ntt128_fourstep_forward_a", "ntt128_fourstep_forward_c", "ntt128_fourstep_inverse_a",
              "ntt128_fourstep_inverse_c", "ntt128_fourstep_forward_pack", "ntt128_fourstep_forward_a_nat",
              "ntt128_fourstep_forward_c_nat", "ntt128_fourstep_forward_unpack", "ntt128_fourstep_inverse_pack",
              "ntt128_fourstep_inverse_a_nat", "ntt128_fourstep_inverse_c_nat", "ntt128_fourstep_inverse_unpack"):
    getattr(_L, _name).argtypes = [_vp, _vp, _vp, _vp]
    getattr(_L, _name).restype = ctypes.c_int
for _name in ("ntt128_fourstep_forward_a_peers", "ntt128_fourstep_inverse_a_peers"):
    getattr(_L, _name).argtypes = [_vp, _vp, ctypes.POINTER(ctypes.c_uint64), _vp]
    getattr(_L, _name).restype = ctypes.c_int
_L.ntt128_fourstep_destroy.argtypes = [_vp]
_L.ntt128_fourstep_destroy.restype = None


# ----------------------------------------------------------------------------- layouts (host index maps)
def split(log2n: int) -> tuple[int, int]:
    """(log2 n1, log2 n2): n1 = 2^min(9, floor(log2n / 2)) is the length of pass C's forward
    transforms (one 9-stage pass), n2 = N / n1 the length of pass A's (2^9 x 2^17 at
    N = 2^26: pass A two passes 9 + 8, pass C one, the same three passes as the
    single-GPU plan)"""
    l1 = min(9, log2n // 2)
    return l1, log2n - l1


def to_columns(x: np.ndarray, n1: int, n2: int, rank: int, world: int) -> np.ndarray:
    """natural x[N, 2] -> X_rank[R1][n2][2]"""
    R1 = n1 // world
    v = x.reshape(n2, n1, 2)                     # v[j2][j1] = x[j1 + n1 j2]
    return np.ascontiguousarray(v[:, rank * R1:(rank + 1) * R1].transpose(1, 0, 2))


def from_columns(parts, n1: int, n2: int) -> np.ndarray:
    """[X_0 .. X_{G-1}] -> natural x[N, 2]"""
    cols = np.concatenate(parts, axis=0)         # [n1][n2]: cols[j1][j2] = x[j1 + n1 j2]
    return np.ascontiguousarray(cols.transpose(1, 0, 2)).reshape(n1 * n2, 2)


def to_rows(y: np.ndarray, n1: int, n2: int, rank: int, world: int) -> np.ndarray:
    """natural y[N, 2] -> Y_rank[R2][n1][2]"""
    R2 = n2 // world
    v = y.reshape(n1, n2, 2)                     # v[k1][k2] = y[k2 + n2 k1]
    return np.ascontiguousarray(v[:, rank * R2:(rank + 1) * R2].transpose(1, 0, 2))


def from_rows(parts, n1: int, n2: int) -> np.ndarray:
    """[Y_0 .. Y_{G-1}] -> natural y[N, 2]"""
    rows = np.concatenate(parts, axis=0)         # [n2][n1]: rows[k2][k1] = y[k2 + n2 k1]
    return np.ascontiguousarray(rows.transpose(1, 0, 2)).reshape(n1 * n2, 2)


# ----------------------------------------------------------------------------- device object
class FourStepLocal:
    """One rank's share of a four-step transform (ntt128_fourstep_create)."""

    def __init__(self, log2n: int, q: int, omega: int, rank: int = 0, world: int = 1, device: int | None = None):
        import torch
        self.log2n = int(log2n)
        self.l1, self.l2 = split(self.log2n)
        self.n1, self.n2 = 1 << self.l1, 1 << self.l2
        self.rank, self.world = int(rank), int(world)
        self.R1, self.R2 = self.n1 // self.world, self.n2 // self.world
        self.device = torch.cuda.current_device() if device is None else int(device)
        h = _vp()
        self._h = None
        _n._check(_L.ntt128_fourstep_create(ctypes.byref(h), self.l1, self.l2, _n._pairs([q]), _n._pairs([omega]),
                                            self.rank, self.world, self.device), "ntt128_fourstep_create")
        self._h = h

    def _call(self, name, a, b):
        _n._check(getattr(_L, name)(self._h, _n._ptr(a, "in"), _n._ptr(b, "out"), _n._stream(a)), name)
        return b

    def forward_a(self, cols, send):
        return self._call("ntt128_fourstep_forward_a", cols, send)

    def forward_c(self, recv, rows):
        return self._call("ntt128_fourstep_forward_c", recv, rows)

    def inverse_a(self, rows, send):
        return self._call("ntt128_fourstep_inverse_a", rows, send)

    def inverse_c(self, recv, cols):
        return self._call("ntt128_fourstep_inverse_c", recv, cols)

    # natural block layout (include/ntt128.h "Natural block layout"): rank g holds the
    # contiguous slice [g N/G, (g+1) N/G) of x (forward input) and of y (forward output)
    def forward_pack(self, nat, send):
        return self._call("ntt128_fourstep_forward_pack", nat, send)

    def forward_a_nat(self, recv, send):
        return self._call("ntt128_fourstep_forward_a_nat", recv, send)

    def forward_c_nat(self, recv, send):
        return self._call("ntt128_fourstep_forward_c_nat", recv, send)

    def forward_unpack(self, recv, nat):
        return self._call("ntt128_fourstep_forward_unpack", recv, nat)

    def inverse_pack(self, nat, send):
        return self._call("ntt128_fourstep_inverse_pack", nat, send)

    def inverse_a_nat(self, recv, send):
        return self._call("ntt128_fourstep_inverse_a_nat", recv, send)

    def inverse_c_nat(self, recv, send):
        return self._call("ntt128_fourstep_inverse_c_nat", recv, send)

    def inverse_unpack(self, recv, nat):
        return self._call("ntt128_fourstep_inverse_unpack", recv, nat)

    def _call_peers(self, name, a, peer_ptrs):
        if len(peer_ptrs) != self.world:
            raise ValueError(f"{name}: need {self.world} peer pointers, got {len(peer_ptrs)}")
        arr = (ctypes.c_uint64 * self.world)(*[int(p) for p in peer_ptrs])
        _n._check(getattr(_L, name)(self._h, _n._ptr(a, "in"), arr, _n._stream(a)), name)

    def forward_a_peers(self, cols, peer_ptrs):
        """pass A with the exchange fused: block h lands in peer_ptrs[h] (rank h's recv buffer)"""
        self._call_peers("ntt128_fourstep_forward_a_peers", cols, peer_ptrs)

    def inverse_a_peers(self, rows, peer_ptrs):
        self._call_peers("ntt128_fourstep_inverse_a_peers", rows, peer_ptrs)

    def close(self):
        if self._h is not None:
            _L.ntt128_fourstep_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def exchange(send, group=None, world: int = 1):
    """all-to-all of equal blocks along dim 0 (block h -> rank h); world 1 is the identity"""
    if world == 1:
        return send
    import torch
    import torch.distributed as dist
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv.view(-1), send.view(-1), group=group)
    return recv


class FourStep:
    """Distributed forward / inverse of one N-point transform; call on every rank.

    transport="nccl": pass A packs into a local send buffer, one all-to-all moves the
    blocks, pass C reads the received copy.  transport="p2p": the receive
    buffer is symmetric memory (torch.distributed._symmetric_memory, NVLink peer mappings)
    and pass A's pack kernel stores every block straight into its destination rank's
    receive buffer; two device-side barriers order the writes (before: every peer has
    finished reading its buffer; after: every block has landed).  No collective moves data.

    layout="transposed" (default): forward takes the columns layout X_g[R1][n2] and returns
    the rows layout Y_g[R2][n1] (one exchange per direction).  layout="natural" (SURVEY.md
    §8(e)): rank g passes and receives the contiguous slice [g N/G, (g+1) N/G) of x / y as
    [N/G][2]; one more all-to-all at each end (pack -> exchange -> pass A -> exchange ->
    pass C -> exchange -> unpack; include/ntt128.h "Natural block layout").
    """

    def __init__(self, log2n: int, q: int, omega: int, rank: int = 0, world: int = 1, group=None,
                 device: int | None = None, local=None, transport: str = "nccl", layout: str = "transposed",
                 symmetric: bool | None = None):
        # `local` is injectable so the exchange schedule can be exercised by CPU tests (gloo)
        if transport not in ("nccl", "p2p"):
            raise ValueError(f"transport must be 'nccl' or 'p2p', not {transport!r}")
        if layout not in ("transposed", "natural"):
            raise ValueError(f"layout must be 'transposed' or 'natural', not {layout!r}")
        if layout == "natural" and transport != "nccl":
            raise ValueError("the natural block layout exchanges by all-to-all (transport='nccl')")
        self.local = local if local is not None else FourStepLocal(log2n, q, omega, rank, world, device)
        self.group, self.world = group, world
        self.transport, self.layout = transport, layout
        self._recv = self._hdl = None
        # p2p receive buffer: symmetric memory whenever world > 1; `symmetric=True` forces it at
        # world 1 too (a one-rank process group), so a single GPU exercises the same allocation,
        # rendezvous, peer pointers and device barriers
        self._symmetric = (world > 1) if symmetric is None else bool(symmetric)
        if transport == "p2p":
            self._setup_p2p()

    def _setup_p2p(self):
        import torch
        L = self.local
        dev = torch.device("cuda", L.device)
        elems = L.R1 * L.n2                            # = R2 * n1 = N / G: both directions fit
        if not self._symmetric:
            if self.world != 1:
                raise ValueError("transport='p2p' with world > 1 needs symmetric memory")
            self._recv = torch.empty((elems, 2), dtype=torch.int64, device=dev)
            self._peers = [self._recv.data_ptr()]
            return
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        self._recv = symm_mem.empty((elems, 2), dtype=torch.int64, device=dev)
        self._hdl = symm_mem.rendezvous(self._recv, self.group if self.group is not None else dist.group.WORLD)
        self._peers = [int(p) for p in self._hdl.buffer_ptrs]

    def _barrier(self):
        if self._hdl is not None:
            self._hdl.barrier(channel=0, timeout_ms=30000)   # device-side, stream-ordered; errors instead of hanging

    def _natural(self, nat, out, pack, pass_a, pass_c, unpack, blocks):
        """pack -> exchange -> pass A -> exchange -> pass C -> exchange -> unpack; blocks =
        the [rows][cols] shape of one exchange block after pack, pass A and pass C"""
        import torch
        out = torch.empty_like(nat) if out is None else out
        cur = nat
        for step, shp in zip((pack, pass_a, pass_c), blocks):
            send = torch.empty((self.world, *shp, 2), dtype=nat.dtype, device=nat.device)
            step(cur, send)
            cur = exchange(send, self.group, self.world)
        unpack(cur, out)
        return out

    def forward(self, cols, out=None):
        import torch
        L = self.local
        if self.layout == "natural":   # cols: this rank's slice of x, [N/G][2]
            return self._natural(cols, out, L.forward_pack, L.forward_a_nat, L.forward_c_nat, L.forward_unpack,
                                 ((L.R2, L.R1), (L.R1, L.R2), (L.R2, L.R1)))
        out = torch.empty((L.R2, L.n1, 2), dtype=cols.dtype, device=cols.device) if out is None else out
        if self.transport == "p2p":
            self._barrier()
            L.forward_a_peers(cols, self._peers)
            self._barrier()
            return L.forward_c(self._recv.view(self.world, L.R1, L.R2, 2), out)
        send = torch.empty((self.world, L.R1, L.R2, 2), dtype=cols.dtype, device=cols.device)
        L.forward_a(cols, send)
        recv = exchange(send, self.group, self.world)
        return L.forward_c(recv, out)

    def inverse(self, rows, out=None):
        import torch
        L = self.local
        if self.layout == "natural":   # rows: this rank's slice of y, [N/G][2]
            return self._natural(rows, out, L.inverse_pack, L.inverse_a_nat, L.inverse_c_nat, L.inverse_unpack,
                                 ((L.R1, L.R2), (L.R2, L.R1), (L.R1, L.R2)))
        out = torch.empty((L.R1, L.n2, 2), dtype=rows.dtype, device=rows.device) if out is None else out
        if self.transport == "p2p":
            self._barrier()
            L.inverse_a_peers(rows, self._peers)
            self._barrier()
            return L.inverse_c(self._recv.view(self.world, L.R2, L.R1, 2), out)
        send = torch.empty((self.world, L.R2, L.R1, 2), dtype=rows.dtype, device=rows.device)
        L.inverse_a(rows, send)
        recv = exchange(send, self.group, self.world)
        return L.inverse_c(recv, out)

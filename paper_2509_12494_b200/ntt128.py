"""Thin Python binding of libntt128.so (include/ntt128.h): argument marshalling only.

Every step of the transform and the BLAS ops runs in the library's sm_100a kernels.
PyTorch supplies device memory and streams.  There is no CPU fallback: if the
in-tree library is missing this module raises at import time.

Tensors are contiguous CUDA tensors of dtype uint64 or int64 (same bits), shaped
[..., 2] with [lo, hi] limbs (include/ntt128.h "Data layout").
"""
from __future__ import annotations

import ctypes
import os

import torch

from . import _lib_override

_PKG = os.path.dirname(os.path.abspath(__file__))
# The product path always loads the in-tree library.  Experiment scripts (tools/) may point
# `paper_2509_12494_b200._lib_override.PATH` at an experiment build BEFORE importing this
# module; nothing here reads the environment.
LIB_PATH = _lib_override.PATH or os.path.join(_PKG, "libntt128.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2509_12494_b200.build` (no fallback path exists)")

_L = ctypes.CDLL(LIB_PATH)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_vp = ctypes.c_void_p

_L.ntt128_plan_create.argtypes = [ctypes.POINTER(_vp), ctypes.c_uint32, ctypes.c_uint32, _u64p, _u64p,
                                  ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int]
_L.ntt128_plan_create.restype = ctypes.c_int
for _name in ("ntt128_forward", "ntt128_inverse", "ntt128_forward_bitrev", "ntt128_inverse_bitrev"):
    getattr(_L, _name).argtypes = [_vp, _vp, _vp, _vp]
    getattr(_L, _name).restype = ctypes.c_int
_L.ntt128_polymul.argtypes = [_vp, _vp, _vp, _vp, _vp]
_L.ntt128_polymul.restype = ctypes.c_int
_L.ntt128_plan_info.argtypes = [_vp] + [ctypes.POINTER(ctypes.c_uint32)] * 5
_L.ntt128_plan_info.restype = ctypes.c_int
_L.ntt128_plan_arith_class.argtypes = [_vp, ctypes.POINTER(ctypes.c_uint32)]
_L.ntt128_plan_arith_class.restype = ctypes.c_int
_L.ntt128_plan_destroy.argtypes = [_vp]
_L.ntt128_plan_destroy.restype = None
for _name in ("vec128_add", "vec128_sub", "vec128_mul"):
    getattr(_L, _name).argtypes = [_vp, _vp, _vp, ctypes.c_size_t, _u64p, ctypes.c_uint32, _vp]
    getattr(_L, _name).restype = ctypes.c_int
_L.vec128_axpy.argtypes = [_vp, _u64p, _vp, ctypes.c_size_t, _u64p, ctypes.c_uint32, _vp]
_L.vec128_axpy.restype = ctypes.c_int
_L.ntt256_plan_create.argtypes = [ctypes.POINTER(_vp), ctypes.c_uint32, ctypes.c_uint32, _u64p, _u64p,
                                  ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int]
_L.ntt256_plan_create.restype = ctypes.c_int
for _name in ("ntt256_forward", "ntt256_inverse"):
    getattr(_L, _name).argtypes = [_vp, _vp, _vp, _vp]
    getattr(_L, _name).restype = ctypes.c_int
_L.ntt256_plan_destroy.argtypes = [_vp]
_L.ntt256_plan_destroy.restype = None
_L.vec256_mul.argtypes = [_vp, _vp, _vp, ctypes.c_size_t, _u64p, _vp]
_L.vec256_mul.restype = ctypes.c_int
_L.ntt128_status_string.argtypes = [ctypes.c_int]
_L.ntt128_status_string.restype = ctypes.c_char_p
_L.ntt128_launch_count.argtypes = []
_L.ntt128_launch_count.restype = ctypes.c_uint64

CYCLIC, NEGACYCLIC, FLAG_CHECK_INPUT, FLAG_CHAIN = 0, 1, 0x100, 0x200   # include/ntt128.h
OK = 0
_ARG_ERRORS = {1, 2, 3, 4, 5, 6, 7}

EXPORTED = ("ntt128_plan_create", "ntt128_forward", "ntt128_inverse", "ntt128_forward_bitrev",
            "ntt128_inverse_bitrev", "ntt128_polymul", "ntt128_plan_info", "ntt128_plan_arith_class",
            "ntt128_plan_destroy", "vec128_add", "vec128_sub", "vec128_mul", "vec128_axpy",
            "ntt128_status_string", "ntt128_launch_count", "ntt128_fourstep_create", "ntt128_fourstep_forward_a",
            "ntt128_fourstep_forward_c", "ntt128_fourstep_inverse_a", "ntt128_fourstep_inverse_c",
            "ntt128_fourstep_forward_a_peers", "ntt128_fourstep_inverse_a_peers", "ntt128_fourstep_forward_pack",
            "ntt128_fourstep_forward_a_nat", "ntt128_fourstep_forward_c_nat", "ntt128_fourstep_forward_unpack",
            "ntt128_fourstep_inverse_pack", "ntt128_fourstep_inverse_a_nat", "ntt128_fourstep_inverse_c_nat",
            "ntt128_fourstep_inverse_unpack", "ntt128_fourstep_destroy",
            "ntt256_plan_create", "ntt256_forward", "ntt256_inverse", "ntt256_plan_destroy", "vec256_mul")


class NTT128Error(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {status_string(status)}")


class NTT128ArgError(NTT128Error, ValueError):
    pass


def status_string(s: int) -> str:
    return _L.ntt128_status_string(int(s)).decode()


def launch_count() -> int:
    return int(_L.ntt128_launch_count())


def _check(status: int, what: str) -> None:
    if status != OK:
        raise (NTT128ArgError if status in _ARG_ERRORS else NTT128Error)(status, what)


def _pairs(vals) -> ctypes.Array:
    vals = [int(v) for v in vals]
    arr = (ctypes.c_uint64 * (2 * len(vals)))()
    for i, v in enumerate(vals):
        if not 0 <= v < (1 << 128):
            raise ValueError("value out of the 128-bit range")
        arr[2 * i] = v & 0xFFFFFFFFFFFFFFFF
        arr[2 * i + 1] = v >> 64
    return arr


def _ptr(t: torch.Tensor, name: str, limbs: int = 2, device: int | None = None) -> int:
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if device is not None and t.device.index != device:
        raise ValueError(f"{name} is on cuda:{t.device.index}, the plan on cuda:{device}")
    if t.dtype not in (torch.uint64, torch.int64):
        raise TypeError(f"{name} must have dtype uint64 or int64")
    if not t.is_contiguous() or t.shape[-1] != limbs:
        raise ValueError(f"{name} must be contiguous with a trailing limb dimension of {limbs}")
    return t.data_ptr()


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


class Plan:
    """Batched 128-bit NTT plan (ntt128_plan_create).

    log2n: 1..26; q, root: int (shared) or a sequence of `batch` ints (one prime per
    polynomial, the RNS case); negacyclic: root is psi of order 2N; chain: NTT128_FLAG_CHAIN
    (consecutive calls on a stream overlap polynomial by polynomial; include/ntt128.h).
    """

    def __init__(self, log2n: int, q, root, batch: int = 1, negacyclic: bool = False, check_input: bool = False,
                 device: int | None = None, chain: bool = False):
        qs = list(q) if isinstance(q, (list, tuple)) else [q]
        rs = list(root) if isinstance(root, (list, tuple)) else [root]
        if len(qs) != len(rs):
            raise ValueError("q and root must have the same length")
        self.log2n, self.batch, self.n = int(log2n), int(batch), 1 << int(log2n)
        self.negacyclic = bool(negacyclic)
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.q = [int(v) for v in qs]
        flags = ((NEGACYCLIC if negacyclic else CYCLIC) | (FLAG_CHECK_INPUT if check_input else 0)
                 | (FLAG_CHAIN if chain else 0))
        h = _vp()
        self._h = None
        _check(_L.ntt128_plan_create(ctypes.byref(h), self.log2n, self.batch, _pairs(qs), _pairs(rs), len(qs), flags,
                                     self.device), "ntt128_plan_create")
        self._h = h

    def info(self) -> dict:
        v = [ctypes.c_uint32() for _ in range(5)]
        _check(_L.ntt128_plan_info(self._h, *[ctypes.byref(x) for x in v]), "ntt128_plan_info")
        return dict(zip(("log2n", "batch", "n_moduli", "flags", "num_passes"), [x.value for x in v]))

    def arith_class(self) -> str:
        """'pseudo_mersenne' or 'montgomery' (ntt128_plan_arith_class)"""
        c = ctypes.c_uint32()
        _check(_L.ntt128_plan_arith_class(self._h, ctypes.byref(c)), "ntt128_plan_arith_class")
        return "pseudo_mersenne" if c.value == 1 else "montgomery"

    def _shape_ok(self, t: torch.Tensor, name: str) -> None:
        if t.numel() != 2 * self.n * self.batch:
            raise ValueError(f"{name} must hold batch * N = {self.batch} * {self.n} residues")

    def forward(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        self._shape_ok(x, "x")
        out = torch.empty_like(x) if out is None else out
        self._shape_ok(out, "out")
        _check(_L.ntt128_forward(self._h, _ptr(x, "x", device=self.device), _ptr(out, "out", device=self.device), _stream(x)), "ntt128_forward")
        return out

    def inverse(self, y: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        self._shape_ok(y, "y")
        out = torch.empty_like(y) if out is None else out
        self._shape_ok(out, "out")
        _check(_L.ntt128_inverse(self._h, _ptr(y, "y", device=self.device), _ptr(out, "out", device=self.device), _stream(y)), "ntt128_inverse")
        return out

    def forward_bitrev(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """negacyclic spectrum in bit-reversed order (ntt128_forward_bitrev)"""
        self._shape_ok(x, "x")
        out = torch.empty_like(x) if out is None else out
        self._shape_ok(out, "out")
        _check(_L.ntt128_forward_bitrev(self._h, _ptr(x, "x", device=self.device), _ptr(out, "out", device=self.device), _stream(x)), "ntt128_forward_bitrev")
        return out

    def inverse_bitrev(self, y: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        self._shape_ok(y, "y")
        out = torch.empty_like(y) if out is None else out
        self._shape_ok(out, "out")
        _check(_L.ntt128_inverse_bitrev(self._h, _ptr(y, "y", device=self.device), _ptr(out, "out", device=self.device), _stream(y)), "ntt128_inverse_bitrev")
        return out

    def polymul(self, a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        self._shape_ok(a, "a")
        self._shape_ok(b, "b")
        out = torch.empty_like(a) if out is None else out
        self._shape_ok(out, "out")
        _check(_L.ntt128_polymul(self._h, _ptr(a, "a", device=self.device), _ptr(b, "b", device=self.device), _ptr(out, "out", device=self.device), _stream(a)), "ntt128_polymul")
        return out

    def close(self) -> None:
        if self._h is not None:
            _L.ntt128_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _blas(fn, x, y, q, out, check_input):
    out = torch.empty_like(x) if out is None else out
    n = x.numel() // 2
    if y.numel() != x.numel() or out.numel() != x.numel():
        raise ValueError("length mismatch")
    _check(fn(_ptr(out, "out"), _ptr(x, "x"), _ptr(y, "y"), n, _pairs([q]), FLAG_CHECK_INPUT if check_input else 0,
              _stream(x)), fn.__name__)
    return out


def vadd(x, y, q: int, out=None, check_input=False):
    """z = x + y mod q (vec128_add)"""
    return _blas(_L.vec128_add, x, y, q, out, check_input)


def vsub(x, y, q: int, out=None, check_input=False):
    """z = x - y mod q (vec128_sub)"""
    return _blas(_L.vec128_sub, x, y, q, out, check_input)


def vmul(x, y, q: int, out=None, check_input=False):
    """z = x * y mod q (vec128_mul)"""
    return _blas(_L.vec128_mul, x, y, q, out, check_input)


def axpy(a: int, x, y, q: int, check_input=False):
    """y <- a * x + y mod q, in place on y (vec128_axpy); returns y"""
    if y.numel() != x.numel():
        raise ValueError("length mismatch")
    _check(_L.vec128_axpy(_ptr(y, "y"), _pairs([a]), _ptr(x, "x"), x.numel() // 2, _pairs([q]),
                          FLAG_CHECK_INPUT if check_input else 0, _stream(x)), "vec128_axpy")
    return y


# ----------------------------------------------------------------------------- 256-bit moduli
def _limbs4(vals) -> ctypes.Array:
    vals = list(vals)
    arr = (ctypes.c_uint64 * (4 * len(vals)))()
    for i, v in enumerate(vals):
        v = int(v)
        if v < 0 or v >> 256:
            raise ValueError("256-bit value out of range")
        for k in range(4):
            arr[4 * i + k] = (v >> (64 * k)) & 0xFFFFFFFFFFFFFFFF
    return arr


class Plan256:
    """ntt256_plan_create / ntt256_forward / ntt256_inverse (include/ntt128.h, "Wider moduli").
    Tensors are contiguous CUDA int64/uint64 [..., N, 4] (four little-endian limbs)."""

    def __init__(self, log2n: int, q, root, batch: int = 1, device: int | None = None):
        qs = list(q) if isinstance(q, (list, tuple)) else [q]
        rs = list(root) if isinstance(root, (list, tuple)) else [root]
        if len(qs) != len(rs):
            raise ValueError("q and root lists differ in length")
        self.log2n, self.batch, self.N = int(log2n), int(batch), 1 << int(log2n)
        dev = torch.cuda.current_device() if device is None else int(device)
        h = _vp()
        self._h = None
        _check(_L.ntt256_plan_create(ctypes.byref(h), self.log2n, self.batch, _limbs4(qs), _limbs4(rs), len(qs), 0, dev),
               "ntt256_plan_create")
        self._h = h

    def _shape_ok(self, t, name):
        if t.shape[-2:] != (self.N, 4) or t.numel() != self.batch * self.N * 4:
            raise ValueError(f"{name}: expected [{self.batch}, {self.N}, 4], got {tuple(t.shape)}")

    def forward(self, x, out=None):
        self._shape_ok(x, "x")
        out = torch.empty_like(x) if out is None else out
        self._shape_ok(out, "out")
        _check(_L.ntt256_forward(self._h, _ptr(x, "x", 4), _ptr(out, "out", 4), _stream(x)), "ntt256_forward")
        return out

    def inverse(self, y, out=None):
        self._shape_ok(y, "y")
        out = torch.empty_like(y) if out is None else out
        self._shape_ok(out, "out")
        _check(_L.ntt256_inverse(self._h, _ptr(y, "y", 4), _ptr(out, "out", 4), _stream(y)), "ntt256_inverse")
        return out

    def close(self):
        if self._h is not None:
            _L.ntt256_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def vmul256(x, y, q: int, out=None):
    """z = x * y mod q over 256-bit residues ([..., 4] limbs)"""
    out = torch.empty_like(x) if out is None else out
    if y.numel() != x.numel() or out.numel() != x.numel():
        raise ValueError("length mismatch")
    _check(_L.vec256_mul(_ptr(out, "out", 4), _ptr(x, "x", 4), _ptr(y, "y", 4), x.numel() // 4, _limbs4([q]), _stream(x)),
           "vec256_mul")
    return out

"""Seeded synthetic-input generators shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no modular add/sub/mul, no
transform). It only draws pseudo-random 64-bit words and turns them into
uniform residues in [0, q) by rejection, so both sides of every parity test
consume byte-identical inputs (SURVEY.md App. A "Randomness").

* splitmix64 is counter based: draw i of a stream with seed s is
  mix(s + (i + 1) * 0x9E3779B97F4A7C15), so a whole stream vectorises in numpy.
* uniform residue: two draws (hi first), v = (hi << 64 | lo) >> (128 - bitlen(q)),
  accept if v < q, else draw the next pair.
* stream seed = (config_id << 48) ^ (purpose << 40) ^ index, purpose
  0 = x/a data, 1 = y/b data, 2 = root search, 3 = scalar.

Layout of a residue array: numpy uint64 of shape [..., 2] = [lo, hi], the
memory image of unsigned __int128.
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)

PURPOSE_X, PURPOSE_Y, PURPOSE_ROOT, PURPOSE_SCALAR = 0, 1, 2, 3


def stream_seed(config_id: int, purpose: int, index: int) -> int:
    return ((config_id << 48) ^ (purpose << 40) ^ index) & 0xFFFFFFFFFFFFFFFF


def splitmix64(seed: int, start: int, count: int) -> np.ndarray:
    """Draws start .. start+count-1 of the splitmix64 stream `seed` (uint64 array)."""
    with np.errstate(over="ignore"):
        i = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        z = np.uint64(seed) + i * GAMMA
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        return z ^ (z >> np.uint64(31))


def splitmix64_scalar(seed: int, i: int) -> int:
    """Draw i (0-based) of stream `seed`, in plain Python ints (for tiny cases)."""
    m = (1 << 64) - 1
    z = (seed + (i + 1) * 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def _top_bits(hi: np.ndarray, lo: np.ndarray, bits: int):
    """(hi << 64 | lo) >> (128 - bits) as (vhi, vlo) uint64 arrays, 1 <= bits <= 128."""
    sh = 128 - bits
    if sh == 0:
        return hi.copy(), lo.copy()
    if sh < 64:
        vlo = (lo >> np.uint64(sh)) | (hi << np.uint64(64 - sh))
        vhi = hi >> np.uint64(sh)
        return vhi, vlo
    if sh == 64:
        return np.zeros_like(hi), hi.copy()
    return np.zeros_like(hi), hi >> np.uint64(sh - 64)


def uniform_residues(q: int, n: int, seed: int) -> np.ndarray:
    """n residues uniform in [0, q) from stream `seed`; returns uint64 [n, 2] ([lo, hi])."""
    assert q >= 2
    bits = q.bit_length()
    qhi, qlo = np.uint64(q >> 64), np.uint64(q & 0xFFFFFFFFFFFFFFFF)
    out = np.empty((n, 2), dtype=np.uint64)
    filled, pair_pos = 0, 0
    while filled < n:
        want = n - filled
        # acceptance >= 1/2 always; over-draw so one round nearly always suffices
        m = int(want * (2.0 ** bits / q) * 1.02) + 64
        d = splitmix64(seed, 2 * pair_pos, 2 * m).reshape(m, 2)
        vhi, vlo = _top_bits(d[:, 0], d[:, 1], bits)
        ok = (vhi < qhi) | ((vhi == qhi) & (vlo < qlo))
        idx = np.nonzero(ok)[0]
        take = idx[:want]
        out[filled:filled + len(take), 0] = vlo[take]
        out[filled:filled + len(take), 1] = vhi[take]
        filled += len(take)
        # a short round consumed all m pairs; the next round continues after them
        pair_pos += m
    return out


def uniform_residue_scalar(q: int, seed: int, k: int = 0) -> int:
    """The k-th accepted residue of stream `seed` (plain Python; used for scalars)."""
    bits = q.bit_length()
    found, i = 0, 0
    while True:
        hi, lo = splitmix64_scalar(seed, 2 * i), splitmix64_scalar(seed, 2 * i + 1)
        v = ((hi << 64) | lo) >> (128 - bits)
        i += 1
        if v < q:
            if found == k:
                return v
            found += 1


def to_ints(a: np.ndarray) -> list[int]:
    """uint64 [..., 2] -> flat list of Python ints."""
    f = a.reshape(-1, 2)
    return [int(lo) | (int(hi) << 64) for lo, hi in f.tolist()]


def from_ints(vals, shape=None) -> np.ndarray:
    vals = list(vals)
    out = np.empty((len(vals), 2), dtype=np.uint64)
    for i, v in enumerate(vals):
        out[i, 0] = v & 0xFFFFFFFFFFFFFFFF
        out[i, 1] = v >> 64
    if shape is not None:
        out = out.reshape(tuple(shape) + (2,))
    return out


def int_to_pair(v: int) -> np.ndarray:
    return np.array([v & 0xFFFFFFFFFFFFFFFF, v >> 64], dtype=np.uint64)


# ----------------------------------------------------------------------------- 256-bit residues
def _limbs(v: int) -> list[int]:
    return [(v >> (64 * i)) & 0xFFFFFFFFFFFFFFFF for i in range(4)]


def uniform_residues_w(q: int, n: int, seed: int) -> np.ndarray:
    """n residues uniform in [0, q) for q < 2^256 (the wider-modulus path):
    four draws per candidate, most significant first, top bitlen(q) bits, rejection.
    Returns uint64 [n, 4] (little-endian limbs)."""
    assert 2 <= q < (1 << 256)
    bits = q.bit_length()
    sh = 256 - bits
    qa = _limbs(q)
    out = np.empty((n, 4), dtype=np.uint64)
    filled, pos = 0, 0
    while filled < n:
        want = n - filled
        m = int(want * (2.0 ** bits / q) * 1.02) + 64
        d = splitmix64(seed, 4 * pos, 4 * m).reshape(m, 4)
        v = [d[:, 3], d[:, 2], d[:, 1], d[:, 0]]          # little-endian limbs of the 256-bit draw
        # v >> sh
        w, b = sh // 64, sh % 64
        r = []
        for i in range(4):
            lo = v[i + w] if i + w < 4 else np.zeros_like(v[0])
            hi = v[i + w + 1] if i + w + 1 < 4 else np.zeros_like(v[0])
            r.append((lo >> np.uint64(b)) | (hi << np.uint64(64 - b)) if b else lo.copy())
        lt = np.zeros(m, dtype=bool)
        eq = np.ones(m, dtype=bool)
        for i in (3, 2, 1, 0):
            qi = np.uint64(qa[i])
            lt |= eq & (r[i] < qi)
            eq &= r[i] == qi
        idx = np.nonzero(lt)[0][:want]
        for i in range(4):
            out[filled:filled + len(idx), i] = r[i][idx]
        filled += len(idx)
        pos += m
    return out


def uniform_residue_scalar_w(q: int, seed: int, k: int = 0) -> int:
    """The k-th accepted 256-bit-path residue of stream `seed` (plain Python)."""
    bits = q.bit_length()
    found, i = 0, 0
    while True:
        v = 0
        for j in range(4):
            v = (v << 64) | splitmix64_scalar(seed, 4 * i + j)
        v >>= 256 - bits
        i += 1
        if v < q:
            if found == k:
                return v
            found += 1

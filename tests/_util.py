"""Shared test helpers: numpy [.., 2] uint64 <-> CUDA tensors; edge-case corpora."""
import numpy as np


def to_dev(a: np.ndarray, device="cuda"):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64)).to(device)


def to_host(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)


def edge_values(q: int):
    """SURVEY.md §8(c) e1 edge values restricted to [0, q)"""
    qh, ql = q >> 64, q & ((1 << 64) - 1)
    cand = [0, 1, 2, q - 1, q - 2, (q - 1) // 2, (q + 1) // 2, 2**32 - 1, 2**32, 2**32 + 1, 2**64 - 1, 2**64,
            2**64 + 1, 2**96, 2**127 - 1, 2**127, 2**127 + 1]
    for lo in (0, max(ql - 1, 0), ql, 2**64 - 1):
        cand.append((qh << 64) | lo)
    return sorted({c for c in cand if 0 <= c < q})


def edge_pairs(q: int, rng):
    """(a, b) pairs from the edge corpus e1-e5"""
    ev = edge_values(q)
    out = [(a, b) for a in ev for b in ev]
    for t in (q - 1, q, q + 1, 2**128 - 1, 2**128, 2**128 + 1):      # e2 sums
        for _ in range(8):
            b = rng.randrange(q)
            if 0 <= t - b < q:
                out.append((t - b, b))
    out.append((q - 1, q - 1))                                          # e3
    for _ in range(8):                                                  # e4 differences
        a = rng.randrange(1, q - 1)
        out += [(a, a + 1), (a, a), (a + 1, a)]
    if q > 3:
        for _ in range(8):                                              # e5 products -> 0, 1, q-1
            a = rng.randrange(1, q)
            try:
                ai = pow(a, -1, q)
            except ValueError:
                continue
            out += [(a, ai), (a, q - ai), (a, 0)]
    return out

"""Batch sharding across ranks: independent polynomials (each
with its own RNS prime and plan) split over G GPUs with no data-path collective -- "real
FHE workloads often batch NTTs and BLAS operations without data dependencies"
(PAPER.md:793).  Host logic only: which units a rank owns, and (for verification, never
on the timed path) the gather of every rank's results in unit order."""
from __future__ import annotations


def shard(total: int, world: int, rank: int) -> tuple[int, int]:
    """[start, stop) of rank's share of `total` units: contiguous, in rank order, sizes
    differing by at most one (the first total mod world ranks take one more)"""
    if world < 1 or not 0 <= rank < world or total < 0:
        raise ValueError(f"bad shard request: total={total} world={world} rank={rank}")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def gather_batch(local, world: int, group=None):
    """concatenate every rank's result tensor [units, ...] in rank order (all_gather_object
    so unequal shards work on any backend); world 1 is the identity"""
    if world == 1:
        return local
    import torch
    import torch.distributed as dist
    parts = [None] * world
    dist.all_gather_object(parts, local.cpu(), group=group)
    return torch.cat(parts, 0)

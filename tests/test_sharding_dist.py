"""Batch sharding: the shard ranges, a gloo world-size-2 run in which
each rank transforms only its own polynomials (an oracle-backed stand-in for the rank's
kernels -- test infrastructure) and the gathered result equals the whole batch's oracle
transform, and bench.py's self-launch of --gpus ranks (host-only, gloo)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
import synth
from paper_2509_12494_b200.sharding import gather_batch, shard

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("total,world", [(1024, 1), (1024, 2), (1024, 8), (64, 8), (7, 3), (3, 8), (0, 4), (1 << 20, 8)])
def test_shard_ranges_partition(total, world):
    rs = [shard(total, world, r) for r in range(world)]
    assert rs[0][0] == 0 and rs[-1][1] == total
    for (a0, a1), (b0, b1) in zip(rs, rs[1:]):
        assert a1 == b0                               # contiguous, in rank order
    sizes = [b - a for a, b in rs]
    assert max(sizes) - min(sizes) <= 1 and sum(sizes) == total
    with pytest.raises(ValueError):
        shard(total, world, world)


def _worker(rank, world, port, qs, ws, x, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b0, b1 = shard(x.shape[0], world, rank)
    y = O.ntt(np.ascontiguousarray(x[b0:b1]), qs[b0:b1], ws[b0:b1])     # this rank's polynomials only
    full = gather_batch(torch.from_numpy(y.view(np.int64)), world)
    if rank == 0:
        out["y"] = full.numpy().view(np.uint64).copy()
        out["shards"] = [shard(x.shape[0], world, r) for r in range(world)]
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("B", [16, 13])
def test_batch_split_gloo_world2(params, B):
    """RNS batch (own prime per polynomial) split over 2 ranks; gather == whole-batch oracle"""
    mods = params["cfg3"]["moduli"][:B]
    logn = 8
    qs = [m["q"] for m in mods]
    ws = [pow(m["omega"], 1 << (16 - logn), m["q"]) for m in mods]
    x = np.stack([synth.uniform_residues(qs[i], 1 << logn, 900 + i) for i in range(B)])
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), qs, ws, x, out), nprocs=2)
    assert out["shards"] == [(0, (B + 1) // 2), ((B + 1) // 2, B)]
    assert np.array_equal(out["y"], O.ntt(x, qs, ws))


def test_bench_self_launch_two_ranks():
    """`bench.py --gpus 2` with no WORLD_SIZE re-launches itself under torch.distributed.run;
    the launch self-test gathers every rank's shards of the cfg4 N = 2^16 batch (B = 1024)"""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launch-selftest"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    ranks = json.loads(lines[0])["launch_selftest"]
    assert [d["rank"] for d in ranks] == [0, 1] and all(d["world"] == 2 for d in ranks)
    assert [tuple(d["cfg4_logn16"]) for d in ranks] == [(0, 512), (512, 1024)]
    assert [tuple(d["cfg2"]) for d in ranks] == [(0, 1 << 19), (1 << 19, 1 << 20)]

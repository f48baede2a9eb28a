#!/usr/bin/env python
"""Benchmark of the 128-bit NTT hot path (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--rows|--no-rows]

Workload (BASELINE.json configs[2], "cfg3"): batched forward + inverse cyclic NTT,
N = 2^16, 64 polynomials, each with its own 124..128-bit prime q_i = 1 mod 2N (RNS
limbs), coefficients uniform in [0, q_i) (seeded).  One step = forward + inverse of
the whole batch through the C ABI (ntt128_forward / ntt128_inverse).  Metric: 128-bit
NTT butterflies per second (N/2 log2 N per transform, forward and inverse counted).

Multi-GPU: `--gpus G` re-launches itself under torch.distributed.run with G ranks (one
process per GPU, NCCL) unless WORLD_SIZE is already set (the driver's torchrun form).
Headline: every rank transforms its own 64-polynomial batch (independent RNS limbs; no
data-path collective), value = butterflies of all ranks / max-over-ranks time
("scaling": "weak").  Rows: the cfg4 sweep is STRONG scaling (1 GiB of coefficients in
total, rank g owns polynomials [g B/G, (g+1) B/G); the N = 2^16 row, B = 1024, is the
SURVEY.md §8(d) >= 7x row), cfg2 BLAS splits the vector, cfg1 / cfg3 polymul / cfg5
three-pass / 256-bit rows run one replica per rank, the cfg5 four-step spans all ranks;
every row is timed per rank and reported as max over ranks.  Timing: CUDA events on the
launching stream, barrier + synchronize on both sides, max over ranks.  L2: inputs rotate
over 4 disjoint buffer sets (each step's input was last touched >= 3 steps, >= 576 MiB of
traffic, earlier).

--impl reference runs the oracle (oracle/, the plain CPU implementation written from
the paper) on this host's cores as the reference arm, on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
PARAMS_PATH = os.path.join(ROOT, "tests", "golden", "params.json")
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "ncu_traffic.json")
INT_PEAK_PATH = os.path.join(ROOT, "profiles", "int_peak.json")

# Roofline constants.  P = algorithmic 32x32->64 products per unit
# (SURVEY.md §8(d)): 36 per butterfly / constant mulmod, 42 per general mulmod.
P_BUTTERFLY = 36
P_GENERAL = 42
# word products the kernels actually issue per butterfly, by the plan's arithmetic class
# (DESIGN.md §5): Montgomery CIOS 32 IMAD.WIDE + 4 IMAD; pseudo-Mersenne 16 + 4 + 1 IMAD.WIDE
P_EMITTED = {"montgomery": 36, "pseudo_mersenne": 21}
SMS = 148
IMAD_WIDE_PER_CLK_SM = 32          # fallback only: IMAD.WIDE.U32 at half the IMAD rate
FALLBACK_HBM_GBS = 6650.0


def load_params():
    with open(PARAMS_PATH) as f:
        P = json.load(f)
    return P


def hexint(s):
    return int(s, 16)


def peaks():
    d = {}
    if os.path.exists(PEAKS_PATH):
        with open(PEAKS_PATH) as f:
            d = json.load(f)
    hbm = d.get("hbm_gbs")
    sm_max = d.get("sm_max_mhz", 1965.0)
    # integer-multiply peak R: the measured 32x32->64 products per clock per SM (sustained
    # >= 1.5 s with NVML clocks, tools/micro/int_peak.py -> profiles/int_peak.json) x 148 SMs
    # x the max SM clock; the nominal 32/clk/SM only if that file is missing
    per_clk, src = IMAD_WIDE_PER_CLK_SM, "fallback: 148 SM x 32 IMAD.WIDE.U32/clk x sm_max_mhz (DESIGN.md §6)"
    if os.path.exists(INT_PEAK_PATH):
        try:
            with open(INT_PEAK_PATH) as f:
                per_clk = float(json.load(f)["products_per_clk_per_sm"])
            src = (f"profiles/int_peak.json: measured {per_clk:.3f} products/clk/SM (sustained, NVML clocks) "
                   f"x 148 SM x sm_max_mhz {sm_max:.0f}")
        except Exception:
            per_clk = IMAD_WIDE_PER_CLK_SM
    return {
        "hbm_gbs": hbm if hbm else FALLBACK_HBM_GBS,
        "hbm_src": "measured" if hbm else "fallback",
        "sm_max_mhz": sm_max,
        "tprod_s": SMS * per_clk * sm_max * 1e6 / 1e12,
        "tprod_src": src,
    }


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML samples of SM clock and clock-event reasons during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self._nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._nv:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- distributed
def spawn_ranks(ngpus: int) -> int:
    """re-run this script under torch.distributed.run with `ngpus` ranks (127.0.0.1
    rendezvous); returns the launcher's exit code"""
    import socket
    import subprocess
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ngpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def dist_setup(ngpus: int):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:                                   # host-only self-test of the launch path (gloo)
            dist.init_process_group("gloo")
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world, local


from paper_2509_12494_b200.sharding import shard  # noqa: E402  (host logic, no CUDA)


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------- workloads
def cfg3_inputs(P, rank, nsets):
    mods = P["cfg3"]["moduli"]
    qs = [hexint(m["q"]) for m in mods]
    ws = [hexint(m["omega"]) for m in mods]
    psis = [hexint(m["psi"]) for m in mods]
    import synth
    n = 1 << P["cfg3"]["logn"]
    sets = []
    for s in range(nsets):
        x = np.stack([synth.uniform_residues(qs[i], n, synth.stream_seed(3, 0, (rank << 20) | (s << 8) | i))
                      for i in range(len(qs))])
        sets.append(x)
    return qs, ws, psis, sets


def to_dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


def time_events(fn, iters, stream):
    """average ms per call over iters calls, CUDA events on `stream`"""
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for i in range(iters):
        fn(i)
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / iters


def time_graph(fn, ncalls, replays=20):
    """average ms per call of `fn(i)`, i < ncalls, captured once into a CUDA graph and
    replayed (removes host launch overhead from short kernels)"""
    import torch
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(ncalls):
            fn(i)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(ncalls):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(replays):
        g.replay()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / (replays * ncalls)


def run_gpu(args):
    import torch
    from paper_2509_12494_b200 import ntt128 as N

    rank, world, local = dist_setup(args.gpus)
    P = load_params()
    pk = peaks()
    logn, B = P["cfg3"]["logn"], P["cfg3"]["batch"]
    n = 1 << logn
    NSETS = 4
    qs, ws, psis, sets = cfg3_inputs(P, rank, NSETS)
    # NTT128_FLAG_CHAIN: consecutive transforms on the stream overlap polynomial by polynomial
    # (include/ntt128.h; DESIGN.md §6 "Chained calls") -- same work, same results
    plan = N.Plan(logn, qs, ws, batch=B, chain=True)
    X = [to_dev(x) for x in sets]
    Y = [torch.empty_like(x) for x in X]
    Z = [torch.empty_like(x) for x in X]
    stream = torch.cuda.current_stream()
    bfly_per_transform = (n // 2) * logn
    bfly_per_step = 2 * B * bfly_per_transform

    def step(i):
        k = i % NSETS
        plan.forward(X[k], out=Y[k])
        plan.inverse(Y[k], out=Z[k])

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    # correctness guard on rank data (round trip) before timing
    assert torch.equal(Z[(args.warmup - 1) % NSETS], X[(args.warmup - 1) % NSETS]) if args.warmup else True

    # ---------------- timed region: K steps bracketed by two events only (an event between
    # two calls would serialise the programmatic launch overlap of consecutive transforms)
    launches0 = N.launch_count()
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for i in range(args.steps):
            k = (args.warmup + i) % NSETS
            plan.forward(X[k], out=Y[k])
            plan.inverse(Y[k], out=Z[k])
        t_end.record(stream)
        t_end.synchronize()
    torch.cuda.synchronize()
    barrier(world)
    launches = N.launch_count() - launches0
    ms_local = t_start.elapsed_time(t_end)
    ms = max_over_ranks(ms_local, world)
    ms_per_step = ms / args.steps
    value = bfly_per_step * world * args.steps / (ms / 1e3)
    # diagnostic split (after the timed region): forward and inverse timed separately
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(5)]
    for i in range(5):
        k = i % NSETS
        ev[i][0].record(stream)
        plan.forward(X[k], out=Y[k])
        ev[i][1].record(stream)
        plan.inverse(Y[k], out=Z[k])
        ev[i][2].record(stream)
    torch.cuda.synchronize()
    fwd_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in ev)
    inv_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in ev)

    # dominant kernels: the NTT pass kernels (k_ntt_first_tl, k_ntt_pass); one launch = one pass over the batch.
    # Its average launch duration over the timed region = local step time / launches per step
    # (the step is nothing but these launches, overlapped back to back).
    npasses = plan.info()["num_passes"]
    launch_ms = (ms_local / args.steps) / (2 * npasses)
    prod_per_launch = P_BUTTERFLY * B * (n // 2) * (logn / npasses)
    achieved = prod_per_launch / (launch_ms * 1e-3) / 1e12
    traffic, traffic_src = None, None
    if os.path.exists(TRAFFIC_PATH):   # dram read+write bytes per launch from a committed ncu --set full capture
        try:
            with open(TRAFFIC_PATH) as f:
                tj = json.load(f)
            traffic = tj.get("bytes_per_launch_mean")
            traffic_src = "capture, not measured in this run: " + tj.get("source", TRAFFIC_PATH)
        except Exception:
            traffic = None
    roofline = {"bound": "alu", "kernel": "NTT pass kernels (k_ntt_first_tl first passes, k_ntt_pass later passes)",
                "achieved": round(achieved, 4), "peak": round(pk["tprod_s"], 4),
                "unit": "Tprod/s", "frac": round(achieved / pk["tprod_s"], 4), "traffic": traffic,
                "traffic_src": traffic_src, "peak_src": pk["tprod_src"],
                "step_frac": round(value / world * P_BUTTERFLY / 1e12 / pk["tprod_s"], 4)}
    # `achieved` counts SURVEY §8(d)'s ALGORITHMIC products (P = 36 per butterfly, fixed from the
    # schoolbook + Shoup/Montgomery decomposition whatever the SASS does).  A plan in the
    # pseudo-Mersenne class (every cfg3 prime is 2^b - c with a small c) emits 21 per butterfly,
    # so the pipe itself is busier than `frac` x 21/36 says and `frac` may pass 1: both are stated.
    arith = plan.arith_class()
    roofline["arith_class"] = arith
    roofline["products_emitted_per_butterfly"] = P_EMITTED[arith]
    roofline["frac_emitted"] = round(achieved * P_EMITTED[arith] / P_BUTTERFLY / pk["tprod_s"], 4)

    # ---------------- end to end through the public API with host buffers
    e2e = run_e2e(plan, sets[0], args, stream, bfly_per_step, world)

    rows = run_rows(args, P, pk, stream, rank, world) if args.rows else None
    cpu = cpu_baseline(P) if (rank == 0 and args.cpu_baseline) else None
    if cpu is not None and args.rows:
        cpu["rows"] = oracle_rows(P)
    if rank == 0:
        out = {
            "metric": "128-bit NTT butterflies/sec (N=2^16, fwd+inv, 64 RNS primes)",
            "value": value, "unit": "butterflies/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u128", "data": "synthetic (seeded uniform residues)",
            "config": {"workload": "cfg3: batched forward+inverse cyclic NTT, N=2^16, batch 64 per GPU, 64 distinct "
                                   "124-128-bit primes (BASELINE.json configs[2])",
                       "N": n, "batch_per_gpu": B, "parallelism": f"batch-shard x{world} (no collective)",
                       "l2": "inputs rotate over 4 disjoint buffer sets (768 MiB footprint > 126 MB L2)",
                       "passes": npasses,
                       "chain": "NTT128_FLAG_CHAIN: each transform's first pass starts on a polynomial once the "
                                "previous call finished it (per-polynomial counters) instead of after the whole grid"},
            "ntt_per_s": value / bfly_per_transform,
            "ns_per_butterfly": 1e9 / value,
            "fwd_ms": fwd_ms, "inv_ms": inv_ms,
            "roofline": roofline,
            "clocks": clk.summary(),
            "e2e": e2e,
            "gpu_launches": launches,
            "cpu_baseline": cpu,
        }
        if rows is not None:
            out["rows"] = rows
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_e2e(plan, x_host, args, stream, bfly_per_step, world):
    """The same metric end to end through the public API: every step uploads its input
    from pinned host memory, runs forward + inverse, and downloads the result.  Steps are
    pipelined over three streams (upload of step i+1 and download of step i-1 overlap the
    transforms of step i; three device buffer sets), the way a serving loop would run."""
    import torch
    NB = 3
    hx = [torch.from_numpy(np.ascontiguousarray(x_host).view(np.int64)).pin_memory() for _ in range(NB)]
    hz = [torch.empty_like(hx[0]).pin_memory() for _ in range(NB)]
    dx = [torch.empty(hx[0].shape, dtype=hx[0].dtype, device="cuda") for _ in range(NB)]
    dy = [torch.empty_like(dx[0]) for _ in range(NB)]
    dz = [torch.empty_like(dx[0]) for _ in range(NB)]
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    comp = stream
    up = [torch.cuda.Event() for _ in range(NB)]
    done = [torch.cuda.Event() for _ in range(NB)]
    down = [torch.cuda.Event() for _ in range(NB)]

    def step(i):
        b = i % NB
        s_in.wait_event(done[b])                      # dx[b]'s previous reader (step i - NB) is done
        with torch.cuda.stream(s_in):
            dx[b].copy_(hx[b], non_blocking=True)
            up[b].record(s_in)
        comp.wait_event(up[b])
        comp.wait_event(down[b])                      # dz[b]'s previous result has left the device
        with torch.cuda.stream(comp):
            plan.forward(dx[b], out=dy[b])
            plan.inverse(dy[b], out=dz[b])
            done[b].record(comp)
        s_out.wait_event(done[b])
        with torch.cuda.stream(s_out):
            hz[b].copy_(dz[b], non_blocking=True)
            down[b].record(s_out)

    for i in range(max(2, args.warmup)):
        step(i)
    torch.cuda.synchronize()
    steps = max(2, args.steps)
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    s_in.wait_event(e0)
    for i in range(steps):
        step(i)
    for b in range(NB):
        comp.wait_event(down[b])
    e1.record(comp)
    e1.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1), world)
    assert all(torch.equal(hz[b], hx[b]) for b in range(NB)), "e2e round trip mismatch"
    nbytes = hx[0].numel() * 8
    return {"value": bfly_per_step * world * steps / (ms / 1e3), "unit": "butterflies/s",
            "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "ms_per_step": ms / steps,
            "pipelined": "upload/compute/download on 3 streams, 3 buffer sets"}


# ----------------------------------------------------------------------------- other §8 rows
def timed_rank(fn, iters, world, repeats=3):
    """per-call ms of fn(i): `repeats` runs of `iters` calls, each bracketed by a barrier and
    CUDA events on the current stream, max over ranks; returns the median over repeats"""
    import torch
    out = []
    for r in range(repeats):
        barrier(world)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(iters):
            fn(i)
        e1.record()
        e1.synchronize()
        out.append(max_over_ranks(e0.elapsed_time(e1) / iters, world))
    return statistics.median(out)


def run_rows(args, P, pk, stream, rank, world):
    """One measurement per other SURVEY §8(a) row, on every rank (module docstring): cfg1
    latency, cfg2 BLAS, cfg3 negacyclic polymul, cfg4 size sweep (strong scaling), cfg5
    N = 2^26 (three-pass replicas and the four-step over all ranks), 256-bit moduli."""
    import torch
    from paper_2509_12494_b200 import ntt128 as N
    import synth
    rows = {"rows_scaling": {"cfg1": "replica per rank (max latency)", "cfg2": "strong (n split over ranks)",
                             "cfg3_polymul": "weak (64 per rank)", "cfg4": "strong (1 GiB total, batch split)",
                             "cfg5_three_pass": "replica per rank",
                             "cfg5_fourstep": "one transform over all ranks (transposed layouts: nccl / p2p; "
                                              "natural block layout: nccl, two more all-to-alls per direction)",
                             "f4": "weak (32 per rank)"},
            "rows_timing": "median of 3 repeats, each max over ranks of CUDA-event time"}
    # cfg1: single N = 1024 forward + inverse (latency) -- one replica per rank
    e = P["cfg1"]
    q, w = hexint(e["q"]), hexint(e["omega"])
    p1 = N.Plan(10, q, w)
    x = to_dev(synth.uniform_residues(q, 1024, synth.stream_seed(1, 0, 0)).reshape(1, 1024, 2))
    y, z = torch.empty_like(x), torch.empty_like(x)
    ms = max_over_ranks(time_graph(lambda i: (p1.forward(x, out=y), p1.inverse(y, out=z)), 50), world)
    assert torch.equal(z, x), "cfg1 round trip"
    rows["cfg1_n1024_fwd_inv_us"] = ms * 1e3           # CUDA-graph replay (launch overhead excluded)
    rows["cfg1_ns_per_butterfly"] = ms * 1e6 / (2 * 5120)
    # cfg2: BLAS n = 2^20 split over the ranks (HBM-bound; 48 B/element); 8 rotating sets
    q2, a2, n2 = hexint(P["cfg2"]["q"]), hexint(P["cfg2"]["a"]), P["cfg2"]["n"]
    s0, s1 = shard(n2, world, rank)
    nl = s1 - s0
    xs = [to_dev(synth.uniform_residues(q2, n2, synth.stream_seed(2, 0, s))[s0:s1]) for s in range(8)]
    ys = [to_dev(synth.uniform_residues(q2, n2, synth.stream_seed(2, 1, s))[s0:s1]) for s in range(8)]
    zs = [torch.empty_like(v) for v in xs]
    ops = {"add": lambda i: N.vadd(xs[i % 8], ys[i % 8], q2, out=zs[i % 8]),
           "sub": lambda i: N.vsub(xs[i % 8], ys[i % 8], q2, out=zs[i % 8]),
           "mul": lambda i: N.vmul(xs[i % 8], ys[i % 8], q2, out=zs[i % 8]),
           "axpy": lambda i: N.axpy(a2, xs[i % 8], ys[i % 8], q2)}
    for name, fn in ops.items():
        ms = max_over_ranks(time_graph(fn, 64), world)
        rows[f"cfg2_{name}_elem_per_s"] = n2 / (ms * 1e-3)
        rows[f"cfg2_{name}_hbm_frac"] = 48 * nl / (ms * 1e-3) / 1e9 / pk["hbm_gbs"]   # per GPU
    del xs, ys, zs
    # cfg3 negacyclic polymul (B = 64 per rank)
    mods = P["cfg3"]["moduli"]
    qs, psis = [hexint(m["q"]) for m in mods], [hexint(m["psi"]) for m in mods]
    n3 = 1 << 16
    pn = N.Plan(16, qs, psis, batch=64, negacyclic=True, chain=True)
    a = to_dev(np.stack([synth.uniform_residues(qs[i], n3, synth.stream_seed(3, 0, i)) for i in range(64)]))
    b = to_dev(np.stack([synth.uniform_residues(qs[i], n3, synth.stream_seed(3, 1, i)) for i in range(64)]))
    c = torch.empty_like(a)
    for _ in range(3):
        pn.polymul(a, b, out=c)
    ms = timed_rank(lambda i: pn.polymul(a, b, out=c), 10, world)
    rows["cfg3_negacyclic_polymul_per_s"] = 64 * world / (ms * 1e-3)
    rows["cfg3_negacyclic_polymul_ms"] = ms
    del pn, a, b, c
    # cfg4 sweep: 1 GiB of coefficients in TOTAL per size, rank g owns polynomials
    # [g B/G, (g+1) B/G) of the same seeded batch (strong scaling; no collective)
    for logn in args.sweep:
        e = P["cfg4"][str(logn)]
        q, w = hexint(e["q"]), hexint(e["omega"])
        nn = 1 << logn
        Bn = (1 << 26) // nn
        b0, b1 = shard(Bn, world, rank)
        xfull = synth.uniform_residues(q, 1 << 26, synth.stream_seed(4, 0, logn)).reshape(Bn, nn, 2)
        ps = N.Plan(logn, q, w, batch=b1 - b0)
        xx = to_dev(xfull[b0:b1])
        del xfull
        yy, zz = torch.empty_like(xx), torch.empty_like(xx)
        for _ in range(2):
            ps.forward(xx, out=yy); ps.inverse(yy, out=zz)
        torch.cuda.synchronize()
        assert torch.equal(zz, xx), f"cfg4 N=2^{logn} round trip"
        ms = timed_rank(lambda i: (ps.forward(xx, out=yy), ps.inverse(yy, out=zz)), 20, world)
        bf = 2 * Bn * (nn // 2) * logn / (ms * 1e-3)
        rows[f"cfg4_logn{logn}_butterflies_per_s"] = bf
        rows[f"cfg4_logn{logn}_int_frac"] = round(bf / world * P_BUTTERFLY / 1e12 / pk["tprod_s"], 4)   # per GPU
        rows[f"cfg4_logn{logn}_arith_class"] = ps.arith_class()
        del ps, xx, yy, zz
        torch.cuda.empty_cache()
    # cfg5: N = 2^26 single transform through one plan (three passes), a replica per rank
    if args.cfg5:
        e = P["cfg5"]
        q, w = hexint(e["q"]), hexint(e["omega"])
        p5 = N.Plan(26, q, w)
        xx = to_dev(synth.uniform_residues(q, 1 << 26, synth.stream_seed(5, 0, 0)).reshape(1, 1 << 26, 2))
        yy = torch.empty_like(xx)
        zz = torch.empty_like(xx)
        p5.forward(xx, out=yy); p5.inverse(yy, out=zz)
        torch.cuda.synchronize()
        assert torch.equal(zz, xx)
        ms = timed_rank(lambda i: (p5.forward(xx, out=yy), p5.inverse(yy, out=zz)), 5, world)
        rows["cfg5_n2^26_fwd_inv_ms"] = ms
        rows["cfg5_butterflies_per_s"] = 2 * (1 << 25) * 26 / (ms * 1e-3)
        del p5, xx, yy, zz
        torch.cuda.empty_cache()
        rows.update(run_cfg5_fourstep(args, P, rank, world))
    # wider moduli, N = 2^16 x 32 forward + inverse per rank: the largest prime
    # < 2^b with q = 1 mod 2^21 for b = 256 (8 words, canonical), 254 (8 words, lazy class q < R/4),
    # 192 (6 words, canonical), 190 (6 words, lazy); roofline P = 136 (8 words: 128 + 8) or 78
    # (6 words: 72 + 6) word products per butterfly.  Row names keep the round-2 keys for b256 / b192.
    for key, name, P_w, sk in (("b256", "ntt256", 136, 16), ("b254", "ntt254_lazy", 136, 18),
                               ("b192", "ntt192", 78, 17), ("b190", "ntt190_lazy", 78, 19)):
        e = P["w256"][key]
        q = hexint(e["q"])
        w = pow(hexint(e["omega"]), 1 << (e["logn"] - 16), q)
        p6 = N.Plan256(16, q, w, batch=32)
        xx = torch.from_numpy(synth.uniform_residues_w(q, 32 << 16, synth.stream_seed(10, 0, sk))
                              .reshape(32, 1 << 16, 4).view(np.int64)).cuda()
        yy, zz = torch.empty_like(xx), torch.empty_like(xx)
        p6.forward(xx, out=yy); p6.inverse(yy, out=zz)
        torch.cuda.synchronize()
        assert torch.equal(zz, xx)
        ms = timed_rank(lambda i: (p6.forward(xx, out=yy), p6.inverse(yy, out=zz)), 10, world)
        bf = 2 * 32 * (1 << 15) * 16 / (ms * 1e-3)
        rows[f"f4_{name}_n2^16_x32_butterflies_per_s"] = bf * world
        rows[f"f4_{name}_roofline_frac"] = bf * P_w / (pk["tprod_s"] * 1e12)
        del p6, xx, yy, zz
        torch.cuda.empty_cache()
    return rows


def run_cfg5_fourstep(args, P, rank, world):
    """cfg 5: one N = 2^26 forward + inverse NTT as a four-step (2^9 x 2^17) transform
    partitioned over the `world` ranks; every rank holds N/G coefficients
    (columns layout), timing = max over ranks.  Two transports: "nccl" (pass A stores into
    the send blocks, one NCCL all-to-all per direction) and "p2p" (pass A's
    last pass stores each block straight into its destination rank's symmetric-memory
    receive buffer); a transport the box cannot provide is reported as *_unavailable.  Third
    row "_natural": the natural block layout (rank g holds x[g N/G, (g+1) N/G) in and y's
    slice out; pack + unpack and two more all-to-alls per direction)."""
    import torch
    from paper_2509_12494_b200 import fourstep as FS
    import synth
    e = P["cfg5"]
    q, w = hexint(e["q"]), hexint(e["omega"])
    out = {"cfg5_fourstep_gpus": world, "cfg5_fourstep_split": list(FS.split(26))}
    for transport, layout in (("nccl", "transposed"), ("p2p", "transposed"), ("nccl", "natural")):
        tag = {"nccl": "cfg5_fourstep", "p2p": "cfg5_fourstep_p2p"}[transport] + ("_natural" if layout == "natural" else "")
        try:
            fs = FS.FourStep(26, q, w, rank, world, None, transport=transport, layout=layout)
            ok = 1.0
        except Exception as ex:                      # e.g. no peer mappings on this box
            fs, ok = None, 0.0
            out[f"{tag}_unavailable"] = str(ex).splitlines()[0][:200]
        if max_over_ranks(1.0 - ok, world) > 0:      # every rank runs the transport or none does
            out.setdefault(f"{tag}_unavailable", "unavailable on another rank")
            continue
        L = fs.local
        cols = to_dev(synth.uniform_residues(q, L.R1 * L.n2, synth.stream_seed(5, 0, 100 + rank)).reshape(L.R1, L.n2, 2))
        if layout == "natural":   # this rank's contiguous slice of x (and of y)
            cols = cols.reshape(L.R1 * L.n2, 2)
            rows = torch.empty_like(cols)
        else:
            rows = torch.empty((L.R2, L.n1, 2), dtype=cols.dtype, device=cols.device)
        back = torch.empty_like(cols)
        for _ in range(2):
            fs.forward(cols, out=rows)
            fs.inverse(rows, out=back)
        torch.cuda.synchronize()
        assert torch.equal(back, cols), f"cfg5 four-step ({transport}, {layout}) round trip mismatch"
        ms = timed_rank(lambda i: (fs.forward(cols, out=rows), fs.inverse(rows, out=back)), 5, world)
        bfly = 2 * (1 << 25) * 26
        out[f"{tag}_fwd_inv_ms"] = ms
        out[f"{tag}_butterflies_per_s"] = bfly / (ms * 1e-3)
        if transport == "nccl" and layout == "transposed":
            out["cfg5_fourstep_a2a_bytes_per_rank_per_direction"] = 16 * L.R1 * L.R2 * (world - 1)
        del fs, cols, rows, back
        torch.cuda.empty_cache()
    return out


# ----------------------------------------------------------------------------- oracle legs
def cpu_baseline(P, npolys: int = 16):
    """The oracle (radix-2 on unsigned __int128, shift-subtract remainders) timed on this
    host's cores: forward + inverse of `npolys` of the cfg3 polynomials (bounded sample)."""
    from oracle import oracle as O
    mods = P["cfg3"]["moduli"][:npolys]
    qs, ws = [hexint(m["q"]) for m in mods], [hexint(m["omega"]) for m in mods]
    import synth
    n = 1 << P["cfg3"]["logn"]
    x = np.stack([synth.uniform_residues(qs[i], n, synth.stream_seed(3, 0, i)) for i in range(npolys)])
    t0 = time.perf_counter()
    y = O.ntt(x, qs, ws)
    z = O.intt(y, qs, ws)
    dt = time.perf_counter() - t0
    assert np.array_equal(z, x)
    bfly = 2 * npolys * (n // 2) * P["cfg3"]["logn"]
    return {"value": bfly / dt, "unit": "butterflies/s", "cores": O.num_threads(), "kind": "oracle",
            "sample": f"forward+inverse of {npolys} of the 64 cfg3 polynomials (N=2^16), {dt:.2f} s wall"}


def oracle_rows(P, cfg4_coeffs: int = 1 << 20):
    """The oracle beside the other rows (SURVEY.md §8(d) "Oracle timing"), bounded: cfg1 and
    cfg2 in full, cfg4 on `cfg4_coeffs` coefficients per size (2^20 instead of the survey's
    2^23, to keep the default run within minutes), rates per second (extrapolation-free)."""
    from oracle import oracle as O
    import synth
    rows = {"cores": O.num_threads()}
    e = P["cfg1"]
    q, w = hexint(e["q"]), hexint(e["omega"])
    x = synth.uniform_residues(q, 1024, synth.stream_seed(1, 0, 0))
    t0 = time.perf_counter()
    for _ in range(20):
        assert np.array_equal(O.intt(O.ntt(x, q, w), q, w), x)
    rows["cfg1_n1024_fwd_inv_us"] = (time.perf_counter() - t0) / 20 * 1e6
    q2, a2, n2 = hexint(P["cfg2"]["q"]), hexint(P["cfg2"]["a"]), P["cfg2"]["n"]
    xv = synth.uniform_residues(q2, n2, synth.stream_seed(2, 0, 0))
    yv = synth.uniform_residues(q2, n2, synth.stream_seed(2, 1, 0))
    for name, fn in (("add", lambda: O.vadd(xv, yv, q2)), ("sub", lambda: O.vsub(xv, yv, q2)),
                     ("mul", lambda: O.vmul(xv, yv, q2)), ("axpy", lambda: O.axpy(a2, xv, yv, q2))):
        t0 = time.perf_counter()
        fn()
        rows[f"cfg2_{name}_elem_per_s"] = n2 / (time.perf_counter() - t0)
    for logn in range(10, 18):
        e = P["cfg4"][str(logn)]
        q, w = hexint(e["q"]), hexint(e["omega"])
        B = max(1, cfg4_coeffs >> logn)
        x = synth.uniform_residues(q, B << logn, synth.stream_seed(4, 0, logn)).reshape(B, 1 << logn, 2)
        t0 = time.perf_counter()
        assert np.array_equal(O.intt(O.ntt(x, q, w), q, w), x)
        rows[f"cfg4_logn{logn}_butterflies_per_s"] = 2 * B * (1 << (logn - 1)) * logn / (time.perf_counter() - t0)
    rows["sample"] = (f"cfg1 x20, cfg2 full (n=2^20), cfg4 {cfg4_coeffs} coefficients per size; cfg5 not timed "
                      "(the oracle's 2^26 radix-2 transform takes minutes)")
    return rows


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    P = load_params()
    from oracle import oracle as O
    # one polynomial per host thread (the oracle parallelises over polynomials), at most 16:
    # a step is ~1.5 s of host work however many cores the box has
    npolys = max(1, min(16, O.num_threads()))
    vals = []
    cb = None
    for _ in range(args.warmup):
        cpu_baseline(P, npolys=npolys)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cb = cpu_baseline(P, npolys=npolys)
        vals.append(cb["value"])
    wall = time.perf_counter() - t0
    value = statistics.mean(vals)
    n, B = 1 << 16, 64
    out = {"impl": "reference", "metric": "128-bit NTT butterflies/sec (N=2^16, fwd+inv, 64 RNS primes)",
           "value": value, "unit": "butterflies/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * wall / max(1, args.steps), "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "u128", "data": "synthetic (seeded uniform residues)",
           "config": {"workload": "cfg3: batched forward+inverse cyclic NTT, N=2^16, 64 distinct 124-128-bit primes "
                                  f"(BASELINE.json configs[2]); each step a bounded sample of {npolys} of the 64 polynomials",
                      "N": n, "batch_per_gpu": B},
           "cpu_baseline": {"value": value, "unit": "butterflies/s", "cores": cb["cores"], "kind": "oracle",
                            "sample": cb["sample"]},
           "e2e": {"value": value, "unit": "butterflies/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def launch_selftest(args):
    """every rank reports its rank, world size and its shards of the cfg4 N = 2^16 batch and
    the cfg2 vector; rank 0 gathers them (gloo) and prints one JSON line"""
    import torch.distributed as dist
    rank, world, _ = dist_setup(args.gpus)
    mine = {"rank": rank, "world": world, "cfg4_logn16": shard(1024, world, rank), "cfg2": shard(1 << 20, world, rank)}
    allv = [None] * world
    if world > 1:
        dist.all_gather_object(allv, mine)
        dist.destroy_process_group()
    else:
        allv = [mine]
    if rank == 0:
        print(json.dumps({"launch_selftest": allv}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", dest="rows", action="store_true", default=True)
    ap.add_argument("--no-rows", dest="rows", action="store_false")
    ap.add_argument("--sweep", type=lambda s: [int(v) for v in s.split(",") if v], default=list(range(10, 18)))
    ap.add_argument("--no-cfg5", dest="cfg5", action="store_false", default=True)
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false", default=True)
    ap.add_argument("--no-spawn", dest="spawn", action="store_false", default=True,
                    help="with --gpus > 1 and no WORLD_SIZE: run one process instead of launching the ranks")
    ap.add_argument("--launch-selftest", action="store_true", default=False,
                    help="host-only check of the rank launch and the batch shards (gloo; no GPU work)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.spawn:
        sys.exit(spawn_ranks(args.gpus))
    if args.launch_selftest:
        launch_selftest(args)
        return
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()

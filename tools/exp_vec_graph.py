"""Experiment: cfg2 BLAS ops as CUDA-graph replays (launch overhead excluded, as in bench.py),
8 rotating buffer sets (> L2)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2509_12494_b200._lib_override as _libo  # noqa: E402
_libo.PATH = __import__("os").environ.get("NTT128_LIB")  # experiment builds only (tools/)
from paper_2509_12494_b200 import ntt128 as N  # noqa: E402
import synth  # noqa: E402

P = json.load(open("tests/golden/params.json"))
q, n, a = int(P["cfg2"]["q"], 16), P["cfg2"]["n"], int(P["cfg2"]["a"], 16)
xs = [torch.from_numpy(synth.uniform_residues(q, n, 10 + s).view(np.int64)).cuda() for s in range(8)]
ys = [torch.from_numpy(synth.uniform_residues(q, n, 20 + s).view(np.int64)).cuda() for s in range(8)]
zs = [torch.empty_like(v) for v in xs]
hbm = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6500
out = []
# spot check of every op on set 0 against Python integers (experiment kernels must stay exact)
rng = np.random.default_rng(5)
idx = rng.integers(0, n, 2000)
xi, yi = synth.to_ints(xs[0].cpu().numpy().view(np.uint64)[idx]), synth.to_ints(ys[0].cpu().numpy().view(np.uint64)[idx])
for name, ref in (("add", lambda u, v: (u + v) % q), ("mul", lambda u, v: u * v % q), ("axpy", lambda u, v: (a * u + v) % q)):
    if name == "axpy":
        zt = ys[0].clone(); N.axpy(a, xs[0], zt, q)
    else:
        zt = (N.vadd if name == "add" else N.vmul)(xs[0], ys[0], q)
    torch.cuda.synchronize()
    got = synth.to_ints(zt.cpu().numpy().view(np.uint64)[idx])
    assert got == [ref(u, v) for u, v in zip(xi, yi)], name + " mismatch"
for name, fn in [("add", N.vadd), ("mul", N.vmul)] + [("axpy", None)]:
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(8):
            (fn(xs[i], ys[i], q, out=zs[i]) if fn else N.axpy(a, xs[i], ys[i], q))
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(64):
            (fn(xs[i % 8], ys[i % 8], q, out=zs[i % 8]) if fn else N.axpy(a, xs[i % 8], ys[i % 8], q))
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 64
    out.append("%s %.2fus %.1f%%" % (name, ms * 1e3, 100 * 48 * n / (ms * 1e-3) / 1e9 / hbm))
print(os.environ.get("TAG", ""), " | ".join(out))

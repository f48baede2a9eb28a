"""A/B of NTT128_FLAG_CHAIN (DESIGN.md §6 "Chained calls") on the cfg3 headline step (fwd + inv,
64 polys, 4 rotating buffer sets, 100 steps x 3 repeats, best), cfg3 negacyclic polymul x64,
and cfg4 N = 2^12..2^17 (1 GiB) fwd+inv; correctness asserted first."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402
from paper_2509_12494_b200 import ntt128 as N  # noqa: E402
import synth  # noqa: E402

P = json.load(open("tests/golden/params.json"))
mods = P["cfg3"]["moduli"]
qs = [int(m["q"], 16) for m in mods]
ws = [int(m["omega"], 16) for m in mods]
psis = [int(m["psi"], 16) for m in mods]
X = [torch.from_numpy(np.stack([synth.uniform_residues(qs[i], 1 << 16, 100 * s + i) for i in range(64)]).view(np.int64)).cuda() for s in range(4)]
Y = [torch.empty_like(x) for x in X]
Z = [torch.empty_like(x) for x in X]


def best_of(fn, iters, reps=3):
    b = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(iters):
            fn(i)
        e1.record(); e1.synchronize()
        b = min(b, e0.elapsed_time(e1) / iters)
    return b


out = []
for chain in (False, True, False, True):
    plan = N.Plan(16, qs, ws, batch=64, chain=chain)
    plan.forward(X[0], out=Y[0]); plan.inverse(Y[0], out=Z[0])
    torch.cuda.synchronize()
    assert torch.equal(Z[0], X[0])
    sel = [0, 13, 40, 63]
    ref = O.ntt(np.ascontiguousarray(X[0].cpu().numpy().view(np.uint64)[sel]), [qs[i] for i in sel], [ws[i] for i in sel])
    assert np.array_equal(Y[0].cpu().numpy().view(np.uint64)[sel], ref)
    ms = best_of(lambda i: (plan.forward(X[i % 4], out=Y[i % 4]), plan.inverse(Y[i % 4], out=Z[i % 4])), 100)
    pm = N.Plan(16, qs, psis, batch=64, negacyclic=True, chain=chain)
    pm.polymul(X[0], X[1], out=Z[2]); torch.cuda.synchronize()
    ms_pm = best_of(lambda i: pm.polymul(X[i % 4], X[(i + 1) % 4], out=Z[i % 4]), 50)
    row = "chain=%d: cfg3 %.4f ms/step %.3e bfly/s | polymul x64 %.4f ms" % (chain, ms, 2 * 64 * (1 << 15) * 16 / (ms * 1e-3), ms_pm)
    del plan, pm
    for logn in (12, 14, 16, 17):
        e = P["cfg4"][str(logn)]
        q, w = int(e["q"], 16), int(e["omega"], 16)
        B = (1 << 26) >> logn
        p = N.Plan(logn, q, w, batch=B, chain=chain)
        x = torch.from_numpy(synth.uniform_residues(q, 1 << 26, logn).reshape(B, 1 << logn, 2).view(np.int64)).cuda()
        y, z = torch.empty_like(x), torch.empty_like(x)
        p.forward(x, out=y); p.inverse(y, out=z); torch.cuda.synchronize()
        assert torch.equal(z, x)
        t = best_of(lambda i: (p.forward(x, out=y), p.inverse(y, out=z)), 10)
        row += " | 2^%d %.3f ms" % (logn, t)
        del p, x, y, z
        torch.cuda.empty_cache()
    print(row, flush=True)

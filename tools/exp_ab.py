"""A/B of a library build (NTT128_LIB) on the cfg3 headline step (fwd + inv, 64 polys, 4 rotating
buffer sets, 100 steps x 3 repeats, best), with a correctness check first: 4 polynomials of
every modulus class against the oracle, the whole batch round-tripped; plus cfg4 N = 2^12..2^17
(1 GiB) and cfg5 N = 2^26 fwd+inv timings."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2509_12494_b200._lib_override as _libo  # noqa: E402
_libo.PATH = os.environ.get("NTT128_LIB")  # experiment builds only (tools/)
from oracle import oracle as O  # noqa: E402
from paper_2509_12494_b200 import ntt128 as N  # noqa: E402
import synth  # noqa: E402

tag = os.path.basename(os.environ.get("NTT128_LIB", "default"))
P = json.load(open("tests/golden/params.json"))
mods = P["cfg3"]["moduli"]
qs = [int(m["q"], 16) for m in mods]
ws = [int(m["omega"], 16) for m in mods]
plan = N.Plan(16, qs, ws, batch=64)
X = [torch.from_numpy(np.stack([synth.uniform_residues(qs[i], 1 << 16, 100 * s + i) for i in range(64)]).view(np.int64)).cuda() for s in range(4)]
Y = [torch.empty_like(x) for x in X]
Z = [torch.empty_like(x) for x in X]
plan.forward(X[0], out=Y[0]); plan.inverse(Y[0], out=Z[0])
torch.cuda.synchronize()
assert torch.equal(Z[0], X[0]), "round trip"
sel = [0, 1, 2, 63]
x0 = X[0].cpu().numpy().view(np.uint64)
ref = O.ntt(np.ascontiguousarray(x0[sel]), [qs[i] for i in sel], [ws[i] for i in sel])
assert np.array_equal(Y[0].cpu().numpy().view(np.uint64)[sel], ref), "forward != oracle"
steps = 100
best = 1e9
for r in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        plan.forward(X[i % 4], out=Y[i % 4]); plan.inverse(Y[i % 4], out=Z[i % 4])
    e1.record(); e1.synchronize()
    best = min(best, e0.elapsed_time(e1) / steps)
bf = 2 * 64 * (1 << 15) * 16
out = ["%s: cfg3 %.4f ms/step %.3e bfly/s" % (tag, best, bf / (best * 1e-3))]
del plan, X, Y, Z
torch.cuda.empty_cache()
for logn in [int(v) for v in os.environ.get("AB_SIZES", "12,14,16,17").split(",") if v]:
    e = P["cfg4"][str(logn)]
    q, w = int(e["q"], 16), int(e["omega"], 16)
    B = (1 << 26) >> logn
    p = N.Plan(logn, q, w, batch=B)
    x = torch.from_numpy(synth.uniform_residues(q, 1 << 26, logn).reshape(B, 1 << logn, 2).view(np.int64)).cuda()
    y, z = torch.empty_like(x), torch.empty_like(x)
    p.forward(x, out=y); p.inverse(y, out=z)
    torch.cuda.synchronize()
    assert torch.equal(z, x)
    bst = 1e9
    for r in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(10):
            p.forward(x, out=y); p.inverse(y, out=z)
        e1.record(); e1.synchronize()
        bst = min(bst, e0.elapsed_time(e1) / 10)
    out.append("2^%d %.3f ms %.3e" % (logn, bst, B * (1 << (logn - 1)) * logn * 2 / (bst * 1e-3)))
    del p, x, y, z
    torch.cuda.empty_cache()
print(" | ".join(out), flush=True)

"""Experiment: the bench's timed loop with and without per-call events, 1 vs 4 buffer sets."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2509_12494_b200._lib_override as _libo  # noqa: E402
_libo.PATH = __import__("os").environ.get("NTT128_LIB")  # experiment builds only (tools/)
from paper_2509_12494_b200 import ntt128 as N  # noqa: E402
import synth  # noqa: E402

P = json.load(open("tests/golden/params.json"))
mods = P["cfg3"]["moduli"]
qs = [int(m["q"], 16) for m in mods]
ws = [int(m["omega"], 16) for m in mods]
plan = N.Plan(16, qs, ws, batch=64)
X = [torch.from_numpy(np.stack([synth.uniform_residues(qs[i], 1 << 16, 100 * s + i) for i in range(64)]).view(np.int64)).cuda() for s in range(4)]
Y = [torch.empty_like(x) for x in X]
Z = [torch.empty_like(x) for x in X]
steps = 20
for nsets in (1, 4):
    for events in (False, True):
        for i in range(5):
            plan.forward(X[i % nsets], out=Y[i % nsets]); plan.inverse(Y[i % nsets], out=Z[i % nsets])
        torch.cuda.synchronize()
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(steps):
            k = i % nsets
            if events: ev[i][0].record()
            plan.forward(X[k], out=Y[k])
            if events: ev[i][1].record()
            plan.inverse(Y[k], out=Z[k])
            if events: ev[i][2].record()
        e1.record(); e1.synchronize()
        ms = e0.elapsed_time(e1) / steps
        bf = 2 * 64 * (1 << 15) * 16 / (ms * 1e-3)
        print("sets %d events %d: %.4e bfly/s  %.1f%%" % (nsets, events, bf, 100 * bf * 36 / 9.3062e12))

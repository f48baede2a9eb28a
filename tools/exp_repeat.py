"""Experiment: cfg3 fwd+inv step time with the library in NTT128_LIB (no result check), for
the NTT_COMPUTE_REPEAT builds: rep0 (memory phases only), default (1), rep2 (rounds twice).
time(rep2) - time(rep1) = the register rounds' share; time(rep1) minus that = everything else."""
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
mods = P["cfg3"]["moduli"]
qs = [int(m["q"], 16) for m in mods]
ws = [int(m["omega"], 16) for m in mods]
plan = N.Plan(16, qs, ws, batch=64)
X = [torch.from_numpy(np.stack([synth.uniform_residues(qs[i], 1 << 16, 100 * s + i) for i in range(64)]).view(np.int64)).cuda() for s in range(4)]
Y = [torch.empty_like(x) for x in X]
Z = [torch.empty_like(x) for x in X]
steps = 100
for i in range(8):
    plan.forward(X[i % 4], out=Y[i % 4]); plan.inverse(Y[i % 4], out=Z[i % 4])
torch.cuda.synchronize()
best = 1e9
for r in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        plan.forward(X[i % 4], out=Y[i % 4]); plan.inverse(Y[i % 4], out=Z[i % 4])
    e1.record(); e1.synchronize()
    best = min(best, e0.elapsed_time(e1) / steps)
print("%s: %.4f ms/step" % (os.path.basename(os.environ.get("NTT128_LIB", "default")), best))

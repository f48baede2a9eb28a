"""Experiment: cfg3 negacyclic polymul x64 (N = 2^16), permutation-free path vs the
natural-order path (NTT128_NO_NC=1 in the environment selects the latter)."""
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
qs, psis = [int(m["q"], 16) for m in mods], [int(m["psi"], 16) for m in mods]
n, B = 1 << 16, 64
pn = N.Plan(16, qs, psis, batch=B, negacyclic=True)
a = torch.from_numpy(np.stack([synth.uniform_residues(qs[i], n, synth.stream_seed(3, 0, i)) for i in range(B)]).view(np.int64)).cuda()
b = torch.from_numpy(np.stack([synth.uniform_residues(qs[i], n, synth.stream_seed(3, 1, i)) for i in range(B)]).view(np.int64)).cuda()
c = torch.empty_like(a)
for _ in range(3):
    pn.polymul(a, b, out=c)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    pn.polymul(a, b, out=c)
e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1) / 20
print("polymul x64 N=2^16: %.3f ms  %.4e polymul/s" % (ms, B / (ms * 1e-3)))

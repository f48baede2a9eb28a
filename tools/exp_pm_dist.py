"""Experiment: distribution of per-call cfg3 negacyclic polymul times (CUDA events per call)."""
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
ev = [torch.cuda.Event(enable_timing=True) for _ in range(41)]
for _ in range(3):
    pn.polymul(a, b, out=c)
torch.cuda.synchronize()
ev[0].record()
for i in range(40):
    pn.polymul(a, b, out=c)
    ev[i + 1].record()
torch.cuda.synchronize()
print(" ".join("%.0f" % (ev[i].elapsed_time(ev[i + 1]) * 1e3) for i in range(40)))
fa, fb = torch.empty_like(a), torch.empty_like(a)
ev[0].record()
for i in range(40):
    pn.forward_bitrev(a, out=fa); pn.forward_bitrev(b, out=fb); pn.inverse_bitrev(fa, out=c)
    ev[i + 1].record()
torch.cuda.synchronize()
print(" ".join("%.0f" % (ev[i].elapsed_time(ev[i + 1]) * 1e3) for i in range(40)))

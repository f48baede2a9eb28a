"""Experiment: per-transform times at cfg3 size (64 x 2^16, 64 primes): cyclic forward /
inverse, negacyclic natural forward / inverse, and the permutation-free bit-reversed pair."""
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
psis = [int(m["psi"], 16) for m in mods]
n, B = 1 << 16, 64
pc = N.Plan(16, qs, ws, batch=B)
pn = N.Plan(16, qs, psis, batch=B, negacyclic=True)
x = torch.from_numpy(np.stack([synth.uniform_residues(qs[i], n, synth.stream_seed(3, 0, i)) for i in range(B)]).view(np.int64)).cuda()
y = torch.empty_like(x)


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for name, fn in [("cyclic fwd", lambda: pc.forward(x, out=y)), ("cyclic inv", lambda: pc.inverse(x, out=y)),
                 ("nega fwd", lambda: pn.forward(x, out=y)), ("nega inv", lambda: pn.inverse(x, out=y)),
                 ("nega fwd_bitrev", lambda: pn.forward_bitrev(x, out=y)), ("nega inv_bitrev", lambda: pn.inverse_bitrev(x, out=y))]:
    print("%-16s %8.1f us" % (name, t(fn)))
b = torch.from_numpy(np.stack([synth.uniform_residues(qs[i], n, synth.stream_seed(3, 1, i)) for i in range(B)]).view(np.int64)).cuda()
fa, fb, c = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
print("%-16s %8.1f us" % ("3 bitrev seq", t(lambda: (pn.forward_bitrev(x, out=fa), pn.forward_bitrev(b, out=fb), pn.inverse_bitrev(fa, out=c)))))
print("%-16s %8.1f us" % ("polymul", t(lambda: pn.polymul(x, b, out=c))))

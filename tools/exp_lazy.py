"""Experiment: fwd+inv time of a 64 x 2^16 batch whose primes are all 128-bit, all 124-bit
(lazy path), or the cfg3 mix."""
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
sets = {"mix": list(range(64)), "all128": [0] * 64, "all124": [4] * 64, "all126": [2] * 64}
for name, idx in sets.items():
    qs = [int(mods[i]["q"], 16) for i in idx]
    ws = [int(mods[i]["omega"], 16) for i in idx]
    plan = N.Plan(16, qs, ws, batch=64)
    x = torch.from_numpy(np.stack([synth.uniform_residues(qs[i], 1 << 16, i) for i in range(64)]).view(np.int64)).cuda()
    y, z = torch.empty_like(x), torch.empty_like(x)
    for _ in range(5):
        plan.forward(x, out=y); plan.inverse(y, out=z)
    torch.cuda.synchronize()
    assert torch.equal(z, x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        plan.forward(x, out=y); plan.inverse(y, out=z)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(name, "ms/step %.4f" % ms, "bfly/s %.4e" % (2 * 64 * 32768 * 16 / (ms * 1e-3)))

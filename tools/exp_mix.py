"""Experiment: N = 2^16 x 64 forward+inverse with (a) cfg3's 64 moduli (three classes mixed)
and (b) the LAZY-class moduli only, one buffer set; `python tools/exp_mix.py [a|b]` runs one
(for ncu), no argument runs both."""
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
cases = {"a": mods, "b": ([m for m in mods if int(m["q"], 16).bit_length() <= 126] * 2)[:64]}
for name in (sys.argv[1:] or ["a", "b"]):
    sel = cases[name]
    qs = [int(m["q"], 16) for m in sel]
    ws = [int(m["omega"], 16) for m in sel]
    plan = N.Plan(16, qs, ws, batch=64)
    x = torch.from_numpy(np.stack([synth.uniform_residues(qs[i], 1 << 16, i) for i in range(64)]).view(np.int64)).cuda()
    y, z = torch.empty_like(x), torch.empty_like(x)
    for _ in range(3):
        plan.forward(x, out=y); plan.inverse(y, out=z)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        plan.forward(x, out=y); plan.inverse(y, out=z)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    bf = 2 * 64 * (1 << 15) * 16 / (ms * 1e-3)
    print("case %s: %.4e bfly/s  %.1f%% of roofline" % (name, bf, 100 * bf * 36 / 9.3062e12))

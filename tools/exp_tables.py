"""Experiment: cost of per-polynomial twiddle tables.  N = 2^16 x 64 forward+inverse, all
moduli of one class: one shared modulus (nq = 1, tables L2-resident) vs one table per
polynomial (nq = 64, cfg3's moduli of that class repeated)."""
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
for cls, lo, hi in [("LAZY", 0, 126), ("HALF", 126, 127), ("FULL", 127, 128)]:
    sel = [m for m in mods if lo < int(m["q"], 16).bit_length() <= hi or (cls == "LAZY" and int(m["q"], 16).bit_length() <= 126)]
    sel = [m for m in sel if (int(m["q"], 16).bit_length() <= 126) == (cls == "LAZY")]
    sel = (sel * 64)[:64]
    qs = [int(m["q"], 16) for m in sel]
    ws = [int(m["omega"], 16) for m in sel]
    for nq in (1, 64):
        plan = N.Plan(16, qs[0] if nq == 1 else qs, ws[0] if nq == 1 else ws, batch=64)
        x = torch.from_numpy(np.stack([synth.uniform_residues(qs[0 if nq == 1 else i], 1 << 16, i) for i in range(64)]).view(np.int64)).cuda()
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
        print("%s nq=%2d (%d distinct): %.4e bfly/s  %.1f%% of roofline" % (cls, nq, len(set(qs)) if nq > 1 else 1, bf, 100 * bf * 36 / 9.3062e12))
        del plan, x, y, z

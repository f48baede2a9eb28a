"""Experiment: forward-NTT time per butterfly vs batch size at N=2^16 (one 128-bit prime):
exposes wave quantisation (4 groups per CTA, 6 CTAs per SM -> 888 CTAs per wave)."""
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
e = P["cfg4"]["16"]
q, w = int(e["q"], 16), int(e["omega"], 16)
n = 1 << 16
for B in [int(v) for v in sys.argv[1].split(",")]:
    plan = N.Plan(16, q, w, batch=B)
    x = torch.from_numpy(synth.uniform_residues(q, B * n, 16).reshape(B, n, 2).view(np.int64)).cuda()
    y = torch.empty_like(x)
    for _ in range(3):
        plan.forward(x, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        plan.forward(x, out=y)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    bf = B * (n // 2) * 16
    print("B %4d  ctas/pass %6d  waves %.2f  %.3f ms  %.4e bfly/s  %.3f bfly/clk/SM" % (B, B * 64, B * 64 / 888, ms, bf / (ms * 1e-3), bf / (ms * 1e-3) / 148 / 1.965e9))
    del plan, x, y
    torch.cuda.empty_cache()

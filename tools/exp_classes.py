"""Experiment: forward+inverse throughput at N = 2^16 x 64 for one modulus class at a time
(q < 2^126 Harvey, 2^126 <= q < 2^127 half-lazy, q >= 2^127 canonical), against the
register-only ceilings of tools/micro/bfly_rate.cu."""
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
for key, e in [("LAZY b124", P["extra"]["b124"]), ("LAZY b126", P["extra"]["b126"]), ("HALF b127", P["extra"]["b127"]),
               ("FULL rand128", P["extra"]["rand128_0"]), ("FULL cfg4", P["cfg4"]["16"])]:
    q = int(e["q"], 16)
    L = e["logn"]
    w = pow(int(e["psi"], 16), 1 << (L + 1 - 16), q)
    plan = N.Plan(16, q, w, batch=64)
    x = torch.from_numpy(synth.uniform_residues(q, 64 << 16, 3).reshape(64, 1 << 16, 2).view(np.int64)).cuda()
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
    print("%-14s %.4e bfly/s  %.3f bfly/clk/SM  %.1f%% of roofline" % (key, bf, bf / 148 / 1.965e9, 100 * bf * 36 / 9.3062e12))

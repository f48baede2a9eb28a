"""Experiment: cfg2 vec128_mul (n = 2^20, 128-bit q) elements/s and HBM fraction, rotating 8
buffer sets (> L2); NTT128_NO_BARRETT=1 selects the two-Montgomery kernel."""
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
q, n = int(P["cfg2"]["q"], 16), P["cfg2"]["n"]
xs = [torch.from_numpy(synth.uniform_residues(q, n, 10 + s).view(np.int64)).cuda() for s in range(8)]
ys = [torch.from_numpy(synth.uniform_residues(q, n, 20 + s).view(np.int64)).cuda() for s in range(8)]
zs = [torch.empty_like(v) for v in xs]
for i in range(8):
    N.vmul(xs[i], ys[i], q, out=zs[i])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(64):
    N.vmul(xs[i % 8], ys[i % 8], q, out=zs[i % 8])
e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1) / 64
hbm = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if __import__("os").path.exists("MEASURED_PEAKS.json") else 6500
print("vec128_mul n=2^20: %.2f us  %.3e elem/s  %.1f%% of HBM" % (ms * 1e3, n / (ms * 1e-3), 100 * 48 * n / (ms * 1e-3) / 1e9 / hbm))

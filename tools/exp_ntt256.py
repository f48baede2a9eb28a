"""Experiment: 256-bit NTT forward+inverse throughput (w256 prime PRIME, default b256; b192 runs
the 6-word kernels), N = 2^n, batch filling 2^21 residues (64 MiB)."""
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
import os  # noqa: E402
KEY = os.environ.get("PRIME", "b256")
PROD = 78 if KEY in ("b192", "b190") else 136
e = P["w256"][KEY]
q, L = int(e["q"], 16), e["logn"]
for logn in [int(v) for v in sys.argv[1].split(",")]:
    w = pow(int(e["omega"], 16), 1 << (L - logn), q)
    B = (1 << 21) >> logn
    plan = N.Plan256(logn, q, w, batch=B)
    x = torch.from_numpy(synth.uniform_residues_w(q, 1 << 21, logn).reshape(B, 1 << logn, 4).view(np.int64)).cuda()
    y, z = torch.empty_like(x), torch.empty_like(x)
    for _ in range(2):
        plan.forward(x, out=y); plan.inverse(y, out=z)
    torch.cuda.synchronize()
    assert torch.equal(z, x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        plan.forward(x, out=y); plan.inverse(y, out=z)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 5
    bf = 2 * B * (1 << (logn - 1)) * logn
    print("%s logn %2d batch %4d: %.3f ms  %.4e bfly/s  %.1f%% of the %d-product roofline" %
          (KEY, logn, B, ms, bf / (ms * 1e-3), 100 * bf / (ms * 1e-3) * PROD / 9.0992e12, PROD))

"""Experiment: fwd+inv throughput per size (1 GiB of coefficients, one 128-bit prime)."""
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
for logn in [int(v) for v in sys.argv[1].split(",")]:
    # cfg4 primes for 2^10..2^17; smaller sizes use the 2^10 prime's sub-roots, larger cfg5's
    key = str(min(max(logn, 10), 17))
    e = P["cfg4"][key] if logn <= 17 else P["cfg5"]
    q, w = int(e["q"], 16), int(e["omega"], 16)
    w = pow(w, 1 << (e["logn"] - logn), q)
    n = 1 << logn
    B = (1 << 26) // n
    plan = N.Plan(logn, q, w, batch=B)
    x = torch.from_numpy(synth.uniform_residues(q, 1 << 26, logn).reshape(B, n, 2).view(np.int64)).cuda()
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
    print("logn %2d passes %d  %.4e bfly/s" % (logn, plan.info()["num_passes"], 2 * B * (n // 2) * logn / (ms * 1e-3)))
    del plan, x, y, z
    torch.cuda.empty_cache()

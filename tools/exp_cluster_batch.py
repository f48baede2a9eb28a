"""Experiment: N = 1024 fwd+inv latency (graph replay) against the batch size, for the
cluster threshold NTT_CLU_MAX_BATCH (cluster kernel vs one-CTA latency shape vs batched)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2509_12494_b200._lib_override as _libo  # noqa: E402
_libo.PATH = __import__("os").environ.get("NTT128_LIB")  # experiment builds only (tools/)
from paper_2509_12494_b200 import ntt128 as N  # noqa: E402
import synth  # noqa: E402

P = json.load(open("tests/golden/params.json"))
e = P["cfg1"]
q, w = int(e["q"], 16), int(e["omega"], 16)
out = []
for B in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1,4,8,16,24,32,48,64").split(",")]:
    plan = N.Plan(10, q, w, batch=B)
    x = torch.from_numpy(synth.uniform_residues(q, 1024 * B, 1).reshape(B, 1024, 2).view(np.int64)).cuda()
    y, z = torch.empty_like(x), torch.empty_like(x)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            plan.forward(x, out=y); plan.inverse(y, out=z)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            plan.forward(x, out=y); plan.inverse(y, out=z)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); e1.synchronize()
    assert torch.equal(z, x)
    out.append("B=%d %.2fus" % (B, e0.elapsed_time(e1) * 1e3 / 20))
print(os.path.basename(os.environ.get("NTT128_LIB", "default")), " ".join(out))

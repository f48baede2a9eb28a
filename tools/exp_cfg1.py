"""Experiment: cfg1 (one N = 1024 polynomial) forward / inverse latency: CUDA events around
single calls, and CUDA-graph replays of forward + inverse."""
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
e = P["cfg1"]
q, w = int(e["q"], 16), int(e["omega"], 16)
plan = N.Plan(10, q, w)
x = torch.from_numpy(synth.uniform_residues(q, 1024, 1).reshape(1, 1024, 2).view(np.int64)).cuda()
y, z = torch.empty_like(x), torch.empty_like(x)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(5):
        plan.forward(x, out=y); plan.inverse(y, out=z)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for _ in range(50):
        plan.forward(x, out=y); plan.inverse(y, out=z)
g.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record(); e1.synchronize()
print("graph fwd+inv: %.2f us" % (e0.elapsed_time(e1) * 1e3 / 50))
assert torch.equal(z, x)

"""Plain calls (no graphs) of the non-headline kernels, for one ncu capture each: the cfg1
cluster transform (k_ntt_cluster) and the cfg2 BLAS kernels (k_vec)."""
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
q2, n2, a2 = int(P["cfg2"]["q"], 16), P["cfg2"]["n"], int(P["cfg2"]["a"], 16)
u = torch.from_numpy(synth.uniform_residues(q2, n2, 10).view(np.int64)).cuda()
v = torch.from_numpy(synth.uniform_residues(q2, n2, 20).view(np.int64)).cuda()
for _ in range(3):
    y = plan.forward(x)
    z = plan.inverse(y)
    N.vadd(u, v, q2)
    N.vmul(u, v, q2)
    N.axpy(a2, u, v, q2)
torch.cuda.synchronize()
assert torch.equal(z, x)
print("ok")

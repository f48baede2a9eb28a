"""cfg5 N = 2^26 forward + inverse on one GPU: three-pass plan vs the four-step (G = 1, both
transports), CUDA events, 10 iterations x 3 repeats, best of the repeats."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2509_12494_b200._lib_override as _libo  # noqa: E402
_libo.PATH = os.environ.get("NTT128_LIB")  # experiment builds only (tools/)
from paper_2509_12494_b200 import fourstep as FS  # noqa: E402
from paper_2509_12494_b200 import ntt128 as N  # noqa: E402
import synth  # noqa: E402

P = json.load(open("tests/golden/params.json"))
q, w = int(P["cfg5"]["q"], 16), int(P["cfg5"]["omega"], 16)
x = synth.uniform_residues(q, 1 << 26, 5)


def timeit(fn, it=10, rep=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(rep):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(it):
            fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / it)
    return best


p = N.Plan(26, q, w)
dx = torch.from_numpy(x.reshape(1, -1, 2).view(np.int64)).cuda()
dy, dz = torch.empty_like(dx), torch.empty_like(dx)
t3 = timeit(lambda: (p.forward(dx, out=dy), p.inverse(dy, out=dz)))
print(f"three-pass fwd+inv {t3:.3f} ms")
del p
torch.cuda.empty_cache()
l1, l2 = FS.split(26)
cols = torch.from_numpy(FS.to_columns(x, 1 << l1, 1 << l2, 0, 1).view(np.int64)).cuda()
for tr in ("nccl", "p2p"):
    fs = FS.FourStep(26, q, w, transport=tr)
    rows = torch.empty((fs.local.R2, fs.local.n1, 2), dtype=torch.int64, device="cuda")
    back = torch.empty_like(cols)
    t = timeit(lambda: (fs.forward(cols, out=rows), fs.inverse(rows, out=back)))
    assert torch.equal(back, cols)
    tf = timeit(lambda: fs.forward(cols, out=rows))
    print(f"four-step {tr} split {l1}x{l2}: fwd+inv {t:.3f} ms (fwd {tf:.3f}), vs three-pass {t3 / t:.3f}")
    del fs
    torch.cuda.empty_cache()

"""One cfg5 four-step forward + inverse at G = 1 in the natural block layout (after warm-up),
for an ncu capture of the pack / transpose kernels around the exchanges:
ncu -k regex:k_fs_ ... python tools/exp_fourstep_nat_prof.py"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2509_12494_b200 import fourstep as FS  # noqa: E402
import synth  # noqa: E402

P = json.load(open("tests/golden/params.json"))
q, w = int(P["cfg5"]["q"], 16), int(P["cfg5"]["omega"], 16)
x = torch.from_numpy(synth.uniform_residues(q, 1 << 26, 5).view(np.int64)).cuda()
fs = FS.FourStep(26, q, w, layout="natural")
y = torch.empty_like(x)
back = torch.empty_like(x)
for _ in range(2):
    fs.forward(x, out=y)
    fs.inverse(y, out=back)
torch.cuda.synchronize()
assert torch.equal(back, x)

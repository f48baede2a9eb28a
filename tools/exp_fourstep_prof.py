"""One cfg5 four-step forward + inverse at G = 1 (after warm-up), for an ncu launch list:
ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/exp_fourstep_prof.py"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2509_12494_b200 import fourstep as FS  # noqa: E402
import synth  # noqa: E402

P = json.load(open("tests/golden/params.json"))
q, w = int(P["cfg5"]["q"], 16), int(P["cfg5"]["omega"], 16)
l1, l2 = FS.split(26)
x = synth.uniform_residues(q, 1 << 26, 5)
cols = torch.from_numpy(FS.to_columns(x, 1 << l1, 1 << l2, 0, 1).view(np.int64)).cuda()
fs = FS.FourStep(26, q, w)
rows = torch.empty((fs.local.R2, fs.local.n1, 2), dtype=torch.int64, device="cuda")
back = torch.empty_like(cols)
for _ in range(2):
    fs.forward(cols, out=rows)
    fs.inverse(rows, out=back)
torch.cuda.synchronize()
assert torch.equal(back, cols)

"""Experiment: per-tile timeline of cfg3 fwd+inv steps with the -DNTT_TRACE=1 library
(paper_2509_12494_b200/libntt128_trace.so).  Every multi-pass tile records globaltimer at
start, after its loads, after its stores, with its SM and pass.  Reports, per pass, the
span, the time-weighted number of tiles resident / computing per SM, and the gaps where an
SM had no tile computing (ramp-up, drains, boundaries).

    NTT128_LIB=$PWD/paper_2509_12494_b200/libntt128_trace.so python tools/exp_trace.py
"""
import ctypes
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
mods = P["cfg3"]["moduli"]
qs = [int(m["q"], 16) for m in mods]
ws = [int(m["omega"], 16) for m in mods]
plan = N.Plan(16, qs, ws, batch=64)
X = [torch.from_numpy(np.stack([synth.uniform_residues(qs[i], 1 << 16, 100 * s + i) for i in range(64)]).view(np.int64)).cuda() for s in range(4)]
Y = [torch.empty_like(x) for x in X]
Z = [torch.empty_like(x) for x in X]
for i in range(8):
    plan.forward(X[i % 4], out=Y[i % 4]); plan.inverse(Y[i % 4], out=Z[i % 4])
torch.cuda.synchronize()
cap = 1 << 20
buf = torch.zeros(cap * 2, dtype=torch.int64, device="cuda")
N._L.ntt128_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_ulonglong]
assert N._L.ntt128_debug_trace(buf.data_ptr(), cap) == 0
torch.cuda.synchronize()
steps = 4
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(steps):
    plan.forward(X[i % 4], out=Y[i % 4]); plan.inverse(Y[i % 4], out=Z[i % 4])
e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1)
raw = buf.cpu().numpy().view(np.uint32).reshape(-1, 4)
raw = raw[raw[:, 2] != 0]
t0 = raw[:, 0].astype(np.int64)
base = t0.min()
def rel(v):
    return ((v.astype(np.int64) - base) & 0xffffffff) / 1e3     # us (globaltimer ns, 32-bit wrap)
start, loaded, end = rel(raw[:, 0]), rel(raw[:, 1]), rel(raw[:, 2])
sm = raw[:, 3] >> 16
first = raw[:, 3] & 1
print(f"{len(raw)} tiles, {steps} steps, {ms / steps * 1e3:.1f} us/step by events, trace span {end.max():.1f} us")
print(f"tile duration: mean {np.mean(end - start):.2f} us, load phase mean {np.mean(loaded - start):.2f} us "
      f"(p10 {np.percentile(loaded - start, 10):.2f}, p90 {np.percentile(loaded - start, 90):.2f})")
# passes in launch order: split by start time clusters of (first flag) changes
order = np.argsort(start)
# time grid per SM: computing tiles count
T = end.max()
dt = 0.5
bins = np.arange(0, T + dt, dt)
nsm = int(sm.max()) + 1
comp = np.zeros((nsm, len(bins)))
resid = np.zeros((nsm, len(bins)))
for s_, l_, e_, m_ in zip(start, loaded, end, sm):
    i0, i1, i2 = int(s_ / dt), int(l_ / dt), int(e_ / dt)
    resid[m_, i0:i2 + 1] += 1
    comp[m_, i1:i2 + 1] += 1
idle = (comp == 0).mean()
print(f"SM-time with no tile past its load phase: {100 * idle:.1f} %; mean resident tiles/SM {resid.mean():.2f}, "
      f"computing {comp.mean():.2f}")
# timeline summary (per 10 us): mean computing tiles per SM
w = int(10 / dt)
line = []
for k in range(0, len(bins), w):
    line.append("%.1f" % comp[:, k:k + w].mean())
print("computing tiles per SM, per 10 us:", " ".join(line))
# per pass spans (first pass = flag 1)
for f in (1, 0):
    sel = first == f
    print(f"first={f}: tiles {sel.sum()}, load mean {np.mean(loaded[sel] - start[sel]):.2f} us, "
          f"compute+store mean {np.mean(end[sel] - loaded[sel]):.2f} us")
np.save("gpurun_out/trace.npy", raw)

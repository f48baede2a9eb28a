"""Small invocations of every kernel family, for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck): SURVEY §4 "Sanitizers".  Self-checking without the oracle: round
trips, and the same transform through different launch shapes must agree bit for bit.

    compute-sanitizer --tool racecheck python tools/sanitize_driver.py

Shapes: the 8-CTA cluster kernel (N = 2^10, 1 polynomial), the one-CTA latency shape
(40 polynomials), the batched single pass (400), two passes with pass-overlap counters
(N = 2^14), the permutation-free negacyclic passes and polymul (N = 2^12), the BLAS ops
(ragged n), the 256-bit and 192-bit (6-word) passes, and the four-step in the natural block
layout (pack / transpose kernels) against the three-pass plan.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_12494_b200 import ntt128 as N  # noqa: E402
import synth  # noqa: E402

P = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                                "params.json")))


def h(v):
    return int(v, 16) if isinstance(v, str) else int(v)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


def sub_root(e, logn, nega=False):
    q, L = h(e["q"]), e["logn"]
    return pow(h(e["psi"]), 1 << ((L - logn) if nega else (L + 1 - logn)), q)


def main():
    e = P["cfg4"]["16"]
    q = h(e["q"])
    # N = 2^10 through three launch shapes: cluster (1), latency shape (40), batched (400)
    w = sub_root(e, 10)
    x = synth.uniform_residues(q, 400 << 10, 11).reshape(400, 1 << 10, 2)
    ys = []
    for b in (1, 40, 400):
        plan = N.Plan(10, q, w, batch=b)
        d = dev(x[:b])
        y = plan.forward(d)
        assert torch.equal(plan.inverse(y), d), f"round trip b={b}"
        ys.append(y[:1].clone())
    assert torch.equal(ys[0], ys[1]) and torch.equal(ys[0], ys[2]), "launch shapes disagree"
    # two passes with overlap counters, in place
    w14 = sub_root(e, 14)
    x14 = dev(synth.uniform_residues(q, 2 << 14, 12).reshape(2, 1 << 14, 2))
    p14 = N.Plan(14, q, w14, batch=2)
    d = x14.clone()
    p14.forward(d, out=d)
    p14.inverse(d, out=d)
    assert torch.equal(d, x14), "two-pass round trip"
    # negacyclic permutation-free path and polymul
    psi = sub_root(e, 12, nega=True)
    a = dev(synth.uniform_residues(q, 2 << 12, 13).reshape(2, 1 << 12, 2))
    bb = dev(synth.uniform_residues(q, 2 << 12, 14).reshape(2, 1 << 12, 2))
    pn = N.Plan(12, q, psi, batch=2, negacyclic=True)
    assert torch.equal(pn.inverse_bitrev(pn.forward_bitrev(a)), a), "bit-reversed round trip"
    c = pn.polymul(a, bb)
    # a * b through the natural-order transforms: INTT(NTT(a) . NTT(b)) (vmul is Z_q)
    ref = pn.inverse(N.vmul(pn.forward(a), pn.forward(bb), q))
    assert torch.equal(c, ref), "polymul paths disagree"
    # BLAS, ragged length
    n = 5003
    u = dev(synth.uniform_residues(q, n, 15))
    v = dev(synth.uniform_residues(q, n, 16))
    s = N.vadd(u, v, q)
    assert torch.equal(N.vsub(s, v, q), u), "add/sub"
    m = N.vmul(u, v, q)
    y = v.clone()
    N.axpy(1, u, y, q)
    assert torch.equal(y, s), "axpy(1)"
    assert m.shape == u.shape
    # 256-bit passes
    e4 = P["w256"]["b256"]
    q4 = h(e4["q"])
    w4 = pow(h(e4["omega"]), 1 << (e4["logn"] - 10), q4)
    x4 = torch.from_numpy(synth.uniform_residues_w(q4, 2 << 10, 17).reshape(2, 1 << 10, 4).view(np.int64)).cuda()
    p4 = N.Plan256(10, q4, w4, batch=2)
    assert torch.equal(p4.inverse(p4.forward(x4)), x4), "256-bit round trip"
    # 192-bit moduli (6-word kernels): round trip, and vec256_mul against Python integers
    e6 = P["w256"]["b192"]
    q6 = h(e6["q"])
    w6 = pow(h(e6["omega"]), 1 << (e6["logn"] - 12), q6)
    x6 = torch.from_numpy(synth.uniform_residues_w(q6, 2 << 12, 18).reshape(2, 1 << 12, 4).view(np.int64)).cuda()
    p6 = N.Plan256(12, q6, w6, batch=2)
    assert torch.equal(p6.inverse(p6.forward(x6)), x6), "192-bit round trip"
    a6 = synth.uniform_residues_w(q6, 64, 19)
    b6 = synth.uniform_residues_w(q6, 64, 20)
    z6 = N.vmul256(torch.from_numpy(a6.view(np.int64)).cuda(), torch.from_numpy(b6.view(np.int64)).cuda(), q6)
    ints = lambda arr: [sum(int(r[k]) << (64 * k) for k in range(4)) for r in arr]  # noqa: E731
    assert ints(z6.cpu().numpy().view(np.uint64)) == [u * v % q6 for u, v in zip(ints(a6), ints(b6))], "vec256_mul (192-bit)"
    # four-step in the natural block layout at one rank == the three-pass plan, bit for bit
    from paper_2509_12494_b200 import fourstep as FS
    e5 = P["cfg5"]
    q5 = h(e5["q"])
    w5 = pow(h(e5["omega"]), 1 << (26 - 14), q5)
    x5 = dev(synth.uniform_residues(q5, 1 << 14, 21))
    fs = FS.FourStep(14, q5, w5, layout="natural")
    y5 = fs.forward(x5)
    assert torch.equal(y5, N.Plan(14, q5, w5).forward(x5.reshape(1, -1, 2)).reshape(-1, 2)), "four-step vs plan"
    assert torch.equal(fs.inverse(y5), x5), "four-step natural round trip"
    torch.cuda.synchronize()
    print("sanitize driver: all checks passed; library launches", N.launch_count())


if __name__ == "__main__":
    main()

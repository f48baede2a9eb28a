"""The seeded generator module shared by both sides: splitmix64 reference values,
vectorised == sequential rejection sampling, range."""
import numpy as np

import synth


def test_splitmix64_reference():
    # splitmix64 seeded with 0: first outputs of the reference generator (Vigna)
    assert [int(v) for v in synth.splitmix64(0, 0, 3)] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    assert synth.splitmix64_scalar(0, 0) == 0xE220A8397B1DCDAF


def test_uniform_matches_sequential():
    for q in (17, 65537, (1 << 100) + 3, (1 << 127) + 1, (1 << 128) - 8257535, (3 << 126) + 1):
        seed = synth.stream_seed(7, 0, q & 0xFFFF)
        v = synth.to_ints(synth.uniform_residues(q, 40, seed))
        assert v == [synth.uniform_residue_scalar(q, seed, k) for k in range(40)]
        assert all(0 <= x < q for x in v)


def test_uniform_range_large():
    q = (1 << 127) + 1   # acceptance ~1/2: exercises the retry path
    a = synth.uniform_residues(q, 100000, 5)
    v = synth.to_ints(a[:1000])
    assert all(0 <= x < q for x in v)
    assert int(a[:, 1].max()) <= (q >> 64)

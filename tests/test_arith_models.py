"""Host checks of the wide-modulus kernel arithmetic (no GPU): the committed
arith256_gen.cuh is exactly what tools/gen_arith256.py writes, and the word-level model of
its Montgomery carry chains (tools/model/mont_eo_model_w.py) accounts for every dropped
carry, for the canonical products (a < R, b < q: T < 2q) and the lazy class of the
8- and 6-word kernels (q < R/4, a < 4q: word W of T is zero, Harvey butterflies stay in
[0, 4q)).  Development models of the kernels, not the oracle."""
import importlib.util
import os
import random

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _load(rel, name):
    spec = importlib.util.spec_from_file_location(name, os.path.join(ROOT, rel))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_generated_header_is_current(tmp_path):
    gen = _load("tools/gen_arith256.py", "gen_arith256")
    committed = open(gen.OUT).read()
    gen.OUT = str(tmp_path / "arith256_gen.cuh")
    gen.main()
    assert open(gen.OUT).read() == committed


@pytest.mark.parametrize("W", [6, 8])
def test_mont_model_canonical_and_lazy(W):
    m = _load("tools/model/mont_eo_model_w.py", "mont_eo_model_w")
    bits = 32 * W
    rng = random.Random(100 + W)
    for q in [(1 << bits) - 189, (1 << (bits - 1)) + 1, rng.randrange(1 << (bits - 1), 1 << bits) | 1]:
        for _ in range(300):
            m.check(W, q, rng.randrange(1 << bits), rng.randrange(q))
    for q in [(1 << (bits - 2)) - 57 | 1, rng.randrange(1 << (bits - 3), 1 << (bits - 2)) | 1, 65537]:
        m.check_lazy(W, q, rng, 300)


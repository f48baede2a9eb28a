import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs through the C-ABI library")
    config.addinivalue_line("markers", "slow: long CPU oracle runs")


@pytest.fixture(scope="session")
def params():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "params.json")) as f:
        P = json.load(f)

    def conv(d):
        if isinstance(d, dict):
            return {k: conv(v) for k, v in d.items()}
        if isinstance(d, list):
            return [conv(v) for v in d]
        if isinstance(d, str) and d.startswith("0x"):
            return int(d, 16)
        return d
    return conv(P)

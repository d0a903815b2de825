import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running (exhaustive FP32 etc.)")


def read_golden(name):
    """Non-comment lines of tests/golden/<name>, split on whitespace."""
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


@pytest.fixture(scope="session")
def golden_table1():
    """Table 1 from tests/golden/table1.txt -> (E, r, b) lists by index t."""
    E = [None] * 32; r = [None] * 32; b = [None] * 32
    for t, e, rr, bb in read_golden("table1.txt"):
        i = int(t, 2)
        E[i], r[i], b[i] = int(e), int(rr), int(bb)
    assert None not in E
    return E, r, b

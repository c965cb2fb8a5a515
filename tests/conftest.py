import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA device); run with -m gpu")
    config.addinivalue_line("markers", "slow: takes more than ~20 s on the CPU")


def golden_table1():
    """PAPER.md Table 1 as {(k, p): (size, opc, iters)}; None where the paper has †."""
    out = {}
    with open(os.path.join(ROOT, "tests", "golden", "table1_cube.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            k, p, size, opc, it = line.split()
            out[(int(k), int(p))] = None if size == "-" else (int(size), float(opc), int(it))
    return out


@pytest.fixture(scope="session")
def table1():
    return golden_table1()

"""Shared fixtures. `-m "not gpu"` runs on CPU (oracle vs reference/goldens, host
logic, C-ABI load/exports); `-m gpu` runs the CUDA engine against the oracle."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the oracle restatement (and libhddm.so if missing) once."""
    import subprocess
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    if not os.path.exists(os.path.join(ROOT, "paper_1807_04180_b200", "libhddm.so")):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "paper_1807_04180_b200")],
                       check=True)


def rel_l2(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def golden(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))


def golden_cases():
    """The golden cases with their Problem (tests/golden/make_golden.py)."""
    sys.path.insert(0, GOLDEN)
    import make_golden
    return list(make_golden.cases())

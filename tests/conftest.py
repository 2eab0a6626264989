import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(os.path.join(ROOT, "tests", "golden", "golden.npz")))


@pytest.fixture(scope="session")
def reflib():
    from oracle import ref_lib
    if not ref_lib.available():
        pytest.skip("oracle/_ref not built (make -C oracle)")
    return ref_lib.RefLib()


@pytest.fixture(scope="session")
def ctx():
    from paper_1507_01239_b200 import parnn as P
    return P.Context(0)


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))

"""Shared fixtures.  `-m gpu` tests need a B200 and libh2ldl.so; the rest run on CPU.

The oracle (oracle/) is imported here and in the tests only, as the checker.
"""

import glob
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
import pin_host_fp  # noqa: E402,F401  (before numpy: payloads rebuilt here round like the reference's)
import numpy as np  # noqa: E402
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100) device and libh2ldl.so")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def instance_names():
    return sorted(os.path.basename(p)[2:-4] for p in glob.glob(os.path.join(GOLDEN, "h_*.npz")))


@pytest.fixture(scope="session")
def rng():
    return np.random.default_rng(20240817)

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: longer CPU tests")


@pytest.fixture(scope="session")
def orc():
    from oracle import load_oracle

    return load_oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle import load_ref, ref_available

    if not ref_available():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return load_ref()


@pytest.fixture(scope="session")
def golden():
    path = os.path.join(ROOT, "tests", "golden", "golden_v1.npz")
    return np.load(path, allow_pickle=False)


@pytest.fixture(scope="session")
def eng():
    """The product package on a CUDA device (GPU tests only)."""
    import paper_2303_09855_b200 as ads

    if ads.device_count() < 1:
        pytest.fail("no CUDA device visible: the -m gpu tests need a B200")
    return ads


def pytest_sessionstart(session):
    """Build the in-tree libraries if absent (the driver's build() normally has)."""
    import subprocess

    so = os.path.join(ROOT, "paper_2303_09855_b200", "libadsann_b200.so")
    if not os.path.exists(so):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2303_09855_b200", "csrc"), "-j8"],
                       check=True, capture_output=True)
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "restate"], check=True,
                       capture_output=True)

"""Shared fixtures.  `-m gpu` tests need a B200; everything else runs on CPU."""
from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(GOLDEN, "golden.npz"))


@pytest.fixture(scope="session")
def port():
    from oracle import PORT_PATH, Port
    if not os.path.exists(PORT_PATH):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True,
                       capture_output=True)
    return Port()


@pytest.fixture(scope="session")
def small(golden):
    from oracle import CorpusArrays
    return CorpusArrays(golden["small_offsets"], golden["small_words"], golden["small_counts"],
                        int(golden["small_phi"].shape[1]), golden["small_phi_true"])


@pytest.fixture(scope="session")
def small_split(port, small):
    """split_holdout(small, 0.2, 9) -- pinned against the reference in test_oracle."""
    return port.split_holdout(small, 0.2, 9)


@pytest.fixture(scope="session")
def cuda_ctx():
    from paper_1409_5402_b200 import samelda
    return samelda.Context(0)

"""Shared fixtures. `-m gpu` tests need a B200 and the built sm_100a library;
everything else runs on the CPU (oracle, host logic, library symbol table)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_PATH = os.path.join(ROOT, "tests", "golden", "reference_golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the native library")
    config.addinivalue_line("markers", "slow: long-running (large q) checks")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN_PATH, allow_pickle=False) as z:
        data = {k: z[k] for k in z.files}
    return data


@pytest.fixture
def rng():
    # the reference's fixture seed (tests/conftest.py:72-74)
    return np.random.default_rng(20240817)


def golden_cases(prefix=""):
    with np.load(GOLDEN_PATH, allow_pickle=False) as z:
        return [str(c) for c in z["cases"] if str(c).startswith(prefix)]


def golden_tables():
    with np.load(GOLDEN_PATH, allow_pickle=False) as z:
        return [str(c) for c in z["tables"]]

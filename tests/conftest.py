import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer CPU test")


def rel_err_per_state(x, ref, floor=0.0):
    """Parity metric (A13): per state max_i |x - ref| / max_i |ref|.

    x, ref are [n, B] (link-major) or [n]; returns the per-state array.
    `floor` guards states whose reference is (near) zero.
    """
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if ref.ndim == 1:
        x, ref = x[:, None], ref[:, None]
    den = np.maximum(np.abs(ref).max(axis=0), floor)
    return np.abs(x - ref).max(axis=0) / den


@pytest.fixture(scope="session")
def rng():
    return np.random.default_rng(1609_04493)

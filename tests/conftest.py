import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C ABI)")
    config.addinivalue_line("markers", "slow: larger parity cases")


@pytest.fixture(scope="session")
def gkb():
    import paper_1808_03374_b200 as P
    return P


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle


def rel_err(a, b):
    """Max-norm relative error of a vector (normalised by max|b|): for
    matvec outputs and bases; singular values use sigma_rel_err."""
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(1e-300, np.max(np.abs(b))))


def sigma_rel_err(a, b):
    """Largest per-value relative error max_i |a_i - b_i| / |b_i| (BASELINE:
    "top-k singular values within 1e-9 relative" -- every sigma, not
    normalised by sigma_1)."""
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape, (a.shape, b.shape)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def principal_angles(A, B):
    """Largest principal angle between span(A) and span(B) (QR first: the
    reference returns un-renormalized Ritz vectors, gkl.cpp:500-505)."""
    qa = np.linalg.qr(A)[0]
    qb = np.linalg.qr(B)[0]
    s = np.linalg.svd(qa.T @ qb, compute_uv=False)
    return float(np.max(np.arccos(np.clip(s, 0.0, 1.0))))

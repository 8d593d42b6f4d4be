import math
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line(
        "markers", "gpu: needs a B200 (CUDA device); parity through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session", autouse=True)
def built():
    """Build the native artefacts once (no-op when up to date)."""
    import __graft_entry__
    __graft_entry__.build()


def golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def f_rms(f):
    f = np.asarray(f)
    return math.sqrt(float((f * f).sum()) / f.shape[0])


def rel(a, b):
    return abs(a - b) / abs(b) if b != 0 else abs(a - b)


def random_neutral(n, L, seed, min_sep=0.8):
    """Rejection-sampled neutral system with +-q charge pairs."""
    rng = np.random.default_rng(seed)
    pos = np.empty((n, 3))
    k = 0
    while k < n:
        c = rng.random(3) * L
        d = pos[:k] - c
        d -= L * np.floor(d / L + 0.5)
        if k and (d * d).sum(axis=1).min() < min_sep**2:
            continue
        pos[k] = c
        k += 1
    mag = rng.random(n // 2) + 0.5
    return pos, np.concatenate([mag, -mag])

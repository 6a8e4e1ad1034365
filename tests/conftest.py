import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libskm_b200.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


def make_blobs(n, d, n_centers, seed, spread=5.0, noise=1.0):
    """Same RNG call sequence as the reference's test generator (pkg/tests/conftest.py:7-13)
    so seeded inputs are identical to the ones the reference's own tests use."""
    rng = np.random.default_rng(seed)
    centers = (rng.standard_normal((n_centers, d)) * spread).astype(np.float32)
    which = rng.integers(0, n_centers, n)
    noise_part = (rng.standard_normal((n, d)) * noise).astype(np.float32)
    return np.ascontiguousarray(centers[which] + noise_part, dtype=np.float32)


def make_skewed_blobs(n, d, n_centers, seed, spread=1.5, noise=1.0, decay=0.995):
    """Per-dimension variance decaying geometrically (pkg/tests/conftest.py:16-20)."""
    x = make_blobs(n, d, n_centers, seed, spread=spread, noise=noise)
    return np.ascontiguousarray(x * (decay ** np.arange(d)).astype(np.float32), dtype=np.float32)


def have_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def pytest_collection_modifyitems(config, items):
    if have_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)

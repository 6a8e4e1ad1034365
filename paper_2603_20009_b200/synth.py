"""Synthetic inputs of the BASELINE configs, bit-identical to the reference's own test generators
(pkg/tests/conftest.py:7-20: ``make_blobs`` / ``make_skewed_blobs``), produced in row chunks.

The reference draws the whole (n, d) f64 noise matrix at once (12 GB at c2, 82 GB at c5); the
PCG64 normal stream is sequential, so drawing it chunk by chunk after the same centre and label
draws yields the same values with a bounded working set.  Used by bench.py and the
full-size parity tests so the timed trajectory is the one checked against the reference."""

from __future__ import annotations

import numpy as np


def make_blobs(n: int, d: int, n_centers: int, seed, spread: float = 5.0, noise: float = 1.0,
               decay: float | None = None, chunk_rows: int = 1 << 16, out: np.ndarray | None = None) -> np.ndarray:
    rng = np.random.default_rng(seed)
    centers = (rng.standard_normal((n_centers, d)) * spread).astype(np.float32)
    which = rng.integers(0, n_centers, n)
    x = np.empty((n, d), dtype=np.float32) if out is None else out
    scale = (decay ** np.arange(d)).astype(np.float32) if decay is not None else None
    for r0 in range(0, n, chunk_rows):
        m = min(chunk_rows, n - r0)
        part = (rng.standard_normal((m, d)) * noise).astype(np.float32)
        np.add(centers[which[r0:r0 + m]], part, out=x[r0:r0 + m])
        if scale is not None:
            np.multiply(x[r0:r0 + m], scale, out=x[r0:r0 + m])
    return x


def make_skewed_blobs(n: int, d: int, n_centers: int, seed, spread: float = 1.5, noise: float = 1.0,
                      decay: float = 0.995, **kw) -> np.ndarray:
    return make_blobs(n, d, n_centers, seed, spread=spread, noise=noise, decay=decay, **kw)

"""Synthetic inputs of the BASELINE configs, bit-identical to the reference's own test generators
(pkg/tests/conftest.py:7-20: ``make_blobs`` / ``make_skewed_blobs``), produced in row chunks.

The reference draws the whole (n, d) f64 noise matrix at once (12 GB at c2, 82 GB at c5); the
PCG64 normal stream is sequential, so drawing it chunk by chunk after the same centre and label
draws yields the same values with a bounded working set.  Used by bench.py and the
full-size parity tests so the timed trajectory is the one checked against the reference."""

from __future__ import annotations

import numpy as np


def make_blobs(n: int, d: int, n_centers: int, seed, spread: float = 5.0, noise: float = 1.0,
               decay: float | None = None, chunk_rows: int = 1 << 16, out: np.ndarray | None = None,
               out_rows: int | None = None) -> np.ndarray:
    """``out_rows``: generate only rows [0, out_rows) of the n-row matrix (the same values; a
    shard [lo, hi) of a multi-GPU run needs rows < hi)."""
    rng = np.random.default_rng(seed)
    centers = (rng.standard_normal((n_centers, d)) * spread).astype(np.float32)
    which = rng.integers(0, n_centers, n)
    m_out = n if out_rows is None else min(n, out_rows)
    x = np.empty((m_out, d), dtype=np.float32) if out is None else out
    scale = (decay ** np.arange(d)).astype(np.float32) if decay is not None else None
    for r0 in range(0, m_out, chunk_rows):
        m = min(chunk_rows, m_out - r0)
        part = (rng.standard_normal((m, d)) * noise).astype(np.float32)
        np.add(centers[which[r0:r0 + m]], part, out=x[r0:r0 + m])
        if scale is not None:
            np.multiply(x[r0:r0 + m], scale, out=x[r0:r0 + m])
    return x


def make_skewed_blobs(n: int, d: int, n_centers: int, seed, spread: float = 1.5, noise: float = 1.0,
                      decay: float = 0.995, **kw) -> np.ndarray:
    return make_blobs(n, d, n_centers, seed, spread=spread, noise=noise, decay=decay, **kw)


def make_shard_device(n, d, centers, lo, hi, seed, dev):
    """Skewed-blob rows [lo, hi) generated on the GPU: the distribution of make_skewed_blobs
    (centres ~ N(0, 1.5^2), unit noise, per-dim scale 0.995^t) but NOT its values -- for scale
    runs (10M rows) where the host generator would take minutes; parity runs use the generators
    above."""
    import torch
    from .device import padded_ld
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    cen = torch.randn((centers, d), generator=g, device=dev) * 1.5
    scale = (0.995 ** torch.arange(d, device=dev, dtype=torch.float64)).to(torch.float32)
    ld = padded_ld(d)
    x = torch.zeros((hi - lo, ld), dtype=torch.float32, device=dev)
    chunk = 1 << 16
    for s in range(lo, hi, chunk):
        e = min(hi, s + chunk)
        gg = torch.Generator(device=dev)
        gg.manual_seed(seed * 1_000_003 + s)
        which = torch.randint(0, centers, (e - s,), generator=gg, device=dev)
        x[s - lo:e - lo, :d] = (cen[which] + torch.randn((e - s, d), generator=gg, device=dev)) * scale
    return x

"""ORACLE -- test infrastructure only.  Never imported by the product package.

NumPy restatement of the reference's four hot kernels with their exact float semantics:

* scan_bank       follows pkg/src/superkmeans/_kernels.pyx:14-82 (sequential-tau ADSampling
                  scan; per-block sums are fresh sequential fp32 chains, no FMA).
* seed_thresholds follows _kernels.pyx:85-103.
* accumulate_centroid_sums follows _kernels.pyx:106-119 (serial row-order f64 sums).
* portable_matmul follows _kernels.pyx:122-142 (sequential fp32 dot per cell).

Vectorisation is over vectors for one centroid at a time, which preserves the
per-vector order of tau updates (tau only changes between centroids).  Sequential fp32
chains use ``np.cumsum(..., dtype=float32)``, which accumulates left to right.
"""

from __future__ import annotations

import numpy as np

INF32 = np.float32(np.inf)


def _seq_sum_sq(diff: np.ndarray) -> np.ndarray:
    """Row-wise sequential fp32 sum of squares (ascending column order)."""
    if diff.shape[1] == 0:
        return np.zeros(diff.shape[0], np.float32)
    sq = (diff * diff).astype(np.float32, copy=False)
    return np.cumsum(sq, axis=1, dtype=np.float32)[:, -1]


def seed_thresholds(x, centroids, assign, out, n_threads=1, chunk=2048):
    for s in range(0, x.shape[0], chunk):
        e = min(x.shape[0], s + chunk)
        out[s:e] = _seq_sum_sq(x[s:e] - centroids[assign[s:e]])


def scan_bank(partial_dists, x, tail, block_offsets, block_dims, theta_factors, d_prime, bank_offset, tau,
              assign, sentinel, n_threads=1):
    """Returns (survivors, dims_touched); updates tau/assign in place."""
    n, kb = partial_dists.shape
    nb = len(block_dims)
    theta = np.asarray(theta_factors, np.float32)
    surv = 0
    touched = 0
    for j in range(kb):
        gate0 = np.full(n, INF32) if sentinel else (tau * theta[0]).astype(np.float32)
        alive = np.flatnonzero(~(partial_dists[:, j] > gate0))
        surv += alive.size
        if alive.size == 0:
            continue
        run = partial_dists[alive, j].astype(np.float32, copy=True)
        pos = d_prime
        for b in range(nb):
            bd = int(block_dims[b])
            off = int(block_offsets[b])
            col = tail[off: off + bd * kb].reshape(bd, kb)[:, j]
            run = (run + _seq_sum_sq(x[alive, pos: pos + bd] - col[None, :])).astype(np.float32)
            touched += alive.size * bd
            pos += bd
            if sentinel and b < nb - 1:
                continue
            keep = ~(run > (tau[alive] * theta[b + 1]).astype(np.float32))
            alive, run = alive[keep], run[keep]
            if alive.size == 0:
                break
        if alive.size == 0:
            continue
        gid = bank_offset + j
        cur = tau[alive]
        better = run < cur
        tie = (run == cur) & (gid < assign[alive])
        assign[alive[better | tie]] = gid
        tau[alive[better]] = run[better]
    return surv, touched


def accumulate_centroid_sums(x, assign, sums, counts):
    # np.add.at applies updates in index order -> serial row-order f64 accumulation
    np.add.at(sums, assign, x.astype(np.float64))
    counts += np.bincount(assign, minlength=counts.shape[0]).astype(np.int64)


def portable_matmul(a, b, dims, out, n_threads=1):
    acc = np.zeros((a.shape[0], b.shape[0]), np.float32)
    for t in range(dims):
        acc = (acc + np.multiply.outer(a[:, t], b[:, t]).astype(np.float32)).astype(np.float32)
    out[:] = acc

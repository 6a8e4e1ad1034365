"""Host-side scalar logic of the loop: everything that is RNG-, LAPACK- or control-flow-bound
and must stay bit-identical to the reference.  No per-vector work happens here.

* rotation: PCG64 normal draw + LAPACK QR + sign fix (preprocess.py:22-34).  Kept on the
  host on purpose: it is part of the persisted-model contract (a model stores only the seed)
  and the device receives R once.
* sampling / Forgy init index draws (preprocess.py:55-92).
* ADSampling gate factors (pruning.py:35-56), prune rate (pruning.py:144-147),
  cutoff controller (core.py:131-154), empty-cluster donor draws (core.py:103-128),
  ETR stop rule (evaluation.py:116-139).
"""

from __future__ import annotations

import numpy as np

from .config import (
    D_PRIME_ALIGN,
    D_PRIME_MIN,
    PDX_BLOCK,
    DimensionMismatch,
    EmptySample,
    KMeansConfig,
    KTooLarge,
    RotationMatrix,
)

SPLIT_EPS = np.float32(1.0 / 1024.0)


QR_BLAS_THREADS = 4


def blas_threads(n: int = QR_BLAS_THREADS):
    """Context pinning the BLAS pool to ``n`` threads.  OpenBLAS's blocked QR rounds differently
    at some thread counts (measured with threadpoolctl: 1, 2 and 4 threads give identical Q for
    d = 1024..3072 whatever OPENBLAS_NUM_THREADS says, 8 does not; via the environment variable
    3, 5-7 and 16 differ too), so the rotation is computed at one fixed count on every machine --
    and a pool smaller than the core count leaves cores to the concurrent H2D copy threads
    instead of oversubscribing them (the QR took 0.67 s instead of 0.18 s with 16 spinning
    BLAS threads beside the copy)."""
    try:
        from threadpoolctl import threadpool_limits
    except ImportError:  # pragma: no cover
        import contextlib
        return contextlib.nullcontext()
    return threadpool_limits(n, user_api="blas")


def generate_rotation(dim: int, seed: int) -> RotationMatrix:
    """Haar-random orthogonal matrix: QR of a PCG64 Gaussian, columns sign-fixed by diag(R)."""
    if dim < 1:
        raise DimensionMismatch("rotation dimension must be >= 1")
    g = np.random.default_rng(seed).standard_normal((dim, dim))
    with blas_threads():
        q, r = np.linalg.qr(g)
    s = np.sign(np.diag(r))
    s[s == 0] = 1.0
    return RotationMatrix(data=(q * s[None, :]).astype(np.float32), dim=dim, seed=seed)


def sample_indices(n: int, fraction: float, seed, k: int | None = None) -> np.ndarray | None:
    """Sorted sample of ceil(fraction*n) rows (None when fraction == 1)."""
    if not 0 < fraction <= 1:
        raise ValueError("sampling fraction must be in (0, 1]")
    if fraction == 1.0:
        if k is not None and n < k:
            raise EmptySample(f"{n} vectors cannot seed {k} clusters")
        return None
    m = int(np.ceil(fraction * n))
    if k is not None and m < k:
        raise EmptySample(f"sample of {m} vectors cannot seed {k} clusters")
    idx = np.random.default_rng(seed).choice(n, size=m, replace=False)
    idx.sort()
    return idx


def init_indices(n: int, k: int, seed) -> np.ndarray:
    """Forgy init: k distinct rows drawn uniformly."""
    if k > n:
        raise KTooLarge(f"k={k} exceeds {n} available vectors")
    return np.random.default_rng(seed).choice(n, size=k, replace=False)


def adsampling_threshold(m: int, tau: float, d: int, epsilon0: float) -> float:
    if not 1 <= m <= d:
        raise ValueError(f"m={m} out of range [1, {d}]")
    if m == d:
        return tau
    g = 1.0 + epsilon0 / np.sqrt(m)
    return tau * (m / d) * g * g


def threshold_factors(d: int, d_prime: int, block_bounds, epsilon0: float) -> np.ndarray:
    """Checkpoint multipliers (m/d)(1+eps0/sqrt(m))^2 at m = d' and each block end; 1.0 at m = d."""
    m = np.concatenate(([d_prime], np.asarray(block_bounds, dtype=np.int64)))
    g = 1.0 + epsilon0 / np.sqrt(m.astype(np.float64))
    f = (m / d) * g * g
    f[m == d] = 1.0
    return f.astype(np.float32)


def sentinel_factors(factors: np.ndarray) -> np.ndarray:
    """Test-only exhaustive scan: +inf gates everywhere except the exact final comparison."""
    f = np.full_like(factors, np.inf)
    f[-1] = factors[-1]
    return f


def prune_rate_from_totals(survivors_total: int, n_vectors: int, k_total: int) -> float:
    if n_vectors == 0:
        raise ValueError("no vectors processed")
    return 1.0 - survivors_total / (n_vectors * k_total)


def adjust_d_prime(current: int, prune_rate: float, cfg: KMeansConfig, dim: int) -> int:
    """Shrink d' by the adjust factor above the target band, grow it below; clamp to
    [16, dim-64] and align to 8 in the direction of the move."""
    lo, hi = D_PRIME_MIN, dim - PDX_BLOCK
    if prune_rate > cfg.prune_target_high:
        new = int(np.floor(current * (1.0 - cfg.d_prime_adjust_factor)))
        up = False
    elif prune_rate < cfg.prune_target_low:
        new = int(np.ceil(current * (1.0 + cfg.d_prime_adjust_factor)))
        up = True
    else:
        return current
    new = min(hi, max(lo, new))
    new = -(-new // D_PRIME_ALIGN) * D_PRIME_ALIGN if up else (new // D_PRIME_ALIGN) * D_PRIME_ALIGN
    return min(hi, max(lo, new))


def plan_splits(counts: np.ndarray, rng: np.random.Generator) -> tuple[list[int], list[int]]:
    """Donor draw for every empty cluster, in ascending empty index, count-proportional with
    the donor's count halved after each split.  Mutates ``counts`` exactly like the
    reference so the RNG stream and final counts match; the row arithmetic runs on device."""
    empties = np.flatnonzero(counts == 0)
    donors: list[int] = []
    k = counts.shape[0]
    for e in empties:
        donor = int(rng.choice(k, p=counts / counts.sum()))
        moved = counts[donor] // 2
        counts[e] = counts[donor] - moved
        counts[donor] = moved
        donors.append(donor)
    return [int(e) for e in empties], donors


def check_convergence(prev: np.ndarray, cur: np.ndarray) -> bool:
    if prev.shape != cur.shape:
        raise ValueError("assignment arrays differ in length")
    return bool(np.array_equal(prev, cur))


def etr_should_stop(history, tolerance: float | None = None, patience: int = 2) -> bool:
    """Stop when, over the last patience+1 recalls, neither the best later value nor any
    single step improved on its predecessor by more than the tolerance."""
    if hasattr(history, "values") and hasattr(history, "tolerance"):
        tolerance = history.tolerance if tolerance is None else tolerance
        patience = history.patience
        history = history.values
    if tolerance is None:
        raise ValueError("tolerance required when history is a plain sequence")
    v = list(history)
    if len(v) < patience + 1:
        return False
    w = v[-(patience + 1):]
    if max(w[1:]) - w[0] > tolerance:
        return False
    return all(b - a <= tolerance for a, b in zip(w[1:], w[2:]))


def sub_seed(seed: int, tag: int) -> int:
    """Per-group seed of the hierarchical fine phase (hierarchical.py:82-83)."""
    return int(np.random.SeedSequence([seed, 5, tag]).generate_state(1)[0])

"""Per-vector pruning API of the reference (pkg/src/superkmeans/pruning.py:26-141) on the device.

``prune_and_assign`` is the reference's per-vector twin of the bank scan; here it runs the device
scan entry (``skm_scan_bank``, bitwise the reference's scan_bank) on the one row, so the
outcome -- survivors, dims touched, final assignment and tau -- is the reference's bit for bit.
``initial_threshold`` is the seed-threshold kernel on one row.  The batched hot path does not use
these; they exist so code written against the reference's pruning module runs unchanged."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .hostmath import adsampling_threshold, prune_rate_from_totals, threshold_factors  # noqa: F401


@dataclass
class PruneOutcome:
    """Result of scanning all banks for one vector (pruning.py:26-32)."""

    survivors_after_gemm: int
    final_assignment: int
    final_sq_dist: float
    dims_touched: int


def _dev_rows(*arrs):
    import torch
    from .device import require_cuda
    dev = require_cuda()
    return [torch.as_tensor(np.ascontiguousarray(a), device=dev) for a in arrs]


def initial_threshold(x: np.ndarray, prev_centroid: np.ndarray) -> float:
    """Exact squared distance to the previous assignment's updated position (pruning.py:59-66):
    the sequential fp32 chain of seed_thresholds, computed by the device kernel."""
    import torch
    from . import device
    xv = np.asarray(x, dtype=np.float32).reshape(1, -1)
    cv = np.asarray(prev_centroid, dtype=np.float32).reshape(1, -1)
    X, Cm = device.to_device_matrix(xv), device.to_device_matrix(cv)
    a = torch.zeros(1, dtype=torch.int32, device=X.device)
    out = torch.empty(1, dtype=torch.float32, device=X.device)
    device.seed_thresholds(X, Cm, a, out, d=xv.shape[1])
    return float(out.item())


def prune_and_assign(x_idx: int, partial_dists, bank, state, cfg, x_row: np.ndarray,
                     bank_offset: int = 0) -> PruneOutcome:
    """Scan one bank for one vector with the reference semantics (pruning.py:69-132): the device
    scan_bank over the single row; updates state.assignment / state.best_sq_dist[x_idx]."""
    import torch
    from . import device
    d, dp = bank.dim, bank.d_prime
    bounds = dp + np.cumsum(bank.block_dims, dtype=np.int64)
    f = threshold_factors(d, dp, bounds, cfg.epsilon0)
    row = np.asarray(partial_dists.values, dtype=np.float32)[x_idx:x_idx + 1, :bank.k_batch]
    X = device.to_device_matrix(np.asarray(x_row, dtype=np.float32).reshape(1, -1))
    pd, tail, offs, dims, theta = _dev_rows(row, bank.tail, bank.block_offsets.astype(np.int64),
                                            bank.block_dims.astype(np.int32), f)
    tau = torch.tensor([float(state.best_sq_dist[x_idx])], dtype=torch.float32, device=X.device)
    assign = torch.tensor([int(state.assignment[x_idx])], dtype=torch.int32, device=X.device)
    sv, td = device.scan_bank(pd, X, tail, offs, dims, theta, dp, bank_offset, tau, assign, cfg.pruning_sentinel)
    state.assignment[x_idx] = int(assign.item())
    state.best_sq_dist[x_idx] = np.float32(tau.item())
    return PruneOutcome(survivors_after_gemm=sv, final_assignment=int(assign.item()),
                        final_sq_dist=float(tau.item()), dims_touched=td)


def measure_prune_rate(outcomes, k_total: int) -> float:
    """Fraction of (vector, centroid) pairs discarded at d_prime (pruning.py:135-141)."""
    outcomes = list(outcomes)
    if not outcomes:
        raise ValueError("no outcomes to measure")
    mean_survivors = sum(o.survivors_after_gemm for o in outcomes) / len(outcomes)
    return 1.0 - mean_survivors / k_total

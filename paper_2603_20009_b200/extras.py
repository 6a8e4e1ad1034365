"""Reference-compatible helper entry points taking/returning host arrays; the per-vector work
runs on the device.  (core.update_centroids core.py:79-100, core.split_empty_clusters
core.py:103-128, preprocess.* preprocess.py:37-112.)"""

from __future__ import annotations

import numpy as np
import torch

from . import native
from .config import DimensionMismatch, NormCache, RotationMatrix
from .device import on_device, ptr, require_cuda, stream_handle
from .hostmath import SPLIT_EPS, init_indices, plan_splits, sample_indices


@on_device
def apply_rotation(x: np.ndarray, rotation: RotationMatrix, device=None) -> np.ndarray:
    """x @ R on the tensor cores (3xTF32)."""
    from .api import DeviceRotation, _h2d
    if x.shape[1] != rotation.dim:
        raise DimensionMismatch(f"vectors have dim {x.shape[1]}, rotation has dim {rotation.dim}")
    dev = require_cuda(device)
    rot = DeviceRotation(rotation, dev)
    return rot.apply(_h2d(np.ascontiguousarray(x, dtype=np.float32), dev))[:, :rotation.dim].cpu().numpy()


@on_device
def unapply_rotation(x: np.ndarray, rotation: RotationMatrix, device=None) -> np.ndarray:
    from .api import DeviceRotation, _h2d
    if x.shape[1] != rotation.dim:
        raise DimensionMismatch(f"vectors have dim {x.shape[1]}, rotation has dim {rotation.dim}")
    dev = require_cuda(device)
    rot = DeviceRotation(rotation, dev)
    return rot.apply(_h2d(np.ascontiguousarray(x, dtype=np.float32), dev), inverse=True)[:, :rotation.dim].cpu().numpy()


def sample_training_set(x: np.ndarray, fraction: float, seed, k: int | None = None):
    idx = sample_indices(x.shape[0], fraction, seed, k=k)
    return (x, None) if idx is None else (x[idx], idx)


def init_centroids(x: np.ndarray, k: int, seed):
    idx = init_indices(x.shape[0], k, seed)
    return x[idx].copy(), idx


def _row_norms_dev(x: np.ndarray, dims: int, dev) -> np.ndarray:
    from .api import _h2d
    X = _h2d(np.ascontiguousarray(x, dtype=np.float32), dev)
    out = torch.empty(max(x.shape[0], 1), dtype=torch.float32, device=dev)
    if x.shape[0]:
        native.call("skm_row_sq_norms", ptr(X), X.shape[1], x.shape[0], dims, ptr(out), stream_handle())
    return out[: x.shape[0]].cpu().numpy()


@on_device
def compute_norms(m: np.ndarray, d_prime: int, device=None) -> NormCache:
    if not 0 < d_prime <= m.shape[1]:
        raise DimensionMismatch(f"d_prime {d_prime} out of range for dim {m.shape[1]}")
    dev = require_cuda(device)
    return NormCache(full_sq=_row_norms_dev(m, m.shape[1], dev), partial_sq=_row_norms_dev(m, d_prime, dev),
                     d_prime=d_prime)


@on_device
def update_centroids(x: np.ndarray, assignments: np.ndarray, k: int, prev_centroids: np.ndarray | None = None,
                     kernel_impl=None, device=None):
    """Per-cluster means with ordered f64 sums on the device; empties keep their previous
    centroid (zero without one).  Returns (centroids f32 (k, d), counts i64)."""
    from .api import _h2d
    dev = require_cuda(device)
    x = np.ascontiguousarray(x, dtype=np.float32)
    n, d = x.shape
    X = _h2d(x, dev)
    A = torch.from_numpy(np.ascontiguousarray(assignments, dtype=np.int32)).to(dev)
    prev = np.zeros((k, d), np.float32) if prev_centroids is None else np.asarray(prev_centroids, np.float32)
    Cd = _h2d(np.ascontiguousarray(prev), dev)
    lib = native.load()
    order = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    counts = torch.empty(k, dtype=torch.int32, device=dev)
    offs = torch.empty(k, dtype=torch.int32, device=dev)
    ws = torch.empty(int(lib.skm_update_workspace_bytes(n, k)), dtype=torch.uint8, device=dev)
    st = stream_handle()
    native.call("skm_cluster_sort", ptr(A), n, k, ptr(order), ptr(counts), ptr(offs), ptr(ws), ws.numel(), st)
    native.call("skm_cluster_sums", ptr(X), X.shape[1], ptr(order), ptr(offs), ptr(counts), k, d, None, 0, ptr(Cd),
                Cd.shape[1], 0, st)
    return Cd[:, :d].cpu().numpy().copy(), counts.cpu().numpy().astype(np.int64)


@on_device
def split_empty_clusters(centroids: np.ndarray, counts: np.ndarray, rng, device=None):
    """In-place split of donors into empty clusters (host RNG, device row arithmetic)."""
    from .api import _h2d
    empties, donors = plan_splits(counts, rng)
    if not empties:
        return centroids, 0
    dev = require_cuda(device)
    k, d = centroids.shape
    Cd = _h2d(np.ascontiguousarray(centroids, dtype=np.float32), dev)
    e = torch.tensor(empties, dtype=torch.int32, device=dev)
    dn = torch.tensor(donors, dtype=torch.int32, device=dev)
    native.call("skm_apply_splits", ptr(Cd), Cd.shape[1], d, ptr(e), ptr(dn), len(empties), float(SPLIT_EPS),
                stream_handle())
    centroids[:] = Cd[:, :d].cpu().numpy()
    return centroids, len(empties)

"""ORACLE -- test/baseline infrastructure only.  ctypes binding of oracle/skm_oracle.c (the
C + OpenMP restatement of the reference's compiled kernels, _kernels.pyx:14-119), with the
same call signatures as oracle/kernels_np.py.  Built by `make -C oracle`."""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build", "libskm_oracle.so")
_lib = None


def available() -> bool:
    global _lib
    if _lib is None and os.path.exists(_LIB):
        _lib = C.CDLL(_LIB)
        p = C.c_void_p
        L = C.c_long
        _lib.oracle_scan_bank.argtypes = [p, L, L, p, L, p, p, p, L, p, L, L, p, p, C.c_int, C.c_int, p]
        _lib.oracle_seed_thresholds.argtypes = [p, L, L, p, p, p, C.c_int]
        _lib.oracle_accumulate_sums.argtypes = [p, L, L, p, p, p]
    return _lib is not None


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def threads() -> int:
    return os.cpu_count() or 1


def seed_thresholds(x, centroids, assign, out, n_threads=None):
    x = np.ascontiguousarray(x, np.float32)
    c = np.ascontiguousarray(centroids, np.float32)
    a = np.ascontiguousarray(assign, np.int32)
    assert out.dtype == np.float32 and out.flags.c_contiguous
    _lib.oracle_seed_thresholds(_p(x), x.shape[0], x.shape[1], _p(c), _p(a), _p(out), n_threads or threads())


def scan_bank(partial_dists, x, tail, block_offsets, block_dims, theta_factors, d_prime, bank_offset, tau, assign,
              sentinel, n_threads=None):
    pd = np.ascontiguousarray(partial_dists, np.float32)
    x = np.ascontiguousarray(x, np.float32)
    tail = np.ascontiguousarray(tail, np.float32)
    bo = np.ascontiguousarray(block_offsets, np.int64)
    bd = np.ascontiguousarray(block_dims, np.int32)
    th = np.ascontiguousarray(theta_factors, np.float32)
    assert tau.dtype == np.float32 and assign.dtype == np.int32 and tau.flags.c_contiguous and assign.flags.c_contiguous
    cnt = np.zeros(2, np.int64)
    _lib.oracle_scan_bank(_p(pd), pd.shape[0], pd.shape[1], _p(x), x.shape[1], _p(tail), _p(bo), _p(bd), bd.shape[0],
                          _p(th), int(d_prime), int(bank_offset), _p(tau), _p(assign), int(bool(sentinel)),
                          n_threads or threads(), _p(cnt))
    return int(cnt[0]), int(cnt[1])


def accumulate_centroid_sums(x, assign, sums, counts):
    x = np.ascontiguousarray(x, np.float32)
    a = np.ascontiguousarray(assign, np.int32)
    assert sums.dtype == np.float64 and counts.dtype == np.int64
    _lib.oracle_accumulate_sums(_p(x), x.shape[0], x.shape[1], _p(a), _p(sums), _p(counts))

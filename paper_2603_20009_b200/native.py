"""ctypes binding of libskm_b200.so (the C ABI in include/skm_b200.h).

The library is built in-tree by ``paper_2603_20009_b200.build`` (nvcc, sm_100a).  There is no
fallback: if the shared object is missing or fails to load, every entry point raises
``NativeUnavailable`` so a GPU run can never silently take a CPU path.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SKM_LIB", os.path.join(_HERE, "libskm_b200.so"))


class NativeUnavailable(RuntimeError):
    pass


class NativeError(RuntimeError):
    pass


_vp = C.c_void_p
_i = C.c_int
_ll = C.c_longlong
_f = C.c_float


class GemmParams(C.Structure):
    _fields_ = [
        ("a_hi", _vp), ("a_lo", _vp), ("lda", _ll),
        ("b_hi", _vp), ("b_lo", _vp), ("ldb", _ll),
        ("M", _i), ("N", _i), ("K", _i),
        ("mode", _i), ("n_split", _i),
        ("out", _vp), ("ldo", _ll),
        ("xsq", _vp), ("ysq", _vp),
        ("top", _vp),
        ("thr", _vp),
        ("cand", _vp), ("cand_cnt", _vp), ("cand_cap", _i),
        ("row_offset", _ll),
        ("ext_k", _i), ("xsq_ext", _vp), ("ysq_ext", _vp), ("thr1", _vp), ("cert_eps", _f),
        ("row_crange", _vp), ("tile_nrange", _vp),
        ("ext_hi_only", _i),
    ]


class ChainParams(C.Structure):
    _fields_ = [
        ("a", _vp), ("lda", _ll),
        ("b", _vp), ("ldb", _ll),
        ("M", _i), ("N", _i), ("K", _i),
        ("flavour", _i), ("q", _i), ("mode", _i),
        ("out", _vp), ("ldo", _ll),
        ("xsq", _vp), ("ysq", _vp),
        ("b_kmajor", _i),
    ]


class ScanParams(C.Structure):
    _fields_ = [
        ("cand", _vp), ("cand_cnt", _vp), ("cap", _i),
        ("dense", _vp), ("ld_dense", _ll), ("dense_row", _vp), ("k", _i),
        ("rows", _vp), ("n_rows", _i), ("row0", _ll),
        ("row_map", _vp), ("work", _vp),
        ("x", _vp), ("ldx", _ll),
        ("tails", _vp), ("nb", _i), ("d_prime", _i),
        ("theta", _vp), ("block_dims", _vp),
        ("tau", _vp), ("assign", _vp),
        ("counters", _vp),
        ("dense_mode", _i),
        ("counters_ext", _vp),
        ("prune_hist", _vp),
        ("kap", _f), ("xsq", _vp), ("ysq", _vp), ("ysq_max", _vp),
        ("cent", _vp), ("ldc", _ll), ("chain_flavour", _i), ("chain_q", _i),
        ("row_group", _vp), ("group_counters", _vp),
        ("flat", _i), ("fb_rows", _vp), ("fb_count", _vp),
        ("skip_cert", _vp), ("imp", _vp), ("imp_cnt", _vp),
    ]


GEMM_STORE, GEMM_DIST, GEMM_ARGMIN, GEMM_GATE = 0, 1, 2, 3

_SIGS = {
    "skm_kernel_launches": ([], _ll),
    "skm_last_error": ([], C.c_char_p),
    "skm_abi_version": ([], _i),
    "skm_split_hilo": ([_vp, _ll, _i, _i, _vp, _vp, _ll, _vp], _i),
    "skm_row_sq_norms": ([_vp, _ll, _i, _i, _vp, _vp], _i),
    "skm_gather_rows": ([_vp, _ll, _vp, _i, _i, _vp, _ll, _vp], _i),
    "skm_gather_rows_i32": ([_vp, _ll, _vp, _i, _i, _vp, _ll, _vp], _i),
    "skm_fill_f32": ([_vp, _ll, _f, _vp], _i),
    "skm_copy_i32": ([_vp, _vp, _i, _vp], _i),
    "skm_seed_thresholds": ([_vp, _ll, _vp, _ll, _vp, _i, _i, _vp, _vp], _i),
    "skm_scan_bank": ([_vp, _i, _i, _vp, _ll, _vp, _vp, _vp, _i, _vp, _i, _i, _vp, _vp, _i, _vp, _vp], _i),
    "skm_update_workspace_bytes": ([_i, _i], _ll),
    "skm_accumulate_centroid_sums": ([_vp, _ll, _vp, _i, _i, _i, _vp, _vp, _vp, _ll, _vp], _i),
    "skm_portable_matmul": ([_vp, _ll, _vp, _ll, _i, _i, _i, _vp, _ll, _vp], _i),
    "skm_gemm_tf32x3": ([C.POINTER(GemmParams), _vp], _i),
    "skm_argmin_merge": ([_vp, _i, _i, _vp, _vp, _f, _vp, _vp, _vp, _vp, _vp], _i),
    "skm_dense_argmin": ([_vp, _ll, _i, _i, _vp, _vp, _vp, _vp], _i),
    "skm_exact_pair_dist": ([_vp, _ll, _vp, _ll, _vp, _i, _i, _vp, _vp, _i, _i, _vp, _vp], _i),
    "skm_max_f32": ([_vp, _i, _vp, _vp], _i),
    "skm_tau_chunk_sums": ([_vp, _ll, _vp, _vp], _i),
    "skm_argmin_candidates": ([_vp, _i, _vp, _vp, _vp, _f, _vp, _vp, _vp], _i),
    "skm_cand_exact_argmin": ([_vp, _i, _vp, _vp, _i, _vp, _ll, _vp, _ll, _i, _vp, _vp, _i, _i, _vp, _vp, _vp], _i),
    "skm_chain_gemm": ([C.POINTER(ChainParams), _vp], _i),
    "skm_chain_topk_tiles": ([_vp, _ll, _vp, _ll, _i, _i, _i, _i, _i, _vp, _vp, _i, _vp, _vp, _i, _vp], _i),
    "skm_cluster_sort": ([_vp, _i, _i, _vp, _vp, _vp, _vp, _ll, _vp], _i),
    "skm_cluster_sums": ([_vp, _ll, _vp, _vp, _vp, _i, _i, _vp, _i, _vp, _ll, _i, _vp], _i),
    "skm_finalize_centroids": ([_vp, _vp, _i, _i, _vp, _ll, _vp], _i),
    "skm_counts_to_i64": ([_vp, _vp, _i, _i, _vp], _i),
    "skm_apply_splits": ([_vp, _ll, _i, _vp, _vp, _i, _f, _vp], _i),
    "skm_stats_workspace_bytes": ([_i], _ll),
    "skm_assign_stats": ([_vp, _vp, _vp, _i, _vp, _vp, _vp, _ll, _vp], _i),
    "skm_build_tails": ([_vp, _ll, _i, _i, _i, _vp, _vp], _i),
    "skm_gate_threshold": ([_vp, _i, _f, _i, _vp, _vp, _vp, _f, _vp], _i),
    "skm_defer_cert_flags": ([_vp, _vp, _i, _i, _vp, _vp], _i),
    "skm_deferred_cert_count": ([_vp, _vp, _vp], _i),
    "skm_pruned_scan": ([C.POINTER(ScanParams), _vp], _i),
    "skm_first_nonfinite": ([_vp, _ll, _ll, _i, _vp, _vp], _i),
    "skm_wcss_workspace_bytes": ([], _ll),
    "skm_wcss": ([_vp, _ll, _vp, _ll, _vp, _ll, _i, _vp, _vp, _vp], _i),
    "skm_ingest_records": ([_vp, _ll, _i, _i, _i, _ll, _vp, _ll, _vp, _vp, _vp], _i),
    "skm_gather_front": ([_vp, _vp, _ll, _vp, _i, _i, _vp, _vp, _ll, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
                         _i),
    "skm_topk_rows": ([_vp, _ll, _i, _i, _i, _vp, _vp, _ll, _i, _vp], _i),
    "skm_topk_merge": ([_vp, _vp, _i, _i, _i, _vp, _vp, _vp], _i),
    "skm_etr_hits": ([_vp, _i, _i, _vp, _i, _i, _vp, _ll, _ll, _i, _i, _vp, _vp], _i),
    "skm_probe_tally": ([_vp, _i, _i, _vp, _i, _i, _vp, _ll, _i, _i, _vp, _vp, _vp, _vp], _i),
}

EXPORTED_SYMBOLS = tuple(_SIGS)

_lib = None
_load_error: str | None = None


def load():
    """Load (once) and return the ctypes library; raise NativeUnavailable if absent."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        _load_error = f"{LIB_PATH} not built (run paper_2603_20009_b200.build.build())"
        raise NativeUnavailable(_load_error)
    try:
        lib = C.CDLL(LIB_PATH)
    except OSError as e:  # pragma: no cover - depends on the box
        _load_error = str(e)
        raise NativeUnavailable(f"cannot load {LIB_PATH}: {e}") from e
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().skm_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed ({rc}): {msg}")


def call(name: str, *args, flops: float = 0.0, nbytes: float = 0.0, tag: str | None = None) -> None:
    """Invoke an ABI entry point; raise NativeError on failure.  When a profiling.KernelTimer
    is active the launch is bracketed by CUDA events and its algorithmic work recorded."""
    from . import profiling
    prof = profiling.current()
    fn = getattr(load(), name)
    if prof is None:
        check(fn(*args), name)
        return
    e0 = prof.begin()
    check(fn(*args), name)
    prof.end(tag or name, e0, flops, nbytes)

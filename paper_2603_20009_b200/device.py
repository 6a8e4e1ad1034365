"""Device plumbing (torch for allocation + streams) and the device twin of the reference's
4-function kernel protocol (kernels.py:41-51 -> _kernels.pyx:14-142).

The protocol functions here take CUDA tensors instead of NumPy arrays and run the
corresponding libskm_b200 entry point; they are the bitwise-parity surface tested against
the oracle.  ``get_kernels("cuda")`` returns this module's ``KERNELS`` namespace.
"""

from __future__ import annotations

import ctypes as C
from types import SimpleNamespace

import numpy as np
import torch

from . import native


def on_device(fn):
    """Public entry points with a ``device=`` argument run with that device current: native
    kernels launch on the current device's stream (stream_handle), so torch work and native work
    stay on one device and one stream."""
    import functools
    import inspect as _inspect
    pos = list(_inspect.signature(fn).parameters).index("device")

    @functools.wraps(fn)
    def wrapper(*args, **kw):
        dev = kw.get("device", args[pos] if len(args) > pos else None)
        if dev is None or not torch.cuda.is_available():
            return fn(*args, **kw)
        with torch.cuda.device(torch.device(dev)):
            return fn(*args, **kw)
    return wrapper


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise native.NativeUnavailable("a CUDA device is required (no CPU fallback by design)")
    native.load()
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


def ptr(t: torch.Tensor | None):
    return None if t is None else C.c_void_p(t.data_ptr())


def stream_handle():
    """The current CUDA stream of the current device as a raw handle (the fast path of
    torch.cuda.current_stream().cuda_stream: ~15x cheaper per call, which matters for the
    launch-bound small fits and the per-group host work)."""
    return C.c_void_p(torch._C._cuda_getCurrentRawStream(torch.cuda.current_device()))


def to_host(t: torch.Tensor) -> np.ndarray:
    """Device tensor (any strides) -> host NumPy array through one DMA into pinned memory (the
    array owns the pinned storage; a pageable .cpu() runs at a fraction of the link rate)."""
    h = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return h.numpy()


def padded_ld(d: int) -> int:
    """Row stride (elements) for device matrices: multiple of 4 so TMA accepts it."""
    return (d + 3) // 4 * 4


def to_device_matrix(x: np.ndarray | torch.Tensor, ld: int | None = None, device=None) -> torch.Tensor:
    """Copy an (n, d) float32 matrix into a padded (n, ld) device buffer (pad columns = 0)."""
    dev = require_cuda(device)
    n, d = x.shape
    ld = padded_ld(d) if ld is None else ld
    out = torch.zeros((n, ld), dtype=torch.float32, device=dev)
    src = torch.as_tensor(x) if isinstance(x, np.ndarray) else x
    out[:, :d].copy_(src, non_blocking=False)
    return out


def split_hilo(x: torch.Tensor, cols: int) -> tuple[torch.Tensor, torch.Tensor]:
    rows, ld = x.shape
    hi = torch.empty_like(x)
    lo = torch.empty_like(x)
    native.call("skm_split_hilo", ptr(x), ld, rows, cols, ptr(hi), ptr(lo), ld, stream_handle())
    return hi, lo


def row_sq_norms(x: torch.Tensor, dims: int, out: torch.Tensor | None = None) -> torch.Tensor:
    rows, ld = x.shape
    if out is None:
        out = torch.empty(rows, dtype=torch.float32, device=x.device)
    native.call("skm_row_sq_norms", ptr(x), ld, rows, dims, ptr(out), stream_handle())
    return out


def gemm(a_hi, a_lo, b_hi, b_lo, M: int, N: int, K: int, mode: int, *, out=None, xsq=None, ysq=None,
         top=None, thr=None, cand=None, cand_cnt=None,
         cand_cap: int = 0, n_split: int = 1, row_offset: int = 0, ext_k: int = 0, xsq_ext=None, ysq_ext=None,
         thr1=None, cert_eps: float = 0.0) -> None:
    p = native.GemmParams()
    p.a_hi, p.a_lo, p.lda = a_hi.data_ptr(), a_lo.data_ptr(), a_hi.stride(0)
    p.b_hi, p.b_lo, p.ldb = b_hi.data_ptr(), b_lo.data_ptr(), b_hi.stride(0)
    p.M, p.N, p.K, p.mode, p.n_split = M, N, K, mode, n_split
    if out is not None:
        p.out, p.ldo = out.data_ptr(), out.stride(0)
    for name, t in (("xsq", xsq), ("ysq", ysq), ("top", top),
                    ("thr", thr), ("cand", cand), ("cand_cnt", cand_cnt),
                    ("xsq_ext", xsq_ext), ("ysq_ext", ysq_ext), ("thr1", thr1)):
        if t is not None:
            setattr(p, name, t.data_ptr())
    p.cand_cap = cand_cap
    p.row_offset = row_offset
    p.ext_k, p.cert_eps = ext_k, cert_eps
    native.check(native.load().skm_gemm_tf32x3(C.byref(p), stream_handle()), "skm_gemm_tf32x3")


def matmul_nt(a: torch.Tensor, b: torch.Tensor, K: int) -> torch.Tensor:
    """out = a[:, :K] @ b[:, :K].T on the tensor cores (3xTF32), fp32 result (M, N)."""
    a_hi, a_lo = split_hilo(a, K)
    b_hi, b_lo = split_hilo(b, K)
    M, N = a.shape[0], b.shape[0]
    out = torch.empty((M, native_ld(N)), dtype=torch.float32, device=a.device)
    gemm(a_hi, a_lo, b_hi, b_lo, M, N, K, native.GEMM_STORE, out=out)
    return out[:, :N]


def native_ld(n: int) -> int:
    return padded_ld(n)


# ------------------------------------------------------------------ kernel protocol (device)
def seed_thresholds(x: torch.Tensor, centroids: torch.Tensor, assign: torch.Tensor, out: torch.Tensor,
                    n_threads: int = 0, d: int | None = None) -> None:
    n = x.shape[0]
    d = x.shape[1] if d is None else d
    native.call("skm_seed_thresholds", ptr(x), x.stride(0), ptr(centroids), centroids.stride(0), ptr(assign), n, d,
                ptr(out), stream_handle())


def scan_bank(partial_dists, x, tail, block_offsets, block_dims, theta_factors, d_prime, bank_offset, tau, assign,
              sentinel, n_threads=0):
    """Device scan_bank: same arguments as _kernels.pyx:14-27 (CUDA tensors); returns
    (survivors, dims_touched) like the reference."""
    n, kb = partial_dists.shape
    counters = torch.zeros(2, dtype=torch.int64, device=partial_dists.device)
    native.call("skm_scan_bank", ptr(partial_dists), n, kb, ptr(x), x.stride(0), ptr(tail), ptr(block_offsets),
                ptr(block_dims), int(block_dims.shape[0]), ptr(theta_factors), int(d_prime), int(bank_offset),
                ptr(tau), ptr(assign), int(bool(sentinel)), ptr(counters), stream_handle())
    s, t = counters.tolist()
    return int(s), int(t)


def accumulate_centroid_sums(x: torch.Tensor, assign: torch.Tensor, sums: torch.Tensor, counts: torch.Tensor,
                             d: int | None = None) -> None:
    n = x.shape[0]
    d = x.shape[1] if d is None else d
    k = sums.shape[0]
    lib = native.load()
    ws_bytes = lib.skm_update_workspace_bytes(n, k) + 4 * max(n, 1) + 8 * k + 1024
    ws = torch.empty(int(ws_bytes), dtype=torch.uint8, device=x.device)
    native.call("skm_accumulate_centroid_sums", ptr(x), x.stride(0), ptr(assign), n, d, k, ptr(sums), ptr(counts),
                ptr(ws), ws.numel(), stream_handle())


def portable_matmul(a: torch.Tensor, b: torch.Tensor, dims: int, out: torch.Tensor, n_threads: int = 0) -> None:
    n, m = a.shape[0], b.shape[0]
    native.call("skm_portable_matmul", ptr(a), a.stride(0), ptr(b), b.stride(0), n, m, dims, ptr(out),
                out.stride(0), stream_handle())


KERNELS = SimpleNamespace(
    name="cuda",
    scan_bank=scan_bank,
    seed_thresholds=seed_thresholds,
    accumulate_centroid_sums=accumulate_centroid_sums,
    portable_matmul=portable_matmul,
)


def get_kernels(name: str | None = None):
    """Reference-compatible dispatch (kernels.py:41-51); the only backend is the device one."""
    if name in (None, "auto", "", "cuda", "compiled"):
        return KERNELS
    raise ValueError(f"unknown kernel backend {name!r}")


def available_backends() -> list[str]:
    return ["cuda"]

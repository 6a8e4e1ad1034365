"""Device-resident SuperKMeans Lloyd loop (the north-star hot path).

Host orchestration of ``core._fit_rotated`` (pkg/src/superkmeans/core.py:284-414), with every
per-vector operation running in libskm_b200:

  iteration 1 (and every iteration when d < 80):  fused full-distance GEMM + row argmin
                                                   (core.py:169-192)
  iterations >= 2:  seed tau (core.py:237) -> gate threshold -> partial-distance GEMM fused with
                    the ADSampling first gate and ascending-index candidate emission -> exact
                    sequential-tau pruning scan over PDX-quad centroid tails (core.py:195-267)
  update:           stable cluster sort + ordered f64 member sums + divide (core.py:79-100),
                    host-drawn empty-cluster splits applied on device (core.py:103-128)
  control:          d' controller, convergence and ETR decisions on host scalars
                    (core.py:131-161, 305-316, 379-399)

Data never returns to the host inside the loop except O(k) counts (needed by the host RNG of
the split step, exactly like the reference), a handful of scalars, and -- only when an
``inspect`` callback is given -- the snapshot the callback receives.
"""

from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import native
from .config import (
    IterationStats,
    KMeansConfig,
    WorkCounters,
    initial_d_prime,
    pruning_supported,
    tail_block_layout,
)
from .device import padded_ld, ptr, stream_handle
from .hostmath import (
    SPLIT_EPS,
    adjust_d_prime,
    init_indices,
    plan_splits,
    prune_rate_from_totals,
    sentinel_factors,
    threshold_factors,
)

PRUNE_HIST = None  # diagnostics (tools/): device u64[nb + 1] histogram of prune blocks
COLLECT_DIAG = os.environ.get("SKM_DIAG", "0") == "1"  # read scan diagnostics back every iteration
# GEMM-certified tail-block-0 prunes (gemm_tf32x3.cuh, GATE ext_k): the gate GEMM also sums
# the first 64 tail dimensions and flags candidates whose distance there exceeds fl(tau F1)
# by more than cert_eps(K) * (|x|^2 + |c|^2) over those dimensions -- the rigorous bound of
# both the tensor-core value and the reference's own rounding of that running sum (cert_eps) --
# so the scan counts them (survivor, 64 dims) without walking them.
# (a prefix of tail block 0 lower-bounds its running sum, so any ext <= 64 is a valid certificate)
CERT_EXT = int(os.environ.get("SKM_CERT_EXT", "64")) if os.environ.get("SKM_CERT", "1") != "0" else 0
# flat first pass of the scan (csrc/flatscan.cuh): rows whose threshold changes only at their own
# previous centroid are resolved without in-order resolution; the rest take the exact kernel
SCAN_FLAT = os.environ.get("SKM_SCAN_FLAT", "1") != "0"
# ... used once the loop has nearly converged: rows that change assignment fall back to the exact
# kernel after a partial flat walk, so early iterations (10-40 % changing) are faster without it
# (c2: -3 % scan time per iteration at <= 4.4 % changed, +13 % at 40 %; profiles/r2_summary.md)
FLAT_MAX_CHANGED = float(os.environ.get("SKM_SCAN_FLAT_MAX", "0.05"))
# exact_work_stats = False: candidates that cannot win skip the tail walk.  The gate GEMM's
# certification partial then runs over the whole tail (d' front + d - d' extension columns, the
# extension as one TF32 product), about 2.2x the gate's tensor work; the walk it removes pays
# off only while the walk is long.  c2 per pruned iteration (exact -> option, ms): it2 209 -> 97
# (14.8 % of k survived the gate), it3 91 -> 72 (5.6 %), it4 53 -> 66 (2.8 %), it5 50 -> 60; c5's
# meso loop (k = 430) 1.8 -> 0.31 s.  The previous iteration's survivor fraction predicts the
# walk, so the full certificate runs in the first pruned iteration and while the previous
# one kept more than NOWIN_SURV_FRAC of k.
NOWIN_SURV_FRAC = float(os.environ.get("SKM_NOWIN_SURV_FRAC", "0.12"))


def cert_eps(k_dim: int, paired: bool = True) -> float:
    """Margin of the block-0 certificate over k_dim = d' + ext columns, relative to xsq + ysq
    there: the tensor-core distance D~ and the reference's running sum fl(p + block sum) each lie
    within tc_kappa * (xsq + ysq + D) <= 3 tc_kappa * (xsq + ysq) of the exact distance (D <=
    2 (xsq + ysq)), so 6 tc_kappa separates them from the threshold for certain."""
    return 6.0 * tc_kappa(k_dim, paired)


def nowin_cert_eps(d: int, ext: int, hi_only: bool = True) -> float:
    """Margin of the full-d certificate (exact_work_stats = False), relative to xsq + ysq over d.
    The reference's complete running sum (front chain + 64-dim block sums) lies within
    3 kappa_ref (xsq + ysq) of the exact distance, kappa_ref = 2 gamma_d + 16 u (as in cert_eps).
    The tensor-core distance: ``hi_only`` (NOWIN_HI_ONLY) runs the ext / 32 extension k-blocks as
    one TF32 product -- truncated operands, |x c - x_h c_h| <= (2^-9 + 2^-20) |x c|, so the inner
    product is off by <= 2^-10 (xsq + ysq) and the distance by twice that -- plus 4 truncating
    TMEM accumulations per k-block and the 3xTF32 front (2^-16); else 3xTF32 throughout (12 MMAs
    per k-block).  A quarter more on top for slack."""
    g = d * _U / (1.0 - d * _U)
    blocks = (ext + 31) // 32
    ref = 3.0 * (2.0 * g + 16.0 * _U)
    if hi_only:
        tc = 2.0 * ((2.0 ** -10) * (1.0 + 2.0 ** -9) + 4.0 * blocks * 2.0 ** -23 + 2.0 ** -16 + g) + 16.0 * _U
    else:
        tc = 3.0 * (2.0 * (g + max(2.0 ** -16, 12.0 * blocks * 2.0 ** -23)) + 16.0 * _U)
    return 1.25 * (tc + ref)


NOWIN_HI_ONLY = os.environ.get("SKM_NOWIN_HI_ONLY", "1") != "0"
# the certified entries of a full-d certificate leave the in-order scan: it records each row's
# tau improvements and skm_deferred_cert_count settles their survivor decisions in parallel
DEFER_CERT = os.environ.get("SKM_DEFER_CERT", "1") != "0"


def cert_extension(data, cents, plan, tau: torch.Tensor, thr1: torch.Tensor, n: int, nowin: bool) -> dict:
    """The gate GEMM's certification-partial arguments ({} = none), with thr1[:n] filled.
    Default: the block-0 certificate (CERT_EXT columns after d', thr1 = fl(tau F1)).  ``nowin``
    (exact_work_stats = False): the partial covers all d columns (one TF32 product with
    NOWIN_HI_ONLY) and thr1 = tau, so a flagged column's complete distance lies above the seed
    tau -- it never replaces the best (tau only decreases) and the scan settles only its
    survivor decision, as for a block-0 prune.  ``xsq_ext`` is the full-height row-norm vector
    (callers slice or gather it)."""
    d, dp = data.d, plan.d_prime
    if plan.sentinel or dp % 4:
        return {}
    st = stream_handle()
    if nowin and dp < d:
        # the whole tail: a prefix would certify too (block sums >= 0, the running sum only
        # grows), but measured on c2 a 256-768 column prefix certified almost nothing
        ext = d - dp
        native.call("skm_gate_threshold", ptr(tau), n, 1.0, 0, ptr(thr1), None, None, 0.0, st)
        return dict(ext_k=ext, xsq_ext=data.norms(dp + ext), ysq_ext=cents.ext_norms(dp + ext),
                    cert_eps=nowin_cert_eps(d, ext, NOWIN_HI_ONLY), ext_hi_only=NOWIN_HI_ONLY, nowin=True)
    if dp + CERT_EXT > d or plan.widths[0] != 64:
        return {}
    native.call("skm_gate_threshold", ptr(tau), n, float(plan.gate[1]), 0, ptr(thr1), None, None, 0.0, st)
    return dict(ext_k=CERT_EXT, xsq_ext=data.norms(dp + CERT_EXT), ysq_ext=cents.ysq_ext,
                cert_eps=cert_eps(dp + CERT_EXT, GATE_KPAIR), ext_hi_only=False)


# ---------------------------------------------------------------- exact-chain policy
# The reference's contractions are OpenBLAS sgemm (one fma chain per output, K blocked by 448 in
# the threaded driver) or, with gemm_backend="portable", the Cython mul+add chain (no blocking);
# see csrc/sgemm_chain.cuh.  Contractions whose every output bit propagates (the rotation, the
# un-rotation, the ETR distance blocks) run as that chain on the CUDA cores; the Lloyd loop's
# large distance GEMMs run on the tensor cores (3xTF32) and every decision that could depend on
# their rounding is re-evaluated with the chain (argmin near-ties, gate / prune checkpoints and
# winners in the scan), so the loop reproduces the reference bit for bit.
GEMM_Q = 448
_U = 2.0 ** -24
GATE_KPAIR = True  # csrc/gemm_tf32x3.cuh SKM_GEMM_KPAIR: the tensor-core GEMM accumulates 128-wide TMEM partials


def resolve_gemm_backend(backend: str = "auto") -> str:
    """distance.py:33-43 (env SUPERKMEANS_GEMM when "auto")."""
    if backend == "auto":
        env = os.environ.get("SUPERKMEANS_GEMM", "").strip().lower()
        if env in ("blas", "portable"):
            return env
        if env:
            raise ValueError(f"unknown SUPERKMEANS_GEMM value {env!r}")
        return "blas"
    if backend not in ("blas", "portable"):
        raise ValueError(f"unknown gemm backend {backend!r}")
    return backend


def chain_policy(backend: str = "auto") -> tuple[int, int]:
    """(flavour, q) of the distance chain: blas -> (fma, 448), portable -> (mul+add, none)."""
    return (1, 0) if resolve_gemm_backend(backend) == "portable" else (0, GEMM_Q)


def tc_kappa(k_dim: int, paired: bool = True) -> float:
    """Rigorous bound coefficient for |p_tensor_core - p_chain| <= kappa * (xsq + ysq + p) of a
    squared distance over k_dim columns: the chain's own error
    gamma_K = K u / (1 - K u) plus the 3xTF32 error (dropped lo*lo and tf32 truncation of lo:
    3 * 2^-20 per product) and the truncating TMEM accumulation of a partial (12 MMAs of a 32-wide
    k-block: 1.5 * 2^-20; ``paired`` = the GEMM's 128-wide partials, 48 MMAs: 6 * 2^-20, so
    9 * 2^-20 <= 2^-16 in all), then the fp32 adds of the partials (inside gamma_K), with a
    factor 2 of slack, plus 16 u for the expansion's roundings."""
    g = k_dim * _U / (1.0 - k_dim * _U)
    return 2.0 * (g + (2.0 ** -16 if paired else 2.0 ** -17)) + 16.0 * _U


def chain_gemm(a: torch.Tensor, b: torch.Tensor, M: int, N: int, K: int, out: torch.Tensor, flavour: int = 0,
               q: int = GEMM_Q, xsq: torch.Tensor | None = None, ysq: torch.Tensor | None = None,
               b_kmajor: bool = False) -> None:
    """out = the reference's sgemm (flavour 0) / portable_matmul (1) bits of a[:, :K] . b[:, :K]^T
    (b_kmajor: a[:, :K] . b[:K, :N], b stored [K][N] -- the cp.async kernel), or (with xsq / ysq)
    the clamped squared distances of distance.expand_to_sq_l2."""
    p = native.ChainParams()
    p.a, p.lda, p.b, p.ldb = a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0)
    p.M, p.N, p.K, p.flavour, p.q = M, N, K, flavour, q
    p.b_kmajor = 1 if b_kmajor else 0
    p.mode = 1 if xsq is not None else 0
    p.out, p.ldo = out.data_ptr(), out.stride(0)
    if xsq is not None:
        p.xsq, p.ysq = xsq.data_ptr(), ysq.data_ptr()
    native.call("skm_chain_gemm", C.byref(p), stream_handle(), flops=2.0 * M * N * K,
                tag="chain_dist" if xsq is not None else "chain_gemm")


def _i64(t: torch.Tensor) -> int:
    return int(t.item())


SHARD_ALIGN = 8192  # NumPy's reduction buffer: shards of whole buffers keep wcss = np.sum bitwise


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row shard of a rank.  Large inputs take equal shares rounded up to whole
    8192-row buffers, so every rank's partial sums of tau are whole buffers of the reference's
    np.sum (core.py:344) and the reduced wcss is bitwise the single-GPU one; the rounding is skipped
    when it could leave a rank empty (n <= world * world * 8192)."""
    per = -(-n // world)
    if world > 1 and n > world * world * SHARD_ALIGN:
        per = -(-per // SHARD_ALIGN) * SHARD_ALIGN
    lo = min(n, rank * per)
    return lo, min(n, lo + per)


class Comm:
    """Row-sharded data parallelism: one allreduce(sum) per iteration over a packed buffer.

    ``world == 1`` is the identity.  With ``torch.distributed`` initialised (NCCL on GPUs,
    gloo in CPU tests) every rank holds a contiguous row shard and replicated centroids.
    """

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist if dist.is_available() and dist.is_initialized() else None
        self.group = group
        self.world = self.dist.get_world_size(group) if self.dist else 1
        self.rank = self.dist.get_rank(group) if self.dist else 0

    def allreduce_(self, t: torch.Tensor) -> torch.Tensor:
        if self.world > 1:
            self.dist.all_reduce(t, group=self.group)
        return t

    def allreduce_min_(self, t: torch.Tensor) -> torch.Tensor:
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        return t

    @classmethod
    def local(cls) -> "Comm":
        """World-size-1 communicator (identity collectives) for work that is rank-local."""
        c = cls.__new__(cls)
        c.dist, c.group, c.world, c.rank = None, None, 1, 0
        return c

    def all_to_all_rows(self, send: torch.Tensor, send_counts: list[int], recv_counts: list[int]) -> torch.Tensor:
        """Rows [sum(send_counts[:r]), +send_counts[r]) of ``send`` go to rank r; returns the
        rows received from every rank, in rank order.  NCCL moves device memory directly; other
        backends (gloo in the one-GPU multi-rank tests) are staged through host memory."""
        shape = (int(sum(recv_counts)),) + tuple(send.shape[1:])
        if self.world == 1:
            return send[:shape[0]].clone()
        if self.dist.get_backend(self.group) == "nccl":
            out = torch.empty(shape, dtype=send.dtype, device=send.device)
            self.dist.all_to_all_single(out, send.contiguous(), output_split_sizes=list(recv_counts),
                                        input_split_sizes=list(send_counts), group=self.group)
            return out
        out = torch.empty(shape, dtype=send.dtype)
        self.dist.all_to_all_single(out, send.cpu().contiguous(), output_split_sizes=list(recv_counts),
                                    input_split_sizes=list(send_counts), group=self.group)
        return out.to(send.device)

    def shard(self, n: int) -> tuple[int, int]:
        """Contiguous row range of this rank."""
        return shard_bounds(n, self.world, self.rank)


@dataclass
class LoopOutput:
    centroids_rotated: np.ndarray
    assignments: np.ndarray
    best_sq_dist: np.ndarray
    stats: list
    terminated_by: str
    d_prime_final: int | None
    init_indices: np.ndarray
    work: WorkCounters
    recall_history: list
    phase_seconds: dict
    centroids_dev: torch.Tensor | None = None
    assign_dev: torch.Tensor | None = None
    device_ms: dict = field(default_factory=dict)
    scan_blocks: list = field(default_factory=list)  # speculative 64-dim block sums computed per pruned iter
    scan_waves: list = field(default_factory=list)   # warp-waves of the scan per pruned iter
    scan_diag: list = field(default_factory=list)    # [spec blocks, spec waves, exact blocks, exact waves, exact rows]


class _Timer:
    """CUDA-event phase timer (replaces the reference's perf_counter brackets)."""

    def __init__(self):
        self.open: dict[str, torch.cuda.Event] = {}
        self.spans: list[tuple[str, torch.cuda.Event, torch.cuda.Event]] = []

    def start(self, name):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.open[name] = e

    def stop(self, name):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.spans.append((name, self.open.pop(name), e))

    def collect(self) -> dict:
        out: dict[str, float] = {}
        if self.spans:
            self.spans[-1][2].synchronize()
        for name, a, b in self.spans:
            out[name] = out.get(name, 0.0) + a.elapsed_time(b) / 1e3
        self.spans.clear()
        return out


class DeviceData:
    """Rotated training rows resident in HBM, with their 3xTF32 split and norms."""

    def __init__(self, xr: torch.Tensor, d: int):
        self.x = xr            # (n, ld) fp32, pad columns zero
        self.n = xr.shape[0]
        self.d = d
        self.ld = xr.shape[1]
        # 3xTF32 operands: the rows themselves are the hi operand (kind::tf32 truncates fp32
        # inputs bit-identically to the explicit split), only lo = x - trunc(x) is stored
        self.hi = xr
        self.lo = torch.empty_like(xr)
        if self.n:
            native.call("skm_split_hilo", ptr(xr), self.ld, self.n, d, None, ptr(self.lo), self.ld,
                        stream_handle(), nbytes=8.0 * self.n * self.ld)
        self._norms: dict[int, torch.Tensor] = {}

    def norms(self, dims: int) -> torch.Tensor:
        t = self._norms.get(dims)
        if t is None:
            t = torch.empty(max(self.n, 1), dtype=torch.float32, device=self.x.device)
            if self.n:
                native.call("skm_row_sq_norms", ptr(self.x), self.ld, self.n, dims, ptr(t), stream_handle(),
                            nbytes=4.0 * self.n * dims)
            if len(self._norms) > 4:
                self._norms.pop(next(iter(self._norms)))
            self._norms[dims] = t
        return t


class Centroids:
    """Replicated centroid state: row-major matrix, its split, norms, PDX-quad tails."""

    def __init__(self, c: torch.Tensor, d: int):
        self.c = c
        self.k = c.shape[0]
        self.d = d
        self.ld = c.shape[1]
        self.hi = torch.empty_like(c)
        self.lo = torch.empty_like(c)
        self.ysq = torch.empty(self.k, dtype=torch.float32, device=c.device)
        self.tails = None
        self.ysq_ext = None
        self.ysq_max = torch.zeros(1, dtype=torch.float32, device=c.device)  # max_j ysq (error bounds)

    def ext_norms(self, dims: int) -> torch.Tensor:
        """ysq over the first ``dims`` columns for the full-d certificate (exact_work_stats = False)."""
        if getattr(self, "ysq_cert", None) is None:
            self.ysq_cert = torch.empty(self.k, dtype=torch.float32, device=self.c.device)
        native.call("skm_row_sq_norms", ptr(self.c), self.ld, self.k, dims, ptr(self.ysq_cert), stream_handle())
        return self.ysq_cert

    def refresh(self, dims: int, d_prime: int | None):
        """Recompute split + norms over `dims` (+ tails at d_prime) after an update."""
        native.call("skm_split_hilo", ptr(self.c), self.ld, self.k, self.d, ptr(self.hi), ptr(self.lo), self.ld,
                    stream_handle())
        native.call("skm_row_sq_norms", ptr(self.c), self.ld, self.k, dims, ptr(self.ysq), stream_handle())
        native.call("skm_max_f32", ptr(self.ysq), self.k, ptr(self.ysq_max), stream_handle())
        if d_prime is not None:
            if self.ysq_ext is None:
                self.ysq_ext = torch.empty(self.k, dtype=torch.float32, device=self.c.device)
            native.call("skm_row_sq_norms", ptr(self.c), self.ld, self.k, min(self.d, d_prime + 64), ptr(self.ysq_ext),
                        stream_handle())
            nb = (self.d - d_prime + 63) // 64
            need = self.k * 64 * nb
            if self.tails is None or self.tails.numel() < need:
                self.tails = torch.empty(need, dtype=torch.float32, device=self.c.device)
            native.call("skm_build_tails", ptr(self.c), self.ld, self.k, self.d, d_prime, ptr(self.tails),
                        stream_handle())


def _gemm(a_hi, a_lo, b_hi, b_lo, M, N, K, mode, **kw):
    p = native.GemmParams()
    p.a_hi, p.a_lo, p.lda = a_hi.data_ptr(), a_lo.data_ptr(), a_hi.stride(0)
    p.b_hi, p.b_lo, p.ldb = b_hi.data_ptr(), b_lo.data_ptr(), b_hi.stride(0)
    p.M, p.N, p.K, p.mode = M, N, K, mode
    p.n_split = kw.pop("n_split", 1)
    top = kw.pop("top", None)
    if top is not None:
        p.top = top.data_ptr()
    out = kw.pop("out", None)
    if out is not None:
        p.out, p.ldo = out.data_ptr(), out.stride(0)
    p.cand_cap = kw.pop("cand_cap", 0)
    p.row_offset = kw.pop("row_offset", 0)
    p.ext_k = kw.pop("ext_k", 0)
    p.cert_eps = kw.pop("cert_eps", 0.0)
    p.ext_hi_only = int(kw.pop("ext_hi_only", 0))
    kw.pop("nowin", None)
    for name, t in kw.items():
        if t is not None:
            setattr(p, name, t.data_ptr())
    names = {native.GEMM_STORE: "gemm_store", native.GEMM_DIST: "gemm_dist", native.GEMM_ARGMIN: "gemm_argmin",
             native.GEMM_GATE: "gemm_gate"}
    # algorithmic flops of the launch: the certification extension's columns are computed too
    native.call("skm_gemm_tf32x3", C.byref(p), stream_handle(), flops=2.0 * M * N * (K + p.ext_k), tag=names[mode])


def _n_split(m_rows: int, n_cols: int, sms: int = 148) -> int:
    """Spread N over CTAs when there are too few 128-row M tiles to fill the chip."""
    m_tiles = (m_rows + 127) // 128
    n_tiles = (n_cols + 255) // 256
    if m_tiles >= 2 * sms:
        return 1
    return max(1, min(n_tiles, (2 * sms + m_tiles - 1) // m_tiles))


def _l2_split(m_rows: int, n_cols: int, k_dim: int, cap: int, sms: int = 148) -> int:
    """N split for a long GEMM whose concurrent A tiles (one 128-row hi+lo tile per SM, K wide)
    would overflow the 126 MB L2: the CTAs of one M tile run side by side (block order), so A
    is fetched from HBM about once instead of once per N tile (c2 ARGMIN: 148 x 1.5 MB)."""
    s = _n_split(m_rows, n_cols, sms)
    if s == 1 and sms * 128 * k_dim * 8 > (48 << 20):
        s = min(cap, (n_cols + 255) // 256)
    return max(1, s)


def _sm_count(dev) -> int:
    try:
        return int(torch.cuda.get_device_properties(dev).multi_processor_count)
    except Exception:  # pragma: no cover - no device
        return 148


class Workspace:
    def __init__(self, dev, n: int, k: int, d: int, cfg: KMeansConfig):
        self.dev = dev
        self.cap = min(cfg.cand_cap, (k + 31) // 32 * 32)
        # candidate slab (8 B per candidate, rows as wide as k by default so no row overflows
        # into the dense pass) bounded to 16 GiB of the 180 GB; batches are whole waves of
        # 128-row gate-GEMM tiles over the SMs (one CTA per SM) so no launch ends on a
        # partial wave except the last
        per_wave = 128 * _sm_count(dev)
        mem_rows = (16 << 30) // (8 * self.cap)
        b = min(cfg.x_batch_device, mem_rows)
        b = max(per_wave, b // per_wave * per_wave) if b >= per_wave else max(128, b // 128 * 128)
        if n > b:
            if n <= b + b // 4 and n <= mem_rows:
                b = n  # one launch instead of a near-empty tail batch (e.g. 125K-row shards at 8 GPUs)
            else:  # balance the batches, whole waves each
                even = -(-n // -(-n // b))
                b = min(b, -(-even // per_wave) * per_wave if b >= per_wave else max(128, even))
        b = max(128, min(max(n, 1), b))
        self.batch = b
        i32, f32 = torch.int32, torch.float32
        nn = max(n, 1)
        self.assign = torch.zeros(nn, dtype=i32, device=dev)
        self.prev = torch.zeros(nn, dtype=i32, device=dev)
        self.tau = torch.full((nn,), float("inf"), dtype=f32, device=dev)
        self.thr = torch.empty(nn, dtype=f32, device=dev)
        self.top = None
        self.amb_rows = torch.empty(nn, dtype=i32, device=dev)
        self.amb_count = torch.zeros(1, dtype=i32, device=dev)
        self.chain_flavour, self.chain_q = chain_policy(cfg.gemm_backend)
        self.cand = torch.empty((b, self.cap, 2), dtype=i32, device=dev)  # {index, float bits} records
        self.cand_cnt = torch.empty(b, dtype=i32, device=dev)
        self.counters = torch.zeros(3, dtype=torch.int64, device=dev)
        self.work = torch.zeros(256, dtype=torch.int32, device=dev)  # per-SM scan row queues
        # scan diagnostics: spec blocks, spec waves, exact blocks, exact waves, rows routed to the exact phase
        self.diag = torch.zeros(8, dtype=torch.int64, device=dev)
        self.flat = False  # this pass uses the flat scan (the loop decides per iteration)
        self.nowin = False  # this pass certifies the candidates that cannot win (full-d partial)
        self.fb_rows = torch.empty(b, dtype=i32, device=dev)  # flat scan: fallback rows of a batch
        self.fb_count = torch.zeros(1, dtype=i32, device=dev)
        self.bx = torch.empty(b, dtype=f32, device=dev)
        self.bthr = torch.empty(b, dtype=f32, device=dev)
        self.thr1 = torch.empty(nn, dtype=f32, device=dev)
        self.bx_ext = torch.empty(b, dtype=f32, device=dev)
        self.bthr1 = torch.empty(b, dtype=f32, device=dev)
        self._front = None
        self.order = torch.empty(nn, dtype=i32, device=dev)
        self.counts = torch.empty(k, dtype=i32, device=dev)
        self.offsets = torch.empty(k, dtype=i32, device=dev)
        lib = native.load()
        self.sort_ws = torch.empty(int(lib.skm_update_workspace_bytes(n, k)), dtype=torch.uint8, device=dev)
        self.stats_ws = torch.empty(int(lib.skm_stats_workspace_bytes(n)), dtype=torch.uint8, device=dev)
        self.wcss = torch.zeros(1, dtype=torch.float64, device=dev)
        self.changed = torch.zeros(1, dtype=torch.int64, device=dev)

    def defer_buffers(self):
        """Deferred certified entries (exact_work_stats = False): seed-tau copy (global rows),
        per-batch-row skip flags, improvement records [batch][32] {j, tau bits} and counts."""
        if getattr(self, "_defer", None) is None:
            b = self.batch
            self._defer = (torch.empty_like(self.tau), torch.empty(b, dtype=torch.int32, device=self.dev),
                           torch.empty((b, 32, 2), dtype=torch.int32, device=self.dev),
                           torch.empty(b, dtype=torch.int32, device=self.dev))
        return self._defer

    def front_buffers(self, fld: int):
        """Gathered (hi, lo) front rows of one cluster-ordered batch."""
        if self._front is None or self._front[0].shape[1] < fld:
            self._front = (torch.empty((self.batch, fld), dtype=torch.float32, device=self.dev),
                           torch.empty((self.batch, fld), dtype=torch.float32, device=self.dev))
        return self._front[0][:, :fld], self._front[1][:, :fld]

    def top_records(self, n):
        """ARGMIN top-2 records, int4 per (N split, row)."""
        if self.top is None or self.top.numel() < 4 * n:
            self.top = torch.empty(4 * max(n, 1), dtype=torch.int32, device=self.dev)
        return self.top


# ------------------------------------------------------------------------------ passes
def full_assign_pass(data: DeviceData, cents: Centroids, ws: Workspace, row0: int = 0, rows: int | None = None):
    """Exact argmin over all centroids (lowest index on ties) -> ws.assign / ws.tau, bitwise the
    reference's batched sgemm + expansion + argmin (core.py:169-192).

    The tensor-core ARGMIN GEMM keeps each row's best and runner-up distances; its argmin is the
    reference's whenever the runner-up is outside the rigorous error bound of both values (the
    common case).  tau is then recomputed as the reference's own chain distance of that pair, and
    the few rows with a runner-up inside the bound get the whole distance row from the chain GEMM
    (the reference's exact bits, ties to the lowest index)."""
    n = data.n if rows is None else rows
    if n == 0:
        return
    d, k = data.d, cents.k
    st = stream_handle()
    xsq = data.norms(d)[row0:row0 + n]
    n_tiles = (k + 255) // 256  # ARGMIN tile width 256
    split = max(1, min(_l2_split(n, k, d, 4), n_tiles))
    split = -(-n_tiles // -(-n_tiles // split))  # the launcher's effective split (whole tile ranges)
    top = ws.top_records(split * n)
    _gemm(data.hi[row0:row0 + n], data.lo[row0:row0 + n], cents.hi, cents.lo, n, k, d, native.GEMM_ARGMIN,
          xsq=xsq, ysq=cents.ysq, top=top, n_split=split)
    assign, tau = ws.assign[row0:row0 + n], ws.tau[row0:row0 + n]
    ws.amb_count.zero_()
    native.call("skm_argmin_merge", ptr(top), split, n, ptr(xsq), ptr(cents.ysq_max), float(tc_kappa(d, GATE_KPAIR)),
                ptr(assign), ptr(tau), ptr(ws.amb_rows), ptr(ws.amb_count), st)
    native.call("skm_exact_pair_dist", ptr(data.x[row0:row0 + n]), data.ld, ptr(cents.c), cents.ld, ptr(assign), n,
                d, ptr(xsq), ptr(cents.ysq), ws.chain_flavour, ws.chain_q, ptr(tau), st, nbytes=4.0 * n * d)
    n_amb = int(ws.amb_count.item())
    if n_amb:
        resolve_ambiguous_argmin(data, cents, ws, ws.amb_rows[:n_amb], row0, xsq)


def resolve_ambiguous_argmin(data: DeviceData, cents: Centroids, ws: Workspace, rows_local: torch.Tensor, row0: int,
                             xsq: torch.Tensor) -> None:
    """Rows whose runner-up lies within the error bound of the best: a tensor-core GATE pass over
    just these rows lists every column whose exact distance may tie or beat the best (typically
    2-4), and the reference's chain distance of each decides (lowest column on ties).  Rows with
    more candidates than the slab holds take the whole chain-GEMM distance row."""
    st = stream_handle()
    d, k = data.d, cents.k
    kap = tc_kappa(d, GATE_KPAIR)
    xsq_all = data.norms(d)
    glob_all = (rows_local + row0).to(torch.int32)
    for c0 in range(0, int(glob_all.numel()), ws.batch):
        glob = glob_all[c0:c0 + ws.batch].contiguous()
        m = int(glob.numel())
        thr, xs = ws.bthr[:m], ws.bx[:m]
        native.call("skm_argmin_candidates", ptr(glob), m, ptr(ws.tau), ptr(xsq_all), ptr(cents.ysq_max),
                    float(kap), ptr(thr), ptr(xs), st)
        xa_hi = torch.empty((m, data.ld), dtype=torch.float32, device=data.x.device)
        xa_lo = torch.empty_like(xa_hi)
        native.call("skm_gather_rows_i32", ptr(data.hi), data.ld, ptr(glob), m, data.ld, ptr(xa_hi), data.ld, st)
        native.call("skm_gather_rows_i32", ptr(data.lo), data.ld, ptr(glob), m, data.ld, ptr(xa_lo), data.ld, st)
        _gemm(xa_hi, xa_lo, cents.hi, cents.lo, m, k, d, native.GEMM_GATE, xsq=xs, ysq=cents.ysq, thr=thr,
              cand=ws.cand, cand_cnt=ws.cand_cnt, cand_cap=ws.cap)
        native.call("skm_cand_exact_argmin", ptr(glob), m, ptr(ws.cand), ptr(ws.cand_cnt), ws.cap, ptr(data.x),
                    data.ld, ptr(cents.c), cents.ld, d, ptr(xsq_all), ptr(cents.ysq), ws.chain_flavour,
                    ws.chain_q, ptr(ws.assign), ptr(ws.tau), st)
        over = torch.nonzero(ws.cand_cnt[:m] > ws.cap).flatten()
        if over.numel():
            exact_rows_argmin(data, cents, ws, (glob[over] - row0).to(torch.int32), row0, xsq)


def exact_rows_argmin(data: DeviceData, cents: Centroids, ws: Workspace, rows_local: torch.Tensor, row0: int,
                      xsq: torch.Tensor) -> None:
    """Full chain-GEMM distance rows (the reference's bits) + exact argmin for the given rows
    (indices relative to row0)."""
    dev = data.x.device
    st = stream_handle()
    d, k = data.d, cents.k
    m = int(rows_local.numel())
    chunk = max(1, min(m, (1 << 28) // max(k, 1)))  # <= 1 GiB of distances per chunk
    for c0 in range(0, m, chunk):
        cn = min(chunk, m - c0)
        ids = rows_local[c0:c0 + cn]
        glob = (ids + row0).contiguous()
        xa = torch.empty((cn, data.ld), dtype=torch.float32, device=dev)
        native.call("skm_gather_rows_i32", ptr(data.x), data.ld, ptr(glob), cn, data.ld, ptr(xa), data.ld, st)
        xs = xsq[ids.to(torch.int64)].contiguous()
        dense = torch.empty((cn, padded_ld(k)), dtype=torch.float32, device=dev)
        chain_gemm(xa, cents.c, cn, k, d, dense, ws.chain_flavour, ws.chain_q, xsq=xs, ysq=cents.ysq)
        native.call("skm_dense_argmin", ptr(dense), dense.stride(0), cn, k, ptr(ids), ptr(ws.assign[row0:]),
                    ptr(ws.tau[row0:]), st)


SCAN_TAIL_BLOCKS_MAX = 432  # csrc/scan.cuh SCAN_NB_MAX_WIDE (the one-warp instantiation)


class PrunePlan:
    """Per-iteration constants of the pruned pass at a given d'."""

    def __init__(self, d: int, d_prime: int, eps0: float, sentinel: bool, dev):
        widths, bounds = tail_block_layout(d, d_prime)
        f = threshold_factors(d, d_prime, bounds, eps0)
        self.factors = f
        self.gate = sentinel_factors(f) if sentinel else f
        self.widths = widths
        self.nb = len(widths)
        if self.nb > SCAN_TAIL_BLOCKS_MAX:
            from .config import SuperKMeansError
            raise SuperKMeansError(
                f"tail of {d - d_prime} dims ({self.nb} blocks of 64) exceeds the device scan's "
                f"{SCAN_TAIL_BLOCKS_MAX} blocks (d - d' <= {64 * SCAN_TAIL_BLOCKS_MAX})")
        self.d_prime = d_prime
        self.sentinel = sentinel
        key = (str(dev), d, d_prime, float(eps0), bool(sentinel))
        cached = _PLAN_TENSORS.get(key)
        if cached is None:  # device copies of the constants, uploaded once per (d, d', mode)
            cached = (torch.tensor(self.gate, dtype=torch.float32, device=dev),
                      torch.tensor(widths, dtype=torch.int32, device=dev))
            if len(_PLAN_TENSORS) > 256:
                _PLAN_TENSORS.clear()
            _PLAN_TENSORS[key] = cached
        self.theta, self.bdims = cached


_PLAN_TENSORS: dict = {}


def pruned_assign_pass(data: DeviceData, cents: Centroids, ws: Workspace, plan: PrunePlan, seed_tau: bool = True,
                       row0: int = 0, rows: int | None = None, order: torch.Tensor | None = None):
    """Seed tau, gate GEMM -> candidate lists, exact scan.  Accumulates ws.counters =
    {survivors, tail dims touched, changed}.

    With ``order`` (rows sorted by their previous assignment, from the last update) batches
    follow that order: the gate GEMM reads gathered front rows, and concurrently running scan
    warps then work on rows of the same/neighbouring clusters, whose candidate centroid tails
    are shared in L1/L2.  Results do not depend on the order (rows are independent)."""
    n = data.n if rows is None else rows
    if n == 0:
        return
    d, dp = data.d, plan.d_prime
    st = stream_handle()
    x_rows = data.x[row0:row0 + n]
    tau = ws.tau[row0:row0 + n]
    assign = ws.assign[row0:row0 + n]
    if plan.sentinel:
        native.call("skm_fill_f32", ptr(tau), n, float("inf"), st)
    elif seed_tau:
        native.call("skm_seed_thresholds", ptr(x_rows), data.ld, ptr(cents.c), cents.ld, ptr(assign), n, d,
                    ptr(tau), st, nbytes=4.0 * n * d + 8.0 * n)
    xsq = data.norms(dp)
    kap = tc_kappa(dp, GATE_KPAIR)
    # emission threshold of the tensor-core gate: a superset of the candidates whose exact
    # (chain) distance may pass fl(tau F0); the scan settles every decision exactly
    native.call("skm_gate_threshold", ptr(tau), n, float(plan.gate[0]), int(plan.sentinel),
                ptr(ws.thr[row0:row0 + n]), ptr(xsq[row0:row0 + n]), ptr(cents.ysq_max), float(kap), st)
    cx = cert_extension(data, cents, plan, tau, ws.thr1[row0:row0 + n], n, ws.nowin and seed_tau)
    ext = cx.get("ext_k", 0)
    xsq_ext = cx.get("xsq_ext")
    # full-d certificate: the certified entries leave the in-order scan (DEFER_CERT)
    defer = DEFER_CERT and cx.get("nowin", False) and not ws.flat
    if defer:
        tau_seed, skip, imp, imp_cnt = ws.defer_buffers()
        tau_seed[row0:row0 + n].copy_(tau)
    k = cents.k
    ordered = order is not None and row0 == 0 and n == data.n
    if ordered:
        fld = padded_ld(dp + ext)
        ga_hi, ga_lo = ws.front_buffers(fld)
    for b0 in range(0, n, ws.batch):
        bn = min(ws.batch, n - b0)
        r = row0 + b0
        sp = native.ScanParams()
        if ordered:
            rmap = order[b0:b0 + bn]
            # the front buffers may be wider than fld (allocated at a larger d'): use their stride
            native.call("skm_gather_front", ptr(data.hi), ptr(data.lo), data.ld, ptr(rmap), bn, dp + ext, ptr(ga_hi),
                        ptr(ga_lo), ga_hi.stride(0), ptr(xsq), ptr(ws.thr), ptr(ws.bx), ptr(ws.bthr),
                        ptr(xsq_ext) if ext else None, ptr(ws.thr1) if ext else None,
                        ptr(ws.bx_ext) if ext else None, ptr(ws.bthr1) if ext else None, st,
                        nbytes=16.0 * bn * (dp + ext) + 24.0 * bn)
            cert = dict(cx, xsq_ext=ws.bx_ext[:bn], thr1=ws.bthr1[:bn]) if ext else {}
            _gemm(ga_hi[:bn], ga_lo[:bn], cents.hi, cents.lo, bn, k, dp, native.GEMM_GATE, xsq=ws.bx[:bn],
                  ysq=cents.ysq, thr=ws.bthr[:bn], cand=ws.cand, cand_cnt=ws.cand_cnt,
                  cand_cap=ws.cap, **cert)
            sp.row_map = rmap.data_ptr()
        else:
            cert = dict(cx, xsq_ext=xsq_ext[r:r + bn], thr1=ws.thr1[r:r + bn]) if ext else {}
            _gemm(data.hi[r:r + bn], data.lo[r:r + bn], cents.hi, cents.lo, bn, k, dp, native.GEMM_GATE,
                  xsq=xsq[r:r + bn], ysq=cents.ysq, thr=ws.thr[r:r + bn], cand=ws.cand,
                  cand_cnt=ws.cand_cnt, cand_cap=ws.cap, **cert)
        sp.cand, sp.cand_cnt, sp.cap = ws.cand.data_ptr(), ws.cand_cnt.data_ptr(), ws.cap
        sp.k, sp.n_rows, sp.row0 = k, bn, r
        sp.work = ws.work.data_ptr()
        sp.x, sp.ldx = data.x.data_ptr(), data.ld
        sp.tails, sp.nb, sp.d_prime = cents.tails.data_ptr(), plan.nb, dp
        sp.theta, sp.block_dims = plan.theta.data_ptr(), plan.bdims.data_ptr()
        sp.tau, sp.assign, sp.counters = ws.tau.data_ptr(), ws.assign.data_ptr(), ws.counters.data_ptr()
        sp.counters_ext = ws.diag.data_ptr()
        if PRUNE_HIST is not None:
            sp.prune_hist = PRUNE_HIST.data_ptr()
        _scan_exact_args(sp, data, cents, ws, xsq, kap, plan.sentinel)
        if defer:
            native.call("skm_defer_cert_flags", ptr(ws.cand), ptr(ws.cand_cnt), ws.cap, bn, ptr(skip), st)
            sp.skip_cert, sp.imp, sp.imp_cnt = skip.data_ptr(), imp.data_ptr(), imp_cnt.data_ptr()
        native.call("skm_pruned_scan", C.byref(sp), st, tag="pruned_scan", nbytes=4.0 * bn * (d - dp) + 16.0 * bn)
        if defer:
            native.call("skm_deferred_cert_count", C.byref(sp), ptr(tau_seed), st)
        if ws.cap < k:
            # rows whose candidate list overflowed the slab: dense distance rows, same kernel
            over = torch.nonzero(ws.cand_cnt[:bn] > ws.cap).flatten()
            n_over = int(over.numel())
            if n_over:
                gl = (order[b0:b0 + bn][over] if ordered else over + r).to(torch.int64)
                _dense_overflow(data, cents, ws, plan, gl, n_over, xsq)


def _dense_overflow(data, cents, ws, plan, glob_rows, n_over, xsq):
    """Rows with more gate candidates than the slab holds: full partial-distance rows from the
    same GEMM (bit-identical values), then the scan in dense mode."""
    dev = data.x.device
    st = stream_handle()
    idx = glob_rows.to(torch.int64).contiguous()
    a_hi = torch.empty((n_over, data.ld), dtype=torch.float32, device=dev)
    a_lo = torch.empty_like(a_hi)
    xs = torch.empty(n_over, dtype=torch.float32, device=dev)
    native.call("skm_gather_rows", ptr(data.hi), data.ld, ptr(idx), n_over, data.ld, ptr(a_hi), data.ld, st)
    native.call("skm_gather_rows", ptr(data.lo), data.ld, ptr(idx), n_over, data.ld, ptr(a_lo), data.ld, st)
    native.call("skm_gather_rows", ptr(xsq.view(-1, 1)), 1, ptr(idx), n_over, 1, ptr(xs.view(-1, 1)), 1, st)
    k = cents.k
    chunk = max(1, min(n_over, (1 << 28) // max(k, 1)))  # bound the dense buffer (1 GiB)
    rmap_all = idx.to(torch.int32)
    for c0 in range(0, n_over, chunk):
        cn = min(chunk, n_over - c0)
        dense = torch.empty((cn, padded_ld(k)), dtype=torch.float32, device=dev)
        _gemm(a_hi[c0:c0 + cn], a_lo[c0:c0 + cn], cents.hi, cents.lo, cn, k, plan.d_prime, native.GEMM_DIST,
              out=dense, xsq=xs[c0:c0 + cn], ysq=cents.ysq, n_split=_n_split(cn, k))
        ident = torch.arange(cn, dtype=torch.int32, device=dev)
        sp = native.ScanParams()
        sp.dense, sp.ld_dense, sp.dense_row, sp.k = dense.data_ptr(), dense.stride(0), ident.data_ptr(), k
        sp.n_rows, sp.row0 = cn, 0
        sp.row_map = rmap_all[c0:c0 + cn].data_ptr()
        sp.work = ws.work.data_ptr()
        sp.x, sp.ldx = data.x.data_ptr(), data.ld
        sp.tails, sp.nb, sp.d_prime = cents.tails.data_ptr(), plan.nb, plan.d_prime
        sp.theta, sp.block_dims = plan.theta.data_ptr(), plan.bdims.data_ptr()
        sp.tau, sp.assign, sp.counters = ws.tau.data_ptr(), ws.assign.data_ptr(), ws.counters.data_ptr()
        sp.dense_mode = 1
        _scan_exact_args(sp, data, cents, ws, xsq, tc_kappa(plan.d_prime, GATE_KPAIR))
        native.call("skm_pruned_scan", C.byref(sp), st, tag="pruned_scan_dense", nbytes=4.0 * cn * k)


def _scan_exact_args(sp, data: DeviceData, cents: Centroids, ws: Workspace, xsq: torch.Tensor, kap: float,
                     sentinel: bool = False) -> None:
    """Interval decisions on tensor-core distances + the exact chain for the unsettled ones."""
    if SCAN_FLAT and ws.flat and not sentinel:
        sp.flat, sp.fb_rows, sp.fb_count = 1, ws.fb_rows.data_ptr(), ws.fb_count.data_ptr()
    sp.kap = kap
    sp.xsq, sp.ysq, sp.ysq_max = xsq.data_ptr(), cents.ysq.data_ptr(), cents.ysq_max.data_ptr()
    sp.cent, sp.ldc = cents.c.data_ptr(), cents.ld
    sp.chain_flavour, sp.chain_q = ws.chain_flavour, ws.chain_q


def update_centroids_device(data: DeviceData, cents: Centroids, ws: Workspace, comm: Comm,
                            sums_buf: torch.Tensor | None = None, sorted_counts: np.ndarray | None = None
                            ) -> np.ndarray:
    """One-GPU update: mean of member rows (f64 ordered sums, bitwise the reference's serial loop),
    empties keep their previous centroid.  Returns host int64 counts.  ``sorted_counts``: the
    cluster sort already ran (ws.order / counts / offsets current) and these are its counts.
    (Multi-GPU updates go through Reducer, inside the iteration's one allreduce.)"""
    st = stream_handle()
    k, d = cents.k, cents.d
    if comm.world > 1:
        raise RuntimeError("update_centroids_device is the 1-GPU update; sharded loops use Reducer")
    if sorted_counts is None:
        native.call("skm_cluster_sort", ptr(ws.assign), data.n, k, ptr(ws.order), ptr(ws.counts), ptr(ws.offsets),
                    ptr(ws.sort_ws), ws.sort_ws.numel(), st, nbytes=32.0 * data.n)
    native.call("skm_cluster_sums", ptr(data.x), data.ld, ptr(ws.order), ptr(ws.offsets), ptr(ws.counts), k, d,
                None, 0, ptr(cents.c), cents.ld, 0, st, nbytes=4.0 * data.n * d + 4.0 * k * d)
    return sorted_counts if sorted_counts is not None else ws.counts.cpu().numpy().astype(np.int64)


def apply_splits_device(cents: Centroids, counts: np.ndarray, rng) -> int:
    empties, donors = plan_splits(counts, rng)
    if not empties:
        return 0
    dev = cents.c.device
    e = torch.tensor(empties, dtype=torch.int32, device=dev)
    dn = torch.tensor(donors, dtype=torch.int32, device=dev)
    native.call("skm_apply_splits", ptr(cents.c), cents.ld, cents.d, ptr(e), ptr(dn), len(empties),
                float(SPLIT_EPS), stream_handle())
    return len(empties)


def assign_stats(ws: Workspace, n: int, with_prev: bool) -> None:
    native.call("skm_assign_stats", ptr(ws.tau), ptr(ws.assign), ptr(ws.prev) if with_prev else None, n,
                ptr(ws.wcss), ptr(ws.changed), ptr(ws.stats_ws), ws.stats_ws.numel(), stream_handle())


# ------------------------------------------------------------------------------ multi-GPU reduction
class Reducer:
    """The iteration's only collective at N > 1: ONE allreduce(sum) of a packed f64 buffer
    [centroid sums k*d | counts k | n_changed, survivors, dims touched | tau buffer partials]
    (SURVEY.md 8e).  The update's sums are computed before the convergence test and dropped when
    the loop stops there (core.py:354-363).

    * tau buffer partials: NumPy sums tau in 8192-element buffers (core.py:344); shards start on
      buffer boundaries (shard_bounds), so each rank writes its buffers' pairwise sums into their
      global slots and the host adds the slots in order -- wcss is the 1-GPU (= reference) value.
    * exact=True: the f64 member sums are chained in rank order -- rank r continues rank r-1's
      running sums over its own members (rows are sharded in ascending order, so this is the
      reference's serial row order, _kernels.pyx:115-119) -- pipelined over cluster chunks with
      point-to-point sends; only the last rank's sums enter the allreduce (the others add 0.0,
      exact).  Centroids are then bitwise the 1-GPU result.  exact=False: each rank's sums start
      from 0 and the allreduce adds them (centroids equal up to f64 association)."""

    def __init__(self, comm: "Comm", k: int, d: int, n_global: int, row_lo: int, n_local: int, dev, exact: bool):
        self.comm, self.k, self.d, self.exact = comm, k, d, exact
        self.aligned = row_lo % SHARD_ALIGN == 0 and (n_local % SHARD_ALIGN == 0 or row_lo + n_local == n_global)
        self.n_chunks = -(-n_global // SHARD_ALIGN) if self.aligned else 1
        self.chunk0 = row_lo // SHARD_ALIGN if self.aligned else 0
        self.o_cnt = k * d
        self.o_scal = self.o_cnt + k
        self.o_tau = self.o_scal + 3
        self.o_gt = self.o_tau + self.n_chunks
        self.n_gt = 0
        self.gt_slots = self.gt_rows = self.gt_assign = None
        self.buf = torch.zeros(self.o_gt, dtype=torch.float64, device=dev)
        self.pin = torch.empty(self.o_gt - self.o_cnt, dtype=torch.float64, pin_memory=True)
        self.counts64 = torch.empty(k, dtype=torch.int64, device=dev)
        self.row_lo, self.n_local = row_lo, n_local

    def attach_etr(self, gt_idx: torch.Tensor, top_k: int) -> None:
        """ETR without a second collective: the assignments of the ground-truth rows (nq x top_k
        slots, each held by exactly one rank) ride in the iteration's allreduce, so every rank
        tallies every query's hits locally after the update (core.py:379-399)."""
        gi = gt_idx[:, :top_k].reshape(-1).to(torch.int64)
        mine = (gi >= self.row_lo) & (gi < self.row_lo + self.n_local)
        self.gt_slots = torch.nonzero(mine).flatten()
        self.gt_rows = gi[self.gt_slots] - self.row_lo
        self.n_gt = int(gi.numel())
        extra = torch.zeros(self.n_gt, dtype=torch.float64, device=self.buf.device)
        self.buf = torch.cat([self.buf[:self.o_gt], extra])

    def reduce(self, data: "DeviceData", ws: "Workspace", n_local: int) -> tuple[np.ndarray, float, float, float, float]:
        """Local stats + sorted sums -> one allreduce -> (counts, wcss, n_changed, survivors, touched)."""
        st = stream_handle()
        k, d = self.k, self.d
        buf = self.buf
        buf[self.o_tau:].zero_()
        if self.aligned:
            nloc = max(n_local, 0)
            if nloc:
                native.call("skm_tau_chunk_sums", ptr(ws.tau), nloc, ptr(buf[self.o_tau + self.chunk0:]), st)
        else:
            buf[self.o_tau] = ws.wcss[0]
        buf[self.o_scal] = ws.changed[0].to(torch.float64)
        buf[self.o_scal + 1] = ws.counters[0].to(torch.float64)
        buf[self.o_scal + 2] = ws.counters[1].to(torch.float64)
        buf[self.o_cnt:self.o_scal].copy_(ws.counts.to(torch.float64))
        if self.n_gt:
            gt = buf[self.o_gt:]
            gt.zero_()
            gt[self.gt_slots] = ws.assign[self.gt_rows].to(torch.float64)
        sums = buf[:self.o_cnt]
        if self.exact and self.comm.world > 1:
            self._chained_sums(data, ws, sums)
        else:
            native.call("skm_cluster_sums", ptr(data.x), data.ld, ptr(ws.order), ptr(ws.offsets), ptr(ws.counts), k,
                        d, ptr(sums), 0, None, 0, 1, st, nbytes=4.0 * data.n * d)
        self.comm.allreduce_(buf)
        if self.n_gt:
            self.gt_assign = buf[self.o_gt:].to(torch.int32)  # every GT row's assignment, all ranks
        self.pin.copy_(buf[self.o_cnt:self.o_gt], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        h = self.pin.numpy()
        counts = np.rint(h[:k]).astype(np.int64)
        ch, sv, td = (float(v) for v in h[k:k + 3])
        wcss = 0.0
        for v in h[k + 3:]:  # NumPy's buffer order: bitwise the reference's np.sum
            wcss += float(v)
        return counts, wcss, ch, sv, td

    def finalize(self, cents: "Centroids", counts: np.ndarray) -> None:
        """centroid = f32(sum / count); empty clusters keep their previous row (core.py:93-99)."""
        self.counts64.copy_(torch.from_numpy(counts))
        native.call("skm_finalize_centroids", ptr(self.buf), ptr(self.counts64), self.k, self.d, ptr(cents.c),
                    cents.ld, stream_handle())

    def _chained_sums(self, data, ws, sums: torch.Tensor, chunks: int = 16) -> None:
        chained_cluster_sums(self.comm, data, ws, sums, self.k, self.d, chunks)


def chained_cluster_sums(comm: "Comm", data, ws, sums: torch.Tensor, k: int, d: int, chunks: int = 16) -> None:
    """Rank-order f64 member sums, pipelined over cluster chunks: receive rank r-1's running sums
    of a chunk, continue them over this rank's members (ascending, ws.order / offsets / counts),
    send them on; ranks before the last then hold zeros, so an allreduce(sum) of ``sums`` leaves
    the last rank's chain on every rank -- the reference's serial row order (_kernels.pyx:115-119)
    when ranks hold ascending row ranges."""
    r, w = comm.rank, comm.world
    st = stream_handle()
    step = -(-k // chunks)
    nccl = comm.dist.get_backend(comm.group) == "nccl"
    pending = []
    for c0 in range(0, k, step):
        c1 = min(k, c0 + step)
        seg = sums[c0 * d:c1 * d]
        if r > 0:
            if nccl:
                comm.dist.recv(seg, src=r - 1, group=comm.group)
            else:
                tmp = torch.empty(seg.shape, dtype=seg.dtype)
                comm.dist.recv(tmp, src=r - 1, group=comm.group)
                seg.copy_(tmp)
        native.call("skm_cluster_sums", ptr(data.x), data.ld, ptr(ws.order), ptr(ws.offsets[c0:]),
                    ptr(ws.counts[c0:]), c1 - c0, d, ptr(seg), int(r > 0), None, 0, 1, st,
                    nbytes=4.0 * data.n * d * (c1 - c0) / k)
        if r < w - 1:
            if nccl:
                pending.append(comm.dist.isend(seg, dst=r + 1, group=comm.group))
            else:
                comm.dist.send(seg.cpu(), dst=r + 1, group=comm.group)
    for p_ in pending:
        p_.wait()
    if r < w - 1:
        sums.zero_()


# ------------------------------------------------------------------------------ the loop
def sharded_init_rows(data: "DeviceData", k: int, init_idx: np.ndarray, row_lo: int, comm: Comm) -> torch.Tensor:
    """Forgy rows (k, ld) assembled across ranks: each rank fills the rows it owns (global
    indices in [row_lo, row_lo + n_local)) and one allreduce(sum) completes the replica."""
    dev = data.x.device
    rows = torch.zeros((k, data.ld), dtype=torch.float32, device=dev)
    mine = np.flatnonzero((init_idx >= row_lo) & (init_idx < row_lo + data.n))
    if mine.size:
        src = torch.tensor(init_idx[mine] - row_lo, dtype=torch.int64, device=dev)
        tmp = torch.empty((mine.size, data.ld), dtype=torch.float32, device=dev)
        native.call("skm_gather_rows", ptr(data.x), data.ld, ptr(src), int(mine.size), data.ld, ptr(tmp), data.ld,
                    stream_handle())
        rows[torch.tensor(mine, dtype=torch.int64, device=dev)] = tmp
    return comm.allreduce_(rows)


def fit_rotated_device(data: DeviceData, cfg: KMeansConfig, inspect=None, comm: Comm | None = None,
                       n_global: int | None = None, row_lo: int = 0, init_rows: torch.Tensor | None = None,
                       init_idx: np.ndarray | None = None, etr=None, timer: _Timer | None = None,
                       ws: Workspace | None = None, first_pass_done: bool = False) -> LoopOutput:
    """Device twin of core._fit_rotated.  ``data`` holds this rank's rows; ``n_global`` the
    total across ranks.  ``init_rows`` (k, ld) are the Forgy rows gathered from all ranks.
    Without ``comm`` the rows are one process's (sharding is explicit: pass ``Comm()``)."""
    comm = comm or Comm.local()
    dev = data.x.device
    n_local, d = data.n, data.d
    n = n_local if n_global is None else n_global
    k = cfg.k
    work = WorkCounters()
    timer = timer or _Timer()
    if init_idx is None:
        init_idx = init_indices(n, k, [cfg.seed, 2])
    if init_rows is None:
        idx = torch.tensor(init_idx, dtype=torch.int64, device=dev)
        init_rows = torch.zeros((k, data.ld), dtype=torch.float32, device=dev)
        native.call("skm_gather_rows", ptr(data.x), data.ld, ptr(idx), k, data.ld, ptr(init_rows), data.ld,
                    stream_handle())
    cents = Centroids(init_rows, d)
    ws = ws or Workspace(dev, n_local, k, d, cfg)
    rng_split = np.random.default_rng([cfg.seed, 3])
    pruned_mode = pruning_supported(d)
    d_prime = initial_d_prime(d, cfg.d_prime_init_fraction) if pruned_mode else None
    stats: list[IterationStats] = []
    recall_history: list[float] = []
    terminated = "max_iters"
    phase: dict[str, float] = {}
    if etr is not None:
        timer.start("ground_truth")
        etr.setup(data, comm, n_global=n, row_lo=row_lo)
        timer.stop("ground_truth")
    reducer = Reducer(comm, k, d, n, row_lo, n_local, dev, cfg.exact_reduce) if comm.world > 1 else None
    if reducer is not None and etr is not None:
        reducer.attach_etr(etr.gt_idx, etr.top_k)
    scal = torch.zeros(4, dtype=torch.float64, device=dev)
    pin_scal = torch.empty(4, dtype=torch.float64, pin_memory=True)
    pin_counts = torch.empty(k, dtype=torch.int32, pin_memory=True)
    have_order = False
    last_changed = None  # n_changed of the previous iteration (flat-scan policy)
    last_surv_row = None  # survivors per row of the previous pruned iteration (exact_work_stats policy)
    scan_blocks: list[int] = []
    scan_waves: list[int] = []
    scan_diag: list[list[int]] = []

    for it in range(1, cfg.max_iters + 1):
        pruned_iter = pruned_mode and it > 1
        d_used = d_prime if pruned_iter else None
        survivors = touched = 0
        prune_rate = None
        n_changed = None
        if it > 1:
            native.call("skm_copy_i32", ptr(ws.assign), ptr(ws.prev), n_local, stream_handle())
        if not pruned_iter:
            timer.start("gemm")
            if not (it == 1 and first_pass_done):  # else: ran on the unrotated rows (api.fit_device)
                cents.refresh(d, None)
                full_assign_pass(data, cents, ws)
            timer.stop("gemm")
            work.full_pair_dims += n * k * d
        else:
            plan = PrunePlan(d, d_prime, cfg.epsilon0, cfg.pruning_sentinel, dev)
            timer.start("pruning")
            cents.refresh(d_prime, d_prime)
            ws.counters.zero_()
            ws.diag.zero_()
            ws.flat = last_changed is not None and last_changed <= FLAT_MAX_CHANGED * n
            ws.nowin = (not cfg.exact_work_stats and not cfg.pruning_sentinel and not ws.flat
                        and (last_surv_row is None or last_surv_row > NOWIN_SURV_FRAC * k))
            pruned_assign_pass(data, cents, ws, plan, order=ws.order[:n_local] if have_order else None)
            timer.stop("pruning")
            work.front_pair_dims += n * k * d_prime
            if not cfg.pruning_sentinel:
                work.seed_dims += n * d
        assign_stats(ws, n_local, it > 1)
        # the update's stable cluster sort runs before the convergence test (it does not touch
        # the centroids, so a converged stop is unaffected); its counts come back with the scalars
        native.call("skm_cluster_sort", ptr(ws.assign), data.n, k, ptr(ws.order), ptr(ws.counts), ptr(ws.offsets),
                    ptr(ws.sort_ws), ws.sort_ws.numel(), stream_handle(), nbytes=32.0 * data.n)
        sorted_counts = None
        if reducer is None:
            # one host synchronisation per iteration
            scal[0] = ws.wcss[0]
            scal[1] = ws.changed[0].to(torch.float64)
            scal[2] = ws.counters[0].to(torch.float64)
            scal[3] = ws.counters[1].to(torch.float64)
            pin_scal.copy_(scal, non_blocking=True)
            pin_counts.copy_(ws.counts, non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()
            wcss, ch, sv, td = pin_scal.tolist()
            sorted_counts = pin_counts.numpy().astype(np.int64)
        else:
            # sums (computed before the convergence test, dropped if it stops the loop) + counts +
            # scalars + tau buffer partials: the iteration's one collective and one host sync
            sorted_counts, wcss, ch, sv, td = reducer.reduce(data, ws, n_local)
        if it > 1:
            n_changed = int(round(ch))
            last_changed = n_changed
        if pruned_iter:
            if COLLECT_DIAG:
                dg = ws.diag.tolist()
                scan_blocks.append(int(dg[0] + dg[2]))
                scan_waves.append(int(dg[1] + dg[3]))
                scan_diag.append([int(v) for v in dg[:6]])
            survivors, touched = int(round(sv)), int(round(td))
            prune_rate = prune_rate_from_totals(survivors, n, k)
            last_surv_row = survivors / max(n, 1)
            work.tail_dims += touched
        if inspect is not None:
            inspect(it, {
                "assignments": ws.assign[:n_local].cpu().numpy().copy(),
                "best_sq_dist": ws.tau[:n_local].cpu().numpy().copy(),
                "centroids_rotated": cents.c[:, :d].cpu().numpy().copy(),
                "d_prime": d_used,
                "prune_rate": prune_rate,
            })
        if n_changed == 0:
            stats.append(IterationStats(iter_index=it, wcss=wcss, n_empty_splits=0, prune_rate_after_gemm=prune_rate,
                                        d_prime=d_used, survivors=survivors, tail_dims_touched=touched,
                                        n_changed=n_changed, timings=timer.collect()))
            terminated = "converged"
            break
        timer.start("update")
        if reducer is None:
            counts = update_centroids_device(data, cents, ws, comm, sorted_counts=sorted_counts)
        else:
            reducer.finalize(cents, sorted_counts)
            counts = sorted_counts
        have_order = True  # ws.order now lists rows grouped by their current assignment
        n_splits = apply_splits_device(cents, counts, rng_split) if cfg.split_empty else 0
        timer.stop("update")
        if pruned_iter:
            d_prime = adjust_d_prime(d_prime, prune_rate, cfg, d)
        recall = None
        if etr is not None:
            timer.start("etr")
            recall = etr.probe(data, cents, ws, comm, gt_assign=reducer.gt_assign if reducer is not None else None)
            timer.stop("etr")
            recall_history.append(recall)
        stats.append(IterationStats(iter_index=it, wcss=wcss, n_empty_splits=n_splits,
                                    prune_rate_after_gemm=prune_rate, recall=recall, d_prime=d_used,
                                    survivors=survivors, tail_dims_touched=touched, n_changed=n_changed,
                                    timings=timer.collect()))
        if etr is not None and etr.should_stop(recall_history):
            terminated = "etr"
            break

    gt_time = 0.0
    for s in stats:
        gt_time += s.timings.pop("ground_truth", 0.0)
    if etr is not None:
        phase["ground_truth"] = gt_time
    for key in ("gemm", "pruning", "update", "etr"):
        phase[key] = sum(s.timings.get(key, 0.0) for s in stats)
    # results back through pinned buffers (one DMA each, one sync, no second host copy: the
    # arrays own the pinned storage)
    host_c = torch.empty((k, d), dtype=torch.float32, pin_memory=True)
    host_a = torch.empty(n_local, dtype=torch.int32, pin_memory=True)
    host_t = torch.empty(n_local, dtype=torch.float32, pin_memory=True)
    host_c.copy_(cents.c[:, :d], non_blocking=True)
    host_a.copy_(ws.assign[:n_local], non_blocking=True)
    host_t.copy_(ws.tau[:n_local], non_blocking=True)
    torch.cuda.current_stream(dev).synchronize()
    return LoopOutput(
        centroids_rotated=host_c.numpy(),
        assignments=host_a.numpy(),
        best_sq_dist=host_t.numpy(),
        stats=stats,
        terminated_by=terminated,
        d_prime_final=d_prime,
        init_indices=np.asarray(init_idx),
        work=work,
        recall_history=recall_history,
        phase_seconds=phase,
        centroids_dev=cents.c,
        assign_dev=ws.assign[:n_local],
        scan_blocks=scan_blocks,
        scan_waves=scan_waves,
        scan_diag=scan_diag,
    )

"""Drop-in public entry points: ``fit`` / ``final_assign`` / ``hierarchical_fit`` + result type.

Signatures, result fields and error behaviour follow the reference package
(``core.fit`` core.py:417-460, ``core.final_assign`` core.py:463-541, ``KMeansResult``
core.py:55-76, ``hierarchical_fit`` hierarchical.py:91-171).  Inputs are host NumPy (copied to
HBM once); outputs are freshly owned host NumPy arrays.  Everything between runs on the B200.
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
    NonFiniteValue,
    KMeansConfig,
    DimensionMismatch,
    RotationMatrix,
    WorkCounters,
    pruning_supported,
    validate_vector_set,
)
from .device import on_device, padded_ld, ptr, require_cuda, stream_handle, to_host
from .engine import (
    Centroids,
    Comm,
    DeviceData,
    PrunePlan,
    Workspace,
    _gemm,
    _Timer,
    fit_rotated_device,
    full_assign_pass,
    pruned_assign_pass,
)
from .hostmath import generate_rotation, sample_indices


@dataclass
class KMeansResult:
    centroids: np.ndarray
    assignments: np.ndarray
    stats: list
    terminated_by: str
    rotation: RotationMatrix
    centroids_rotated: np.ndarray
    d_prime_final: int | None
    sample_indices: np.ndarray | None
    init_indices: np.ndarray
    work: WorkCounters
    phase_seconds: dict
    peak_aux_values: int
    n_train: int
    recall_history: list = field(default_factory=list)

    @property
    def k(self) -> int:
        return self.centroids.shape[0]


# ------------------------------------------------------------------------------ rotation
class DeviceRotation:
    """R resident on device in both operand orientations; X.R and C.R^T as the exact fma chain of
    OpenBLAS's threaded sgemm (preprocess.py:37-52; csrc/sgemm_chain.cuh), so the rotated rows --
    which every later value of the loop depends on -- are bitwise the reference's.

    ``SKM_FAST_ROTATION=1`` selects the 3xTF32 tensor-core GEMM instead (~4x faster, rows differ
    from the reference at the ulp level; for timing comparisons only)."""

    FAST = os.environ.get("SKM_FAST_ROTATION", "0") == "1"

    def __init__(self, rotation: RotationMatrix, dev):
        d = rotation.dim
        self.d = d
        ld = padded_ld(d)
        r = torch.zeros((d, ld), dtype=torch.float32, device=dev)
        r[:, :d].copy_(torch.from_numpy(np.ascontiguousarray(rotation.data, dtype=np.float32)))  # one upload
        rt = torch.zeros((d, ld), dtype=torch.float32, device=dev)
        rt[:, :d] = r[:, :d].t()  # transposed on the device
        self.r, self.rt = r, rt   # rows of R -> X @ R^T (unrotate); rows of R^T -> X @ R (rotate)
        if self.FAST:
            self.r_hi, self.r_lo = _split(r, d)
            self.rt_hi, self.rt_lo = _split(rt, d)

    def apply(self, x_dev: torch.Tensor, out: torch.Tensor | None = None, inverse: bool = False,
              inplace: bool = False, chunk_rows: int = 1 << 20) -> torch.Tensor:
        """out = x @ R (or x @ R^T); x_dev (n, ld) padded.  ``inplace`` writes the result over the
        input rows, one row chunk at a time through a chunk-sized buffer (the GEMM reads a whole
        row tile while other CTAs write, so it never runs in place)."""
        from .engine import GEMM_Q, chain_gemm
        n = x_dev.shape[0]
        if inplace:
            out = x_dev
        elif out is None:
            out = torch.zeros((n, padded_ld(self.d)), dtype=torch.float32, device=x_dev.device)
        if n == 0:
            return out
        tmp = torch.empty((min(n, chunk_rows), out.shape[1]), dtype=torch.float32, device=x_dev.device) \
            if inplace else None
        for r0 in range(0, n, chunk_rows):
            m = min(chunk_rows, n - r0)
            dst = tmp[:m] if inplace else out[r0:r0 + m]
            if self.FAST:
                b_hi, b_lo = (self.r_hi, self.r_lo) if inverse else (self.rt_hi, self.rt_lo)
                x_hi, x_lo = x_dev[r0:r0 + m], _split_lo(x_dev[r0:r0 + m], self.d)
                _gemm(x_hi, x_lo, b_hi, b_lo, m, self.d, self.d, native.GEMM_STORE, out=dst,
                      n_split=_store_split(m, self.d))
                del x_lo
            else:
                # k-major operand: x @ R reads R's rows, x @ R^T the rows of R^T
                chain_gemm(x_dev[r0:r0 + m], self.rt if inverse else self.r, m, self.d, self.d, dst, 0, GEMM_Q,
                           b_kmajor=True)
            if inplace:
                out[r0:r0 + m].copy_(dst)
        return out


def _store_split(m, n):
    from .engine import _l2_split
    return _l2_split(m, n, n, 6)


def _split_lo(x: torch.Tensor, cols: int) -> torch.Tensor:
    lo = torch.empty_like(x)
    native.call("skm_split_hilo", ptr(x), x.shape[1], x.shape[0], cols, None, ptr(lo), x.shape[1], stream_handle())
    return lo


def _split(x: torch.Tensor, cols: int):
    hi = torch.empty_like(x)
    lo = torch.empty_like(x)
    native.call("skm_split_hilo", ptr(x), x.shape[1], x.shape[0], cols, ptr(hi), ptr(lo), x.shape[1],
                stream_handle())
    return hi, lo


_STAGE_BYTES = 256 << 20  # pinned staging chunk
_STAGE_THREADS = int(os.environ.get("SKM_H2D_THREADS", max(1, min(8, os.cpu_count() or 1))))  # 1: plain copy
_stage_pool = None


def _copy_rows_to_device(x: np.ndarray, out: torch.Tensor, d: int, idx: np.ndarray | None = None) -> None:
    """out[:, :d] = x (or x[idx], a row gather) for a pageable host matrix.  A plain pageable
    copy runs at ~11 GB/s on the B200 hosts (one driver thread staging through its own bounce
    buffer); here the host copy (or gather) into pinned chunks is split over a few threads and
    overlapped with the DMA of the previous chunk (three-chunk ring), ~50 GB/s
    (tools/h2d_probe.py)."""
    global _stage_pool
    n = x.shape[0] if idx is None else idx.shape[0]
    if n * d * 4 <= 2 * _STAGE_BYTES or _STAGE_THREADS == 1:
        out[:, :d].copy_(torch.from_numpy(x if idx is None else x[idx]))
        return
    if _stage_pool is None:
        from concurrent.futures import ThreadPoolExecutor
        _stage_pool = ThreadPoolExecutor(_STAGE_THREADS, thread_name_prefix="skm-h2d")
    rows = max(1, _STAGE_BYTES // (4 * d))
    bufs = [torch.empty((rows, d), dtype=torch.float32, pin_memory=True) for _ in range(3)]
    done = [None] * 3
    stream = torch.cuda.current_stream(out.device)
    for i, r0 in enumerate(range(0, n, rows)):
        b = i % 3
        if done[b] is not None:
            done[b].synchronize()  # the DMA that last read this chunk has finished
        nb = min(rows, n - r0)
        view = bufs[b].numpy()[:nb]
        step = -(-nb // _STAGE_THREADS)
        if idx is None:
            list(_stage_pool.map(lambda j: np.copyto(view[j:min(j + step, nb)], x[r0 + j:r0 + min(j + step, nb)]),
                                 range(0, nb, step)))
        else:  # np.take releases the GIL; mode="clip" writes straight into the pinned view
            list(_stage_pool.map(lambda j: np.take(x, idx[r0 + j:r0 + min(j + step, nb)], axis=0,
                                                   out=view[j:min(j + step, nb)], mode="clip"),
                                 range(0, nb, step)))
        out[r0:r0 + nb, :d].copy_(bufs[b][:nb], non_blocking=True)
        done[b] = torch.cuda.Event()
        done[b].record(stream)
    for e in done:
        if e is not None:
            e.synchronize()  # the ring is released when the function returns


def _pinned_source(x) -> torch.Tensor | None:
    """A 2-D float32 C-contiguous CPU tensor in pinned memory can be copied by one DMA."""
    if isinstance(x, torch.Tensor) and x.device.type == "cpu" and x.dim() == 2 and x.dtype == torch.float32 \
            and x.is_contiguous() and x.is_pinned():
        return x
    return None


def _h2d(x: np.ndarray, dev, check_finite: bool = False, idx: np.ndarray | None = None,
         src: torch.Tensor | None = None) -> torch.Tensor:
    """(n, ld) device copy of x (or of the rows x[idx]) with zero pad columns.  ``check_finite``:
    validate_vector_set's NaN/Inf check (model.py:84-87) on the device after the copy -- the
    host scan costs ~0.3 s per GB, more than the fit -- raising the same NonFiniteValue(first
    row, col) (row numbered within the copied rows)."""
    n = x.shape[0] if idx is None else idx.shape[0]
    d = x.shape[1]
    out = torch.zeros((n, padded_ld(d)), dtype=torch.float32, device=dev)
    if n:
        if src is not None and idx is None:
            out[:, :d].copy_(src, non_blocking=True)  # pinned host rows: one DMA
        else:
            _copy_rows_to_device(x, out, d, idx)
        if check_finite:
            first = torch.empty(1, dtype=torch.int64, device=dev)
            native.call("skm_first_nonfinite", ptr(out), out.shape[1], n, d, ptr(first), stream_handle())
            f = int(first.cpu().numpy().view(np.uint64)[0])
            if f != (1 << 64) - 1:
                from .config import NonFiniteValue
                raise NonFiniteValue(f // d, f % d)
    return out


def _nonfinite_key(out: torch.Tensor, n: int, d: int) -> int:
    """Flat index row * d + col of the first NaN/Inf of a padded device matrix, 2^64 - 1 if none."""
    if n == 0:
        return (1 << 64) - 1
    first = torch.empty(1, dtype=torch.int64, device=out.device)
    native.call("skm_first_nonfinite", ptr(out), out.shape[1], n, d, ptr(first), stream_handle())
    return int(first.cpu().numpy().view(np.uint64)[0])


def _check_finite_sharded(x: np.ndarray, dev, row_offset: int, comm, chunk_rows: int = 1 << 18) -> None:
    """validate_vector_set's finiteness check of a row-sharded host matrix: every rank scans its
    rows [row_offset, row_offset + len(x)) on the device, one allreduce(min) of the first bad
    flat index, and every rank raises the same NonFiniteValue(row, col) (no rank is left
    waiting in a collective)."""
    n, d = x.shape
    key = (1 << 64) - 1
    for r0 in range(0, n, chunk_rows):
        k = _nonfinite_key(_h2d(x[r0:r0 + chunk_rows], dev), min(chunk_rows, n - r0), d)
        if k != (1 << 64) - 1:
            key = (row_offset + r0) * d + k
            break
    t = torch.tensor([min(key, (1 << 63) - 1)], dtype=torch.int64, device=dev)
    comm.allreduce_min_(t)
    g = int(t.item())
    if g != (1 << 63) - 1:
        from .config import NonFiniteValue
        raise NonFiniteValue(g // d, g % d)


def _h2d_check_only(x: np.ndarray, dev, chunk_rows: int = 1 << 18) -> None:
    """Finiteness of a host matrix checked on the device chunk by chunk (bounded memory)."""
    for r0 in range(0, x.shape[0], chunk_rows):
        try:
            _h2d(x[r0:r0 + chunk_rows], dev, check_finite=True)
        except Exception as e:  # re-base the row of the first bad value
            from .config import NonFiniteValue
            if isinstance(e, NonFiniteValue):
                raise NonFiniteValue(e.row + r0, e.col) from None
            raise


class _FiniteCheckJob:
    """validate_vector_set's whole-input NaN/Inf check run on a host thread + its own CUDA
    stream while the caller works on a sample; ``result()`` re-raises the first
    NonFiniteValue(row, col) in row order, exactly the error the up-front check would give."""

    def __init__(self, x: np.ndarray, dev):
        import threading
        self.error = None
        stream = torch.cuda.Stream(dev)

        def run():
            try:
                with torch.cuda.stream(stream):
                    _h2d_check_only(x, dev)
            except BaseException as e:  # surfaced in result()
                self.error = e

        self.thread = threading.Thread(target=run, daemon=True)
        self.thread.start()

    def result(self) -> None:
        self.thread.join()
        if self.error is not None:
            raise self.error


def _prefetch_batches(x: np.ndarray, batch_rows: int, dev):
    """Yield (s0, e0, device rows) for consecutive row batches of a host matrix; batch i + 1 is
    staged (threaded pinned ring, own CUDA stream) while the caller computes on batch i.  The
    main stream waits on each batch's copy event; at most three batches are resident."""
    import queue
    import threading
    n = x.shape[0]
    q: queue.Queue = queue.Queue(maxsize=1)
    stop = threading.Event()
    stream = torch.cuda.Stream(dev)

    def put(item) -> bool:
        while not stop.is_set():
            try:
                q.put(item, timeout=0.05)
                return True
            except queue.Full:
                continue
        return False

    def work():
        try:
            with torch.cuda.stream(stream):
                for s0 in range(0, n, batch_rows):
                    e0 = min(n, s0 + batch_rows)
                    xb = _h2d(x[s0:e0], dev)
                    ev = torch.cuda.Event()
                    ev.record(stream)
                    if not put((s0, e0, xb, ev)):
                        return
        except BaseException as e:  # surfaced on the consumer side
            put(e)
            return
        put(None)

    t = threading.Thread(target=work, daemon=True)
    t.start()
    main = torch.cuda.current_stream(dev)
    try:
        while True:
            item = q.get()
            if item is None:
                break
            if isinstance(item, BaseException):
                raise item
            s0, e0, xb, ev = item
            main.wait_event(ev)
            xb.record_stream(main)
            yield s0, e0, xb
    finally:
        stop.set()
        t.join()


def _device_bytes_values(*ts) -> int:
    return int(sum(t.numel() * t.element_size() for t in ts if t is not None) // 4)


# ------------------------------------------------------------------------------ fit
class _RotationJob:
    """Host QR of the rotation (LAPACK releases the GIL) overlapped with the H2D copy."""

    def __init__(self, d: int, seed: int):
        import threading
        self.result = None
        self.error = None
        self.t0 = time.perf_counter()
        self.seconds = 0.0

        def run():
            try:
                self.result = generate_rotation(d, seed)
            except BaseException as e:  # pragma: no cover - surfaced in get()
                self.error = e
            self.seconds = time.perf_counter() - self.t0

        self.thread = threading.Thread(target=run, daemon=True)
        self.thread.start()

    def get(self) -> RotationMatrix:
        self.thread.join()
        if self.error is not None:
            raise self.error
        return self.result


@dataclass
class DeviceFit:
    """Output of the device-resident fit: loop output + device centroids (original space)."""
    loop: object
    rotation: RotationMatrix
    centroids_dev: torch.Tensor      # (k, ld) original space
    data: DeviceData
    phase: dict


def fit_device(x_dev: torch.Tensor, d: int, cfg: KMeansConfig, rotation: RotationMatrix, inspect=None,
               comm: Comm | None = None, n_global: int | None = None, row_lo: int = 0, keep_data: bool = False,
               init_rows: torch.Tensor | None = None, consume_input: bool = False) -> DeviceFit:
    """The hot path with inputs already in HBM: exact-chain rotation, Lloyd loop, un-rotation.

    ``x_dev`` is this rank's (n_local, ld) shard (pad columns zero); with ``comm.world > 1``
    (pass ``comm=Comm()`` under torch.distributed, plus ``n_global`` / ``row_lo``) the Forgy rows
    are assembled across ranks by one allreduce.  Without ``comm`` the rows are one process's."""
    comm = comm or Comm.local()
    dev = x_dev.device
    timer = _Timer()
    ws = None
    if isinstance(rotation, _RotationJob):
        rotation = rotation.get()  # the host QR ran beside the H2D copy
    timer.start("rotation")
    rot = DeviceRotation(rotation, dev)
    xr = rot.apply(x_dev, inplace=consume_input)  # consume_input: x_dev is a private copy
    data = DeviceData(xr, d)
    timer.stop("rotation")
    n_local = data.n
    n = n_local if n_global is None else n_global
    from .hostmath import init_indices
    init_idx = init_indices(n, cfg.k, [cfg.seed, 2])
    if init_rows is None and comm.world > 1:
        from .engine import sharded_init_rows
        init_rows = sharded_init_rows(data, cfg.k, init_idx, row_lo, comm)
    etr = None
    if cfg.etr is not None:
        from .etr import EtrState
        etr = EtrState(cfg)
    phase = dict(timer.collect())
    out = fit_rotated_device(data, cfg, inspect=inspect, comm=comm, n_global=n, row_lo=row_lo, init_rows=init_rows,
                             init_idx=init_idx, etr=etr, timer=timer, ws=ws)
    for key, v in out.phase_seconds.items():
        phase[key] = phase.get(key, 0.0) + v
    timer.start("unrotate")
    cent = rot.apply(out.centroids_dev, inverse=True)
    timer.stop("unrotate")
    phase.update(timer.collect())
    if not keep_data:
        data = DeviceData.__new__(DeviceData)
        data.n = n_local
    return DeviceFit(loop=out, rotation=rotation, centroids_dev=cent, data=data, phase=phase)


@on_device
def fit(x, cfg: KMeansConfig, inspect=None, device=None, comm: Comm | None = None) -> KMeansResult:
    """Sample, rotate, cluster and un-rotate on the B200 (core.py:417-460).  ``x``: any 2-D
    array-like (a pinned float32 CPU tensor is copied with a single DMA).

    Under torch.distributed (or with ``comm``) every rank passes the same matrix and copies only
    its contiguous row shard (like ``hierarchical_fit``); the loop runs row-sharded with one
    allreduce per iteration, and every rank returns the same result (assignments of all rows).
    ``inspect`` then receives this rank's rows only."""
    comm = comm or Comm()
    if comm.world > 1:
        return _fit_sharded(x, cfg, inspect, device, comm)
    src = _pinned_source(x)
    x = validate_vector_set(x, check_finite=False)  # finiteness: on the device, below
    dev = require_cuda(device)
    n_total, d = x.shape
    job = _RotationJob(d, cfg.seed)       # host PCG64 + LAPACK QR (persisted-model contract) ...
    if cfg.sampling_fraction == 1:
        x_dev = _h2d(x, dev, check_finite=True, src=src)  # ... overlapped with the copy
        # validate_vector_set, then sample_training_set's EmptySample (core.py:419-425,
        # preprocess.py:68-70), before init_centroids' KTooLarge
        sample_indices(n_total, 1.0, [cfg.seed, 1], k=cfg.k)
        sidx = None
        res = fit_device(x_dev, d, cfg, job, inspect=inspect, consume_input=True)
    else:
        # The reference validates the whole input before sampling (core.py:425-436).  Here the
        # whole-input check streams on its own stream while the sample is gathered (threaded,
        # into the pinned ring) and fitted; it is joined before anything is returned, and any
        # earlier error defers to it, so a non-finite input raises exactly the reference's
        # NonFiniteValue(first row, col).
        check = _FiniteCheckJob(x, dev)
        try:
            sidx = sample_indices(n_total, cfg.sampling_fraction, [cfg.seed, 1], k=cfg.k)
            x_dev = _h2d(x, dev, check_finite=True, idx=sidx)
            res = fit_device(x_dev, d, cfg, job, inspect=inspect, consume_input=True)
        except BaseException:
            check.result()
            raise
        check.result()
    rotation = res.rotation
    del x_dev
    out = res.loop
    phase = dict(res.phase)
    phase["rotation_host"] = job.seconds
    cent = to_host(res.centroids_dev[:, :d])
    ld = padded_ld(d)
    peak = 3 * out.assignments.shape[0] * ld + 6 * out.assignments.shape[0] + 4 * cfg.k * ld
    return KMeansResult(
        centroids=cent,
        assignments=out.assignments,
        stats=out.stats,
        terminated_by=out.terminated_by,
        rotation=rotation,
        centroids_rotated=out.centroids_rotated,
        d_prime_final=out.d_prime_final,
        sample_indices=sidx,
        init_indices=out.init_indices,
        work=out.work,
        phase_seconds=phase,
        peak_aux_values=peak,
        n_train=out.assignments.shape[0],
        recall_history=out.recall_history,
    )


def _fit_sharded(x, cfg: KMeansConfig, inspect, device, comm: Comm) -> KMeansResult:
    """fit() across ranks: shard-wise finiteness (same error on every rank), the sample drawn on
    every host with the same stream, each rank's contiguous shard of the sampled rows uploaded,
    the sharded loop, and the assignments assembled by one allreduce."""
    x = validate_vector_set(x, check_finite=False)
    dev = require_cuda(device)
    n_total, d = x.shape
    job = _RotationJob(d, cfg.seed)
    lo0, hi0 = comm.shard(n_total)
    _check_finite_sharded(x[lo0:hi0], dev, lo0, comm)
    sidx = sample_indices(n_total, cfg.sampling_fraction, [cfg.seed, 1], k=cfg.k)
    xs = x if sidx is None else x[sidx]
    n = xs.shape[0]
    lo, hi = comm.shard(n)
    x_dev = _h2d(xs[lo:hi], dev)
    res = fit_device(x_dev, d, cfg, job, inspect=inspect, comm=comm, n_global=n, row_lo=lo, consume_input=True)
    out = res.loop
    full = torch.zeros(n, dtype=torch.int32, device=dev)
    full[lo:hi] = out.assign_dev[:hi - lo]
    comm.allreduce_(full)
    assignments = to_host(full)
    ld = padded_ld(d)
    phase = dict(res.phase)
    phase["rotation_host"] = job.seconds
    return KMeansResult(
        centroids=to_host(res.centroids_dev[:, :d]), assignments=assignments, stats=out.stats,
        terminated_by=out.terminated_by, rotation=res.rotation, centroids_rotated=out.centroids_rotated,
        d_prime_final=out.d_prime_final, sample_indices=sidx, init_indices=out.init_indices, work=out.work,
        phase_seconds=phase, peak_aux_values=3 * (hi - lo) * ld + 6 * (hi - lo) + 4 * cfg.k * ld, n_train=n,
        recall_history=out.recall_history)


@on_device
def final_assign(x_full, result: KMeansResult, cfg: KMeansConfig, device=None, batch_rows: int = 1 << 20
                 ) -> np.ndarray:
    """Assign every vector to the fitted centroids with the pruned pass (core.py:463-541).

    Rows are rotated lazily in batches; tau is seeded from the training assignment for sampled
    rows (centroid 0 otherwise), exactly like the reference."""
    x_full = validate_vector_set(x_full, check_finite=False)  # finiteness: on the device, per batch
    dev = require_cuda(device)
    n, d = x_full.shape
    if d != result.rotation.dim:
        raise ValueError(f"vectors have dim {d}, model has dim {result.rotation.dim}")
    k = result.centroids_rotated.shape[0]
    assign = np.zeros(n, dtype=np.int32)
    if result.sample_indices is not None:
        assign[result.sample_indices] = result.assignments
    elif result.assignments.shape[0] == n:
        assign[:] = result.assignments
    pruned = pruning_supported(d) and result.d_prime_final is not None
    rot = DeviceRotation(result.rotation, dev)
    cents = Centroids(_h2d(np.ascontiguousarray(result.centroids_rotated, dtype=np.float32), dev), d)
    if pruned:
        dp = result.d_prime_final
        cents.refresh(dp, dp)
        plan = PrunePlan(d, dp, cfg.epsilon0, False, dev)
    else:
        cents.refresh(d, None)
        plan = None
    cfg_ws = KMeansConfig(k=k, x_batch_device=cfg.x_batch_device, cand_cap=cfg.cand_cap, gemm_backend=cfg.gemm_backend)
    ws = Workspace(dev, min(batch_rows, max(n, 1)), k, d, cfg_ws)  # reused by every batch
    for s0, e0, xb in _prefetch_batches(x_full, batch_rows, dev):
        key = _nonfinite_key(xb, e0 - s0, d)
        if key != (1 << 64) - 1:
            raise NonFiniteValue(s0 + key // d, key % d)
        data = DeviceData(rot.apply(xb, inplace=True), d)
        ws.assign[: e0 - s0].copy_(torch.from_numpy(assign[s0:e0]))
        if pruned:
            ws.counters.zero_()
            # rows keep their fitted assignment almost always -- unless most rows were outside the
            # training sample (seeded at centroid 0, so nearly all of them change: exact kernel)
            ws.flat = result.sample_indices is None
            pruned_assign_pass(data, cents, ws, plan)
            result.work.seed_dims += (e0 - s0) * d
            result.work.front_pair_dims += (e0 - s0) * k * plan.d_prime
            result.work.tail_dims += int(ws.counters[1].item())
        else:
            full_assign_pass(data, cents, ws)
            result.work.full_pair_dims += (e0 - s0) * k * d
        assign[s0:e0] = ws.assign[: e0 - s0].cpu().numpy()
    return assign

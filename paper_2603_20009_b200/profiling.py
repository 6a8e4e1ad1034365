"""Per-launch device timing of libskm_b200 kernels with CUDA events on the launching stream.

Every ABI call goes through ``native.call`` / ``native.check_call``; while a ``KernelTimer`` is
active those wrappers bracket the launch with two events and attach the launch's algorithmic
work (FLOPs for tensor-core GEMMs, bytes for memory-bound kernels), so ``bench.py`` can report
the dominant kernel's achieved throughput against the measured peaks -- measured live over
the timed region, never under a profiler.
"""

from __future__ import annotations

import contextlib
import json
import os

_ACTIVE = None

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def peaks() -> dict:
    """Measured roofline denominators (driver-written), else the profiling guide's fallback."""
    p = os.path.join(_ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            m = json.load(f)
        return {"hbm_gbs": float(m["hbm_gbs"]), "bf16_tflops": float(m["bf16_tflops"]),
                "bf16_tflops_sustained": float(m.get("bf16_tflops_sustained", m["bf16_tflops"])),
                "source": "MEASURED_PEAKS.json (measured)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "source": "B200_PROFILING.md fallback"}


def _profile_json(name: str) -> dict | None:
    try:
        with open(os.path.join(_ROOT, "profiles", name)) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def fp32_peak() -> float:
    """FFMA / FFMA2 peak measured on B200 (tools/micro/ffma2_bench.cu, profiles/fp32_peak.json)."""
    m = _profile_json("fp32_peak.json")
    return float(m["ffma2_tflops"]) if m else 74.0


def l2_peak() -> dict:
    """L2 read bandwidth measured on B200 (tools/micro/l2_bw.cu, profiles/l2_peak.json)."""
    m = _profile_json("l2_peak.json")
    if m:
        return {"gbs": float(m["l2_read_gbs"]), "source": "profiles/l2_peak.json (measured, tools/micro/l2_bw.cu)"}
    return {"gbs": 18000.0, "source": "estimate"}


def traffic_per_launch(kernel: str, rows_per_launch: float) -> float | None:
    """DRAM bytes (read + write) of one launch from a committed ncu --set full capture, scaled per row."""
    tr = _traffic_record(kernel)
    if not tr:
        return None
    return tr["dram_bytes"] / tr["rows"] * rows_per_launch


class KernelTimer:
    def __init__(self, reserve: int = 0):
        import torch
        self.torch = torch
        self.records = []  # (name, ev0, ev1, flops, bytes)
        self.launches = 0
        # events created up front: creating two per launch inside the timed region costs host
        # time at every post-sync relaunch
        self._pool = [torch.cuda.Event(enable_timing=True) for _ in range(reserve)]

    def _event(self):
        return self._pool.pop() if self._pool else self.torch.cuda.Event(enable_timing=True)

    def begin(self):
        e = self._event()
        e.record()
        return e

    def end(self, name, e0, flops=0.0, nbytes=0.0):
        e1 = self._event()
        e1.record()
        self.records.append((name, e0, e1, float(flops), float(nbytes)))
        self.launches += 1

    def summary(self) -> dict:
        self.torch.cuda.synchronize()
        agg: dict[str, dict] = {}
        for name, a, b, fl, by in self.records:
            s = agg.setdefault(name, {"launches": 0, "ms": 0.0, "flops": 0.0, "bytes": 0.0})
            s["launches"] += 1
            s["ms"] += a.elapsed_time(b)
            s["flops"] += fl
            s["bytes"] += by
        return agg


def _traffic_record(kernel: str) -> dict | None:
    """profiles/traffic.json: {kernel: {"dram_bytes": B, "rows": R, "source": "..."}} written from
    an ncu --set full capture (tools/prof/r1c_capture.sh)."""
    import json
    path = os.path.join(_ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(kernel)
    except (OSError, ValueError):
        return None


@contextlib.contextmanager
def active(timer: KernelTimer):
    global _ACTIVE
    prev = _ACTIVE
    _ACTIVE = timer
    try:
        yield timer
    finally:
        _ACTIVE = prev


def current():
    return _ACTIVE

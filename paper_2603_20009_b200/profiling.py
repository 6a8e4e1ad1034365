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


class KernelTimer:
    def __init__(self):
        import torch
        self.torch = torch
        self.records = []  # (name, ev0, ev1, flops, bytes)
        self.launches = 0

    def begin(self):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def end(self, name, e0, flops=0.0, nbytes=0.0):
        e1 = self.torch.cuda.Event(enable_timing=True)
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

    def roofline(self, steps: int, bytes_override: dict | None = None, rows_per_launch: dict | None = None) -> dict:
        agg = self.summary()
        for k_, v_ in (bytes_override or {}).items():
            if k_ in agg:
                agg[k_]["bytes"] = v_
        if not agg:
            return {}
        pk = peaks()
        name, top = max(agg.items(), key=lambda kv: kv[1]["ms"])
        total_ms = sum(v["ms"] for v in agg.values())
        per_launch_ms = top["ms"] / top["launches"]
        out = {"kernel": name, "share_of_kernel_time": top["ms"] / total_ms, "launches": top["launches"],
               "avg_launch_ms": per_launch_ms, "peak_source": pk["source"], "traffic": None}
        if top["flops"] > 0:
            # 3xTF32: the tensor pipe executes 3 TF32 MMAs per fp32-accurate product; dense TF32
            # peak is half the measured dense BF16 peak.
            alg_tflops = top["flops"] / (top["ms"] * 1e-3) / 1e12
            exec_tflops = 3.0 * alg_tflops
            tf32_peak = pk["bf16_tflops"] / 2.0
            out.update({"bound": "tensor", "achieved": exec_tflops, "peak": tf32_peak, "unit": "TFLOP/s",
                        "frac": exec_tflops / tf32_peak, "algorithmic_fp32_tflops": alg_tflops,
                        "note": "achieved = executed TF32 MMA flops (3 per fp32-accurate product) / time; "
                                "peak = dense TF32 = measured bf16 dense / 2"})
        else:
            gbs = top["bytes"] / (top["ms"] * 1e-3) / 1e9
            out.update({"bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                        "frac": gbs / pk["hbm_gbs"],
                        "note": "achieved = algorithmic bytes / time; for pruned_scan the bytes are the x tail "
                                "rows (HBM) + 4 B per touched (vector, centroid, dim) of the L2-resident "
                                "centroid tails (exact dims-touched counter)"})
        out["per_kernel_ms_per_step"] = {k: round(v["ms"] / steps, 3) for k, v in agg.items()}
        tr = _traffic_record(name)
        if tr and rows_per_launch:
            # DRAM bytes (read + write) of one launch of this kernel from a committed ncu --set full
            # capture, scaled per row to this run's average launch
            out["traffic"] = tr["dram_bytes"] / tr["rows"] * rows_per_launch.get(name, tr["rows"])
            out["traffic_source"] = tr["source"]
        return out


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

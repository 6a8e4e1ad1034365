#!/usr/bin/env python
"""Benchmark: SuperKMeans fit of 1M x 1536 fp32 into k=4096 for 10 fixed iterations
(BASELINE.json configs[1]) on 1..8 B200, one process per GPU.

Data: the reference's own generator, make_skewed_blobs(1_000_000, 1536, 8192, seed=0)
(pkg/tests/conftest.py:16-20, restated bit-exactly in paper_2603_20009_b200/synth.py), i.e. the
input of tests/golden/full_c2.npz: the timed trajectory is compared with the real reference's
(d', survivors, n_changed, wcss) and reported in "parity".

A step = one complete fit of the north-star hot path on device-resident rows: exact-chain rotation,
iteration 1 (tensor-core argmin + exact fix-up), 9 pruned iterations (tensor-core gate + exact
interval scan), ordered centroid update (+ NCCL allreduce at N>1), un-rotation.  Rows are sharded
across ranks (strong scaling: the 1M rows are fixed, split over N GPUs).

  python bench.py [--gpus N --steps K --warmup W]     # our B200 path
  python bench.py --impl reference ...                # the real reference (baseline/_ref) on host cores

Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "kmeans fit throughput (Lloyd iterations/s incl. rotation), 1M x 1536 fp32, k=4096, 10 iterations"
UNIT = "iter/s"
GOLDEN_C2 = os.path.join(ROOT, "tests", "golden", "full_c2.npz")

# secondary BASELINE configs measured after the headline (N=1): (generator, n, d, centres, k, iters, etr)
EXTRA = {
    "c1": ("blobs", 100_000, 128, 256, 256, 10, None),
    "c3": ("skewed", 1_000_000, 1024, 32768, 16384, 25, (1000, 10)),
    "c4_k1024": ("skewed", 1_000_000, 768, 2048, 1024, 10, None),
    "c4_k4096": ("skewed", 1_000_000, 768, 8192, 4096, 10, None),
    "c4_k16384": ("skewed", 1_000_000, 768, 32768, 16384, 10, None),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", "--rows", dest="n", type=int, default=1_000_000)
    ap.add_argument("--d", type=int, default=1536)
    ap.add_argument("--k", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--centers", type=int, default=8192)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the secondary configs (c1, c3, c4 sweep)")
    ap.add_argument("--extra", default=",".join(EXTRA) + ",c5", help="secondary configs to measure at N=1")
    return ap.parse_args()


def workload(args) -> dict:
    return {"workload": f"c2: make_skewed_blobs({args.n}, {args.d}, {args.centers}, seed={args.seed}) fp32, "
                        f"k={args.k}, {args.iters} fixed iterations (the reference's generator and fit config)",
            "n": args.n, "d": args.d, "k": args.k, "iterations": args.iters,
            "l2": "inputs (6 GB) exceed the 126 MB L2 between steps"}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples = []
        self.stop_evt = threading.Event()
        self.th = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop_evt.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) == 6:
                    self.samples.append(parts)
            except Exception:
                pass
            self.stop_evt.wait(0.2)

    def __enter__(self):
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop_evt.set()
        self.th.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------------------------- data
def make_rows(gen: str, n: int, d: int, centers: int, seed: int, hi: int | None = None) -> np.ndarray:
    """Rows [0, hi) of the reference generator's matrix (the RNG stream is sequential, so a shard
    needs every row before it drawn; rows past hi are not generated)."""
    from paper_2603_20009_b200 import synth
    hi = n if hi is None else hi
    if gen == "blobs":
        return synth.make_blobs(n, d, centers, seed, out_rows=hi) if hi != n else synth.make_blobs(n, d, centers, seed)
    return synth.make_skewed_blobs(n, d, centers, seed, out_rows=hi) if hi != n else \
        synth.make_skewed_blobs(n, d, centers, seed)


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    from paper_2603_20009_b200.engine import shard_bounds
    return shard_bounds(n, world, rank)


# ----------------------------------------------------------------------------- reference arm
def _reference_module():
    """The unmodified reference package installed from /root/reference/pkg into baseline/_ref
    (pip --target, its own setup.py builds the compiled kernels)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import superkmeans
    from superkmeans import kernels
    return superkmeans, bool(kernels.HAS_COMPILED)


def run_reference(args, rank, world):
    """The reference's own fit (compiled Cython kernels, OpenBLAS, all host cores) on the full c2
    workload.  A step is one Lloyd iteration of its loop, timed between consecutive `inspect`
    callbacks (rotation + iteration 1 make the first step of each fit; the last update and the
    un-rotation are charged to the next fit's first step): fits run back to back until W + K
    iterations are covered and the K after the warm-up are timed."""
    if rank != 0:
        return
    try:
        skm, compiled = _reference_module()
    except Exception as e:  # pragma: no cover - box without the install
        print(json.dumps({"impl": "reference", "unavailable": f"baseline/_ref not importable: {e}"}), flush=True)
        return
    cores = os.cpu_count() or 1
    x = make_rows("skewed", args.n, args.d, args.centers, args.seed)
    cfg = skm.KMeansConfig(k=args.k, max_iters=args.iters, seed=args.seed)
    need = args.warmup + args.steps
    stamps = [time.perf_counter()]
    traj = []
    while len(stamps) - 1 < need:
        res = skm.fit(x, cfg, inspect=lambda it, ctx: stamps.append(time.perf_counter()))
        traj = [s.d_prime for s in res.stats]
    steps_s = np.diff(np.array(stamps))[args.warmup:need]
    total = float(steps_s.sum())
    value = args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload(args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"the reference's fit on the full workload, {args.steps} timed Lloyd iterations "
                                   f"after {args.warmup} warm-up iterations (compiled kernels: {compiled})"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference": {"package": "baseline/_ref/superkmeans (unmodified, pip --target from /root/reference/pkg)",
                      "step_seconds": [round(float(v), 3) for v in steps_s], "d_prime": traj},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(args, x: np.ndarray) -> dict | None:
    """Bounded sample of the reference on this box's host cores: its fit with max_iters=1 on the full
    c2 rows (rotation + iteration 1, the full-distance pass), ~10-30 s.  The pruned iterations are
    timed by the --impl reference arm (all 10 iterations, same data)."""
    try:
        skm, compiled = _reference_module()
    except Exception:
        return None
    cfg = skm.KMeansConfig(k=args.k, max_iters=1, seed=args.seed)
    t0 = time.perf_counter()
    skm.fit(x, cfg)
    dt = time.perf_counter() - t0
    return {"value": 1.0 / dt, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
            "sample": f"reference fit (baseline/_ref, compiled kernels: {compiled}) with max_iters=1 on the full "
                      f"{args.n}x{args.d} rows: rotation + the iteration-1 full-distance pass, {dt:.1f} s; the "
                      f"--impl reference arm times all iterations"}


def run_extra(name: str, dev) -> dict:
    """One secondary BASELINE config (EXTRA[name]) at N = 1: the reference generator's rows,
    one warm-up fit, the median of 2 timed fits (5 for the small, host-bound c1; CUDA events)."""
    import torch
    from paper_2603_20009_b200 import api
    from paper_2603_20009_b200.config import EtrConfig, KMeansConfig
    from paper_2603_20009_b200.device import to_device_matrix
    from paper_2603_20009_b200.hostmath import generate_rotation
    gen, n, d, centers, k, iters, etr = EXTRA[name]
    t0 = time.perf_counter()
    xh = make_rows(gen, n, d, centers, 0)
    xd = to_device_matrix(xh, device=dev)
    del xh
    gs = time.perf_counter() - t0
    ccfg = KMeansConfig(k=k, max_iters=iters, seed=0,
                        etr=EtrConfig(n_queries=etr[0], top_k=etr[1]) if etr else None)
    rot = generate_rotation(d, 0)
    r = api.fit_device(xd, d, ccfg, rot)  # warm-up
    torch.cuda.synchronize()
    times = []
    # small configs are host/launch-bound and their fit time moves with host noise: more samples
    for _ in range(5 if n * d < 50_000_000 else 2):
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record()
        r = api.fit_device(xd, d, ccfg, rot)
        a1.record()
        torch.cuda.synchronize()
        times.append(a0.elapsed_time(a1))
    s2 = r.loop.stats
    ms = float(np.median(times))
    import dataclasses
    fcfg = dataclasses.replace(ccfg, exact_work_stats=False)
    api.fit_device(xd, d, fcfg, rot)  # warm-up
    a0 = torch.cuda.Event(enable_timing=True)
    a1 = torch.cuda.Event(enable_timing=True)
    a0.record()
    rf = api.fit_device(xd, d, fcfg, rot)
    a1.record()
    torch.cuda.synchronize()
    fms = a0.elapsed_time(a1)
    wso = {"ms_per_fit": round(fms, 2), "iter_per_s": round(len(rf.loop.stats) / (fms * 1e-3), 2),
           "bitwise_equal_to_exact_fit": bool(np.array_equal(rf.loop.assignments, r.loop.assignments)
                                              and torch.equal(rf.centroids_dev, r.centroids_dev)
                                              and [s.survivors for s in rf.loop.stats] == [s.survivors for s in s2])}
    del rf
    out = {
        "workload": f"{'make_blobs' if gen == 'blobs' else 'make_skewed_blobs'}({n}, {d}, {centers}, seed=0), "
                    f"k={k}, max_iters={iters}" + (f", ETR(n_queries={etr[0]}, top_k={etr[1]})" if etr else ""),
        "ms_per_fit": round(ms, 2), "iterations": len(s2), "iter_per_s": round(len(s2) / (ms * 1e-3), 2),
        "terminated_by": r.loop.terminated_by, "d_prime": [s.d_prime for s in s2],
        "prune_rate": [None if s.prune_rate_after_gemm is None else round(s.prune_rate_after_gemm, 5)
                       for s in s2],
        "pruned_dim_fraction": [None if s.d_prime is None else
                                round(1.0 - s.tail_dims_touched / (n * k * (d - s.d_prime)), 6) for s in s2],
        "recall_history": [round(v, 4) for v in r.loop.recall_history], "data_gen_s": round(gs, 1),
        "exact_work_stats_off": wso,
    }
    del xd
    return out


def run_c5(dev, exact_work_stats: bool = True) -> dict:
    """BASELINE c5: hierarchical k-means of 10M x 1024 into k_total = 65536 with meso_k = 430
    (the reference's rule caps near 50.7K at meso_k = 256), rows generated on the GPU
    with the skewed-blob distribution (the host generator would take minutes at 41 GB).  Device-
    resident entry; one warm-up on 200K rows, then one timed fit (CUDA events)."""
    import torch
    from paper_2603_20009_b200.hierarchical import HierarchicalConfig, hierarchical_fit_device
    from paper_2603_20009_b200.hostmath import generate_rotation
    from paper_2603_20009_b200.synth import make_shard_device
    n, d, k_total, meso_k = 10_000_000, 1024, 65536, 430
    rot = generate_rotation(d, 0)
    w = make_shard_device(200_000, d, 4096, 0, 200_000, 1, dev)
    hierarchical_fit_device(w, d, HierarchicalConfig(k_total=2048, seed=0), rotation=rot)
    del w
    t0 = time.perf_counter()
    x = make_shard_device(n, d, 2 * k_total, 0, n, 0, dev)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = hierarchical_fit_device(x, d, HierarchicalConfig(k_total=k_total, meso_k=meso_k, seed=0,
                                                         exact_work_stats=exact_work_stats), rotation=rot)
    e1.record()
    torch.cuda.synchronize()
    del x
    import hashlib
    asg = r.assignments.cpu().numpy() if hasattr(r.assignments, "cpu") else np.asarray(r.assignments)
    cen = r.centroids.cpu().numpy() if hasattr(r.centroids, "cpu") else np.asarray(r.centroids)
    digest = hashlib.sha256(asg.tobytes() + cen.tobytes()).hexdigest()[:16]
    return {"workload": f"hierarchical_fit_device: {n} x {d} skewed blobs generated on the GPU (same distribution as "
                        f"make_skewed_blobs, not its values), HierarchicalConfig(k_total={k_total}, meso_k={meso_k}, "
                        f"seed=0{'' if exact_work_stats else ', exact_work_stats=False'}), meso 3 + fine 5 "
                        f"iterations, groups batched in one loop",
            "s_per_fit": round(e0.elapsed_time(e1) / 1e3, 3), "achieved_k": int(r.k),
            "phase_s": {k_: round(v_, 3) for k_, v_ in r.phase_seconds.items()}, "data_gen_s": round(gen_s, 1),
            "assignments_centroids_sha256_16": digest}


# ----------------------------------------------------------------------------- roofline
def roofline(prof, steps: int, args, stats, n_local: int) -> dict:
    from paper_2603_20009_b200 import profiling
    agg = prof.summary()
    pk = profiling.peaks()
    total_ms = sum(v["ms"] for v in agg.values())
    tf32 = pk["bf16_tflops"] / 2.0
    fp32 = profiling.fp32_peak()
    l2 = profiling.l2_peak()
    pruned = [s for s in stats if s.d_prime is not None]
    n, d, k = args.n, args.d, args.k
    # algorithmic HBM bytes of a pruned iteration (one X read: seed tau needs all d dims,
    # the tail scan the same rows; assign/tau read+write; the centroids)
    hbm_bytes = steps * sum(4.0 * n * d + 16.0 * n + 4.0 * k * d for _ in pruned) * n_local / n
    # bytes the scan reads from L2/L1: x tails + 4 B per touched (row, centroid, dim)
    l2_bytes = steps * sum(4.0 * n * (d - s.d_prime) + 4.0 * s.tail_dims_touched for s in pruned) * n_local / n
    kernels = {}
    for name, v in sorted(agg.items(), key=lambda kv: -kv[1]["ms"])[:10]:
        e = {"ms_per_step": round(v["ms"] / steps, 3), "share": round(v["ms"] / total_ms, 4),
             "launches_per_step": v["launches"] / steps}
        sec = v["ms"] * 1e-3
        if name.startswith("gemm_"):  # 3xTF32: 3 TF32 MMAs per fp32-accurate product
            ex = 3.0 * v["flops"] / sec / 1e12
            e.update(bound="tensor", achieved=round(ex, 1), peak=tf32, unit="TFLOP/s", frac=round(ex / tf32, 3))
        elif name.startswith("chain_"):
            a = v["flops"] / sec / 1e12
            e.update(bound="fp32 (CUDA-core fma chain)", achieved=round(a, 1), peak=fp32, unit="TFLOP/s",
                     frac=round(a / fp32, 3))
        elif v["bytes"] > 0 and name != "pruned_scan":
            a = v["bytes"] / sec / 1e9
            e.update(bound="hbm", achieved=round(a, 1), peak=pk["hbm_gbs"], unit="GB/s", frac=round(a / pk["hbm_gbs"], 3))
        kernels[name] = e
    scan = agg.get("pruned_scan")
    out = {"kernels": kernels, "peak_source": pk["source"]}
    if scan:
        sec = scan["ms"] * 1e-3
        per_launch_ms = scan["ms"] / scan["launches"]
        a_hbm = hbm_bytes / sec / 1e9
        a_l2 = l2_bytes / sec / 1e9
        out.update({
            "kernel": "pruned_scan", "share_of_kernel_time": round(scan["ms"] / total_ms, 4),
            "launches": scan["launches"], "avg_launch_ms": round(per_launch_ms, 4),
            "bound": "hbm", "achieved": round(a_hbm, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": round(a_hbm / pk["hbm_gbs"], 4),
            "traffic": profiling.traffic_per_launch("pruned_scan", n_local * len(pruned) * steps / scan["launches"]),
            "algorithmic_bytes_per_launch": hbm_bytes / scan["launches"],
            "l2": {"bytes_per_launch": l2_bytes / scan["launches"], "achieved": round(a_l2, 1), "peak": l2["gbs"],
                   "unit": "GB/s", "frac": round(a_l2 / l2["gbs"], 4), "peak_source": l2["source"]},
            "limiter": "not HBM: the scan reads the L2-resident centroid tails row by row (LSU / L1 wavefronts "
                       "and the sequential-tau bookkeeping; ncu in profiles/)",
            "note": "achieved = SURVEY 8(d) algorithmic HBM bytes of the pruned iterations (4Nd + 16N + 4kd each) / "
                    "scan time; l2 = x tails + 4 B per touched (row, centroid, dim) from the exact counter",
        })
    return out


# ----------------------------------------------------------------------------- our arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    # test-only overrides (tests/test_gpu_multirank.py runs this bench with 2 ranks on one GPU):
    # SKM_BENCH_DEVICE pins every rank to one device, SKM_DIST_BACKEND=gloo replaces NCCL
    local = int(os.environ.get("SKM_BENCH_DEVICE", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("SKM_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    from paper_2603_20009_b200 import api, native, profiling
    from paper_2603_20009_b200.config import EtrConfig, KMeansConfig
    from paper_2603_20009_b200.device import to_device_matrix
    from paper_2603_20009_b200.engine import Comm
    from paper_2603_20009_b200.hostmath import generate_rotation

    native.load()
    comm = Comm()
    lo, hi = shard_range(args.n, world, rank)
    t_gen = time.perf_counter()
    x_host = make_rows("skewed", args.n, args.d, args.centers, args.seed, hi=hi)[lo:hi]
    gen_s = time.perf_counter() - t_gen
    x = to_device_matrix(x_host, device=dev)
    cfg = KMeansConfig(k=args.k, max_iters=args.iters, seed=args.seed)
    t_qr = time.perf_counter()
    rotation = generate_rotation(args.d, args.seed)
    qr_s = time.perf_counter() - t_qr

    def one_fit():
        return api.fit_device(x, args.d, cfg, rotation, comm=comm, n_global=args.n, row_lo=lo)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        one_fit()
    barrier()
    # ---- timed region: K device-resident fits ----
    prof = profiling.KernelTimer(reserve=2 * 800 * args.steps)  # > 2 events per native call of a c2 fit
    lib = native.load()
    with ClockSampler(local) as clocks:
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        k_launch0 = lib.skm_kernel_launches()
        with profiling.active(prof):
            e0.record()
            res = None
            iters_done = 0
            for _ in range(args.steps):
                res = one_fit()
                iters_done += len(res.loop.stats)
            e1.record()
        k_launches = lib.skm_kernel_launches() - k_launch0
        barrier()
    elapsed = max_over_ranks(e0.elapsed_time(e1) / 1e3)
    value = iters_done / elapsed
    ms_per_step = 1e3 * elapsed / args.steps
    launches = int(k_launches)  # kernels libskm_b200 launched in the timed region (skm_kernel_launches)
    st = res.loop.stats
    roof = roofline(prof, args.steps, args, st, hi - lo)

    # ---- parity of the timed trajectory with the real reference's (tests/golden/full_c2.npz) ----
    parity = None
    if os.path.exists(GOLDEN_C2) and (args.n, args.d, args.k, args.iters, args.centers, args.seed) == \
            (1_000_000, 1536, 4096, 10, 8192, 0):
        g = np.load(GOLDEN_C2)
        checks = {
            "d_prime": [-1 if s.d_prime is None else s.d_prime for s in st] == g["dp"].tolist(),
            "survivors": [s.survivors for s in st] == g["surv"].tolist(),
            "tail_dims": [s.tail_dims_touched for s in st] == g["tail"].tolist(),
            "n_changed": [-1 if s.n_changed is None else s.n_changed for s in st] == g["changed"].tolist(),
            "wcss": [s.wcss for s in st] == g["wcss"].tolist(),
        }
        parity = {"golden": "tests/golden/full_c2.npz (the real reference, 632.7 s on 8 cores)",
                  "bitwise_equal": checks, "all": all(checks.values())}

    # ---- the same fit with exact_work_stats=False (option: candidates that cannot win skip the
    #      tail walk; everything but tail_dims_touched stays bitwise) ----
    wso = None
    if world == 1 and not args.no_extra:
        try:
            import dataclasses
            fcfg = dataclasses.replace(cfg, exact_work_stats=False)
            api.fit_device(x, args.d, fcfg, rotation)  # warm-up
            ftimes = []
            for _ in range(2):
                f0 = torch.cuda.Event(enable_timing=True)
                f1 = torch.cuda.Event(enable_timing=True)
                f0.record()
                rf = api.fit_device(x, args.d, fcfg, rotation)
                f1.record()
                torch.cuda.synchronize()
                ftimes.append(f0.elapsed_time(f1))
            fst = rf.loop.stats
            fms = float(np.median(ftimes))
            wso = {"ms_per_fit": round(fms, 2), "iter_per_s": round(len(fst) / (fms * 1e-3), 3),
                   "tail_dims_touched": [s.tail_dims_touched for s in fst],
                   "pruning_ms": [round(1e3 * s.timings.get("pruning", 0.0), 1) for s in fst],
                   "exact_pruning_ms": [round(1e3 * s.timings.get("pruning", 0.0), 1) for s in st],
                   "all_ms": [round(v, 1) for v in ftimes],
                   "bitwise_equal_to_exact_fit": {
                       "assignments": bool(np.array_equal(rf.loop.assignments, res.loop.assignments)),
                       "centroids": bool(torch.equal(rf.centroids_dev, res.centroids_dev)),
                       "d_prime_survivors_changed_wcss": [(s.d_prime, s.survivors, s.n_changed, s.wcss) for s in fst]
                       == [(s.d_prime, s.survivors, s.n_changed, s.wcss) for s in st]}}
            del rf
        except Exception as exc:
            wso = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    # ---- end to end through the public entry (api.fit) with pinned host input ----
    e2e = None
    if not args.no_e2e:
        try:
            host = torch.empty((hi - lo, args.d), dtype=torch.float32, pin_memory=True)
            host.numpy()[:] = x_host
            ee0 = torch.cuda.Event(enable_timing=True)
            ee1 = torch.cuda.Event(enable_timing=True)
            barrier()
            ee0.record()
            d2h = 0
            iters_e2e = 0
            for _ in range(args.steps):
                if world == 1:
                    r = api.fit(host, cfg)  # H2D (one DMA) + host QR beside it + fit + D2H of the result
                    d2h = r.centroids.nbytes + r.assignments.nbytes + r.centroids_rotated.nbytes
                    iters_e2e += len(r.stats)
                else:
                    job = api._RotationJob(args.d, args.seed)
                    xe = torch.zeros_like(x)
                    xe[:, :args.d].copy_(host, non_blocking=True)
                    r = api.fit_device(xe, args.d, cfg, job, comm=comm, n_global=args.n, row_lo=lo, consume_input=True)
                    cent = r.centroids_dev[:, :args.d].cpu()
                    d2h = cent.numel() * 4 + r.loop.assignments.nbytes
                    iters_e2e += len(r.loop.stats)
            ee1.record()
            barrier()
            e2e_s = max_over_ranks(ee0.elapsed_time(ee1) / 1e3)
            e2e = {"value": iters_e2e / e2e_s, "unit": UNIT,
                   "h2d_bytes_per_step": int(host.numel() * 4) * world, "d2h_bytes_per_step": int(d2h) * world,
                   "note": "api.fit on a pinned host matrix: H2D (one DMA), host QR of R (LAPACK, the persisted-model "
                           "contract) beside the copy, fit, D2H of centroids + assignments" if world == 1 else
                           "per rank: H2D of the shard, host QR beside it, sharded fit, D2H of centroids + assignments"}

        except Exception as exc:  # reported in the line instead of losing the device-timed value
            e2e = {"value": None, "unit": UNIT, "error": f"{type(exc).__name__}: {exc}"[:300]}

    extra = None
    if world == 1 and not args.no_extra:
        extra = {}
        for name in [c for c in args.extra.split(",") if c in EXTRA]:
            try:
                extra[name] = run_extra(name, dev)
            except Exception as exc:  # one config failing must not cost the headline line
                extra[name] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
                torch.cuda.empty_cache()

    if world == 1 and not args.no_extra and "c5" in args.extra.split(","):
        try:
            extra["c5"] = run_c5(dev)
        except Exception as exc:
            extra["c5"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        torch.cuda.empty_cache()
        try:
            c5f = run_c5(dev, exact_work_stats=False)
            c5f["bitwise_equal_to_exact_fit"] = \
                c5f["assignments_centroids_sha256_16"] == extra["c5"].get("assignments_centroids_sha256_16")
            extra["c5_exact_work_stats_off"] = c5f
        except Exception as exc:
            extra["c5_exact_work_stats_off"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    # the host-CPU reference sample runs last: its BLAS threads must not compete with the host
    # orchestration of the (launch-bound) small secondary configs above
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(args, x_host)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32 (reference-exact: fp32 fma-chain rotation, 3xTF32 tensor-core "
                                          "distances settled by the fp32 chain, fp32 scan)",
            "data": "synthetic (the reference's make_skewed_blobs generator)",
            "config": dict(workload(args), **{
                "rows_per_gpu": hi - lo, "data_gen_s": round(gen_s, 1), "rotation_qr_host_ms": round(qr_s * 1e3, 1),
                "d_prime": [s.d_prime for s in st],
                "prune_rate": [None if s.prune_rate_after_gemm is None else round(s.prune_rate_after_gemm, 6)
                               for s in st],
                "pruned_dim_fraction": [None if s.d_prime is None else
                                        round(1.0 - s.tail_dims_touched / (args.n * args.k * (args.d - s.d_prime)), 6)
                                        for s in st],
                "phase_ms_last_step": {k_: round(v_ * 1e3, 2) for k_, v_ in res.phase.items()}}),
            "parity": parity, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks.summary(), "exact_work_stats_off": wso, "configs": extra,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

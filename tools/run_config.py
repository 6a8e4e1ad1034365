"""Run one BASELINE config on the device and print timings/stats.
   python tools/run_config.py c3   (1M x 1024, k=16384, ETR 1000 queries top-10, 25 iters)
   python tools/run_config.py c4 --k 16384   (1M x 768, 10 iters)"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

os.environ.setdefault("SKM_DIAG", "1")  # scan diagnostics read back per iteration

from paper_2603_20009_b200.synth import make_shard_device  # noqa: E402
from paper_2603_20009_b200 import api, profiling  # noqa: E402
from paper_2603_20009_b200.config import EtrConfig, KMeansConfig  # noqa: E402
from paper_2603_20009_b200.hostmath import generate_rotation  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", choices=["c3", "c4"])
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--k", type=int, default=None)
ap.add_argument("--iters", type=int, default=None)
a = ap.parse_args()
if a.config == "c3":
    d, k, iters = 1024, a.k or 16384, a.iters or 25
    cfg = KMeansConfig(k=k, max_iters=iters, seed=0, etr=EtrConfig(n_queries=1000, top_k=10))
else:
    d, k, iters = 768, a.k or 4096, a.iters or 10
    cfg = KMeansConfig(k=k, max_iters=iters, seed=0)
dev = torch.device("cuda", 0)
x = make_shard_device(a.n, d, 2 * k, 0, a.n, 0, dev)
rot = generate_rotation(d, 0)
api.fit_device(x, d, KMeansConfig(k=k, max_iters=2, seed=0), rot)  # warm-up (allocations, attributes)
torch.cuda.synchronize()
prof = profiling.KernelTimer()
t0 = time.perf_counter()
with profiling.active(prof):
    r = api.fit_device(x, d, cfg, rot)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
st = r.loop.stats
print(f"{a.config}: n={a.n} d={d} k={k} iters={len(st)} terminated_by={r.loop.terminated_by} wall={wall:.3f}s")
print("kernels ms:", {kk: round(v["ms"], 1) for kk, v in sorted(prof.summary().items(), key=lambda kv: -kv[1]["ms"])})
print("d'", [s.d_prime for s in st])
print("surv/vec", [round(s.survivors / a.n, 1) for s in st])
print("recall", [round(v, 4) for v in r.loop.recall_history])
print("phase", {kk: round(v * 1e3, 1) for kk, v in r.phase.items()})

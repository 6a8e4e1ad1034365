"""Time hierarchical_fit on device-generated skewed blobs.  python tools/run_hier.py --n 1000000 --d 1024 --k 16384"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import make_shard_device  # noqa: E402
from paper_2603_20009_b200 import profiling  # noqa: E402
from paper_2603_20009_b200.hierarchical import HierarchicalConfig, hierarchical_fit  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--d", type=int, default=1024)
ap.add_argument("--k", type=int, default=16384)
ap.add_argument("--meso-k", type=int, default=None)
a = ap.parse_args()
dev = torch.device("cuda", 0)
x = make_shard_device(a.n, a.d, 2 * a.k, 0, a.n, 0, dev)[:, :a.d].cpu().numpy()
cfg = HierarchicalConfig(k_total=a.k, meso_k=a.meso_k, seed=0) if a.meso_k else HierarchicalConfig(k_total=a.k, seed=0)
hierarchical_fit(x[:50000], HierarchicalConfig(k_total=256, seed=0))  # warm-up
torch.cuda.synchronize()
t0 = time.perf_counter()
prof = profiling.KernelTimer()
with profiling.active(prof):
    r = hierarchical_fit(x, cfg)
torch.cuda.synchronize()
print("kernels ms:", {kk: round(v["ms"], 1) for kk, v in sorted(prof.summary().items(), key=lambda kv: -kv[1]["ms"])})
print(f"hierarchical n={a.n} d={a.d} k_total={a.k}: achieved k={r.k} wall={time.perf_counter() - t0:.3f}s "
      f"phase={ {k: round(v, 3) for k, v in r.phase_seconds.items()} }")

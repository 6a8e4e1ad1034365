"""Run hierarchical_fit / fit twice on identical input and report whether results are bitwise equal.
python tools/determinism.py --n 1000000 --d 1024 --k 16384"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_20009_b200.synth import make_shard_device  # noqa: E402
from paper_2603_20009_b200.hierarchical import HierarchicalConfig, hierarchical_fit  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--d", type=int, default=1024)
ap.add_argument("--k", type=int, default=16384)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
dev = torch.device("cuda", 0)
x = make_shard_device(a.n, a.d, 2 * a.k, 0, a.n, 0, dev)[:, :a.d].cpu().numpy()
print("x checksum", float(np.float64(x[::997].sum())), flush=True)
runs = []
for r in range(a.reps):
    res = hierarchical_fit(x, HierarchicalConfig(k_total=a.k, seed=0))
    meso_dp = [s.d_prime for s in res.stats]
    meso_sv = [s.survivors for s in res.stats]
    print(f"rep {r}: k={res.k} meso d'={meso_dp} survivors={meso_sv} wcss={[round(s.wcss, 3) for s in res.stats]}",
          flush=True)
    runs.append(res)
for r in range(1, a.reps):
    print(f"rep {r} vs 0: assign equal={np.array_equal(runs[0].assignments, runs[r].assignments)} "
          f"cent equal={runs[0].k == runs[r].k and np.array_equal(runs[0].centroids_rotated, runs[r].centroids_rotated)}")

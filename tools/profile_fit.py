"""Small fit driver for ncu captures: c2 shape (d=1536, k=4096) on fewer rows.
   ncu ... python tools/profile_fit.py --n 200000 --iters 4"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

os.environ.setdefault("SKM_DIAG", "1")  # scan diagnostics read back per iteration

from paper_2603_20009_b200.device import to_device_matrix  # noqa: E402
from paper_2603_20009_b200.synth import make_skewed_blobs  # noqa: E402
from paper_2603_20009_b200 import api  # noqa: E402
from paper_2603_20009_b200.config import KMeansConfig  # noqa: E402
from paper_2603_20009_b200.hostmath import generate_rotation  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=200000)
ap.add_argument("--d", type=int, default=1536)
ap.add_argument("--k", type=int, default=4096)
ap.add_argument("--iters", type=int, default=4)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--centers", type=int, default=8192)
ap.add_argument("--device-data", action="store_true", help="device-generated rows (same distribution, fast)")
a = ap.parse_args()
dev = torch.device("cuda", 0)
if a.device_data:
    from paper_2603_20009_b200.synth import make_shard_device
    x = make_shard_device(a.n, a.d, a.centers, 0, a.n, 0, dev)
else:  # the reference's generator (c2 rows when --n 1000000): bench.py's data
    x = to_device_matrix(make_skewed_blobs(a.n, a.d, a.centers, 0))
cfg = KMeansConfig(k=a.k, max_iters=a.iters, seed=0)
rot = generate_rotation(a.d, 0)
from paper_2603_20009_b200 import profiling  # noqa: E402
prof = profiling.KernelTimer()
import time  # noqa: E402
for i in range(a.reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if i == a.reps - 1:
        with profiling.active(prof):
            r = api.fit_device(x, a.d, cfg, rot)
    else:
        r = api.fit_device(x, a.d, cfg, rot)
    torch.cuda.synchronize()
    print(f"rep {i}: fit wall {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
print("kernels ms:", {k: round(v["ms"], 2) for k, v in sorted(prof.summary().items(), key=lambda kv: -kv[1]["ms"])})
st = r.loop.stats
print("d'", [s.d_prime for s in st], "surv/vec", [round(s.survivors / a.n, 1) for s in st],
      "tail/vec", [round(s.tail_dims_touched / a.n) for s in st],
      "computed blocks/vec", [round(b / a.n) for b in r.loop.scan_blocks],
      "waves/vec", [round(w / a.n, 1) for w in r.loop.scan_waves],
      "n_changed", [s.n_changed for s in st], "chain re-evaluations/vec", [round(dg[3] / a.n, 2) for dg in r.loop.scan_diag],
      "lane util", [round(dg[0] / max(1, 32 * dg[1]), 3) for dg in r.loop.scan_diag],
      "phase", {k: round(v * 1e3, 1) for k, v in r.phase.items()})
print("per-iteration pruning ms", [round(1e3 * s.timings.get("pruning", 0.0), 1) for s in st])

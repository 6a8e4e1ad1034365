"""exact_work_stats False vs True on one B200: c2 (device-resident fit, per-iteration pruning
time) and optionally c5 (bench.run_c5).  Checks the assignments / centroids agree bitwise."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_20009_b200 import api, synth  # noqa: E402
from paper_2603_20009_b200.config import KMeansConfig  # noqa: E402
from paper_2603_20009_b200.device import to_device_matrix  # noqa: E402
from paper_2603_20009_b200.hostmath import generate_rotation  # noqa: E402

x = to_device_matrix(synth.make_skewed_blobs(1_000_000, 1536, 8192, 0))
rot = generate_rotation(1536, 0)
res = {}
for flag in (True, False, True, False):
    cfg = KMeansConfig(k=4096, max_iters=10, seed=0, exact_work_stats=flag)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = api.fit_device(x, 1536, cfg, rot)
    e1.record()
    torch.cuda.synchronize()
    st = r.loop.stats
    print(f"exact_work_stats={flag}: {e0.elapsed_time(e1):.1f} ms; pruning ms per iteration",
          [round(1e3 * s.timings.get("pruning", 0.0), 1) for s in st],
          "tail dims/row", [s.tail_dims_touched // 1_000_000 for s in st], flush=True)
    res[flag] = (r.loop.assignments.copy(), r.centroids_dev.cpu().numpy().copy(), [s.survivors for s in st])
print("assignments equal", np.array_equal(res[True][0], res[False][0]),
      "centroids equal", np.array_equal(res[True][1], res[False][1]), "survivors equal", res[True][2] == res[False][2])
del x
if os.environ.get("C5", "0") == "1":
    import bench
    dev = torch.device("cuda:0")
    for flag in (False, True):
        print("c5", flag, bench.run_c5(dev, exact_work_stats=flag), flush=True)

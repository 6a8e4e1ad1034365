"""c1 (100K x 128, k=256, 10 iterations) fit time on the reference generator's rows."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_20009_b200 import api, synth  # noqa: E402
from paper_2603_20009_b200.config import KMeansConfig  # noqa: E402
from paper_2603_20009_b200.device import to_device_matrix  # noqa: E402
from paper_2603_20009_b200.hostmath import generate_rotation  # noqa: E402

x = to_device_matrix(synth.make_blobs(100_000, 128, 256, 0))
cfg = KMeansConfig(k=256, max_iters=10, seed=0)
rot = generate_rotation(128, 0)
for _ in range(2):
    r = api.fit_device(x, 128, cfg, rot)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    r = api.fit_device(x, 128, cfg, rot)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print("c1 ms", [round(1e3 * t, 2) for t in ts], "changed", [s.n_changed for s in r.loop.stats],
      "pruning ms", [round(1e3 * s.timings.get("pruning", 0), 2) for s in r.loop.stats])

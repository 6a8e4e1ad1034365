"""Two c2 fits (1M x 1536, k = 4096, reference generator rows) with exact_work_stats=False, for an
ncu launch list of the option (profiles/r2_nowin_launches.csv.gz)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_20009_b200 import api, synth  # noqa: E402
from paper_2603_20009_b200.config import KMeansConfig  # noqa: E402
from paper_2603_20009_b200.device import to_device_matrix  # noqa: E402
from paper_2603_20009_b200.hostmath import generate_rotation  # noqa: E402

x = to_device_matrix(synth.make_skewed_blobs(1_000_000, 1536, 8192, 0))
rot = generate_rotation(1536, 0)
cfg = KMeansConfig(k=4096, max_iters=10, seed=0, exact_work_stats=False)
for _ in range(2):
    r = api.fit_device(x, 1536, cfg, rot)
torch.cuda.synchronize()
print("tail dims", [s.tail_dims_touched for s in r.loop.stats])

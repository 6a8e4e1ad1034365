"""Per-rank compute of the c2 fit at the 1/2/4/8-GPU shard sizes on one B200 (rows of the
reference generator's c2 matrix, device-resident, the loop without the collective)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_20009_b200 import api, synth  # noqa: E402
from paper_2603_20009_b200.config import KMeansConfig  # noqa: E402
from paper_2603_20009_b200.device import to_device_matrix  # noqa: E402
from paper_2603_20009_b200.hostmath import generate_rotation  # noqa: E402

x_all = synth.make_skewed_blobs(1_000_000, 1536, 8192, 0)
rot = generate_rotation(1536, 0)
cfg = KMeansConfig(k=4096, max_iters=10, seed=0)
for world in (1, 2, 4, 8):
    n = 1_000_000 // world
    x = to_device_matrix(x_all[:n])
    api.fit_device(x, 1536, cfg, rot)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        api.fit_device(x, 1536, cfg, rot)
    e1.record()
    torch.cuda.synchronize()
    print(f"world {world}: {n} rows per rank, {e0.elapsed_time(e1) / 3:.1f} ms per fit", flush=True)
    del x

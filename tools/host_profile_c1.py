"""Host-side cost of the c1 loop (cProfile of 5 fits after warm-up): the launch-bound config."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_20009_b200 import api, synth  # noqa: E402
from paper_2603_20009_b200.config import KMeansConfig  # noqa: E402
from paper_2603_20009_b200.device import to_device_matrix  # noqa: E402
from paper_2603_20009_b200.hostmath import generate_rotation  # noqa: E402

x = to_device_matrix(synth.make_blobs(100_000, 128, 256, 0))
cfg = KMeansConfig(k=256, max_iters=10, seed=0)
rot = generate_rotation(128, 0)
for _ in range(3):
    api.fit_device(x, 128, cfg, rot)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    api.fit_device(x, 128, cfg, rot)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)

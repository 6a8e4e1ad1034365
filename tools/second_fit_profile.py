"""cProfile of the second c2 fit in a process (the one-time slow fit, profiles/r2_summary.md)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_20009_b200 import api  # noqa: E402
from paper_2603_20009_b200.config import KMeansConfig  # noqa: E402
from paper_2603_20009_b200.hostmath import generate_rotation  # noqa: E402
from paper_2603_20009_b200.synth import make_shard_device  # noqa: E402

dev = torch.device("cuda", 0)
x = make_shard_device(1_000_000, 1536, 8192, 0, 1_000_000, 0, dev)
rot = generate_rotation(1536, 0)
cfg = KMeansConfig(k=4096, max_iters=10, seed=0)
api.fit_device(x, 1536, cfg, rot)
torch.cuda.synchronize()
for rep in (1, 2):
    pr = cProfile.Profile()
    pr.enable()
    api.fit_device(x, 1536, cfg, rot)
    torch.cuda.synchronize()
    pr.disable()
    print(f"==== fit {rep}")
    pstats.Stats(pr).sort_stats("tottime").print_stats(12)

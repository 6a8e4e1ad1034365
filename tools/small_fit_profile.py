"""Host vs device time of one hierarchical fine-group-sized fit (23K x 1024, k = 152, 5 iterations):
wall per fit, device time per fit (CUDA events), and the top host functions (cProfile)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_20009_b200 import api  # noqa: E402
from paper_2603_20009_b200.config import KMeansConfig  # noqa: E402
from paper_2603_20009_b200.engine import DeviceData, fit_rotated_device  # noqa: E402
from paper_2603_20009_b200.synth import make_shard_device  # noqa: E402

n, d, k = int(sys.argv[1]) if len(sys.argv) > 1 else 23000, 1024, 152
dev = torch.device("cuda", 0)
x = make_shard_device(n, d, 300, 0, n, 0, dev)
cfg = KMeansConfig(k=k, max_iters=5, seed=3)
data = DeviceData(x, d)
for _ in range(3):
    fit_rotated_device(data, cfg)
torch.cuda.synchronize()
reps = 20
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for _ in range(reps):
    out = fit_rotated_device(data, cfg)
e1.record()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / reps
print(f"fit {n}x{d} k={k} 5 iters: wall {wall * 1e3:.2f} ms, device span {e0.elapsed_time(e1) / reps:.2f} ms, "
      f"d' {[s.d_prime for s in out.stats]}")
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    fit_rotated_device(data, cfg)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)

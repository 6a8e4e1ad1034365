"""Where the e2e fit's time goes beyond the device fit: host QR, H2D DMA, finiteness check."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_20009_b200 import api, synth  # noqa: E402
from paper_2603_20009_b200.config import KMeansConfig  # noqa: E402
from paper_2603_20009_b200.hostmath import generate_rotation  # noqa: E402

n, d = int(os.environ.get("N", 1_000_000)), 1536
x = synth.make_skewed_blobs(n, d, 8192, 0)
host = torch.empty((n, d), dtype=torch.float32, pin_memory=True)
host.numpy()[:] = x
print("cpus", os.cpu_count(), "torch threads", torch.get_num_threads())
for _ in range(3):
    t = time.perf_counter(); generate_rotation(d, 0); print(f"host QR {time.perf_counter() - t:.3f} s")
dev = torch.device("cuda:0")
buf = torch.empty((n, d), dtype=torch.float32, device=dev)
for _ in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    buf.copy_(host, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"H2D {dt * 1e3:.1f} ms {n * d * 4 / dt / 1e9:.1f} GB/s")
del buf
cfg = KMeansConfig(k=4096, max_iters=10, seed=0)
for _ in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    r = api.fit(host, cfg)
    torch.cuda.synchronize()
    print(f"api.fit {(time.perf_counter() - t) * 1e3:.1f} ms", {k: round(v, 4) for k, v in r.phase_seconds.items()})

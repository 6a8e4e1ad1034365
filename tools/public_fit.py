"""Wall time of the public host-NumPy entry (api.fit) at the c2 shape, phase breakdown.
python tools/public_fit.py --n 1000000 --d 1536 --k 4096"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_20009_b200.synth import make_shard_device  # noqa: E402
import paper_2603_20009_b200 as skb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--d", type=int, default=1536)
ap.add_argument("--k", type=int, default=4096)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
x = make_shard_device(a.n, a.d, 8192, 0, a.n, 0, torch.device("cuda", 0))[:, :a.d].cpu().numpy()
for r in range(a.reps):
    t0 = time.perf_counter()
    res = skb.fit(x, skb.KMeansConfig(k=a.k, max_iters=10, seed=0))
    dt = time.perf_counter() - t0
    print(f"rep {r}: fit wall {dt * 1e3:.1f} ms = {10 / dt:.2f} it/s; phases "
          f"{ {k: round(v * 1e3, 1) for k, v in res.phase_seconds.items()} }", flush=True)

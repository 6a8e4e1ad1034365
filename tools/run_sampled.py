"""SURVEY 8f-4 at scale: fit on a sample (sampling_fraction < 1) of N rows, then out-of-sample
final_assign of all N rows.  python tools/run_sampled.py --n 10000000 --d 1024 --k 4096 --frac 0.1
Property check (the oracle cannot run at this size): agreement of final_assign with the exact
fp64 argmin on 20 000 random rows (ADSampling may prune a true nearest centroid, so not 100%)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_20009_b200.synth import make_shard_device  # noqa: E402
import paper_2603_20009_b200 as skb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--d", type=int, default=1024)
ap.add_argument("--k", type=int, default=4096)
ap.add_argument("--frac", type=float, default=0.1)
a = ap.parse_args()
dev = torch.device("cuda", 0)
x = make_shard_device(a.n, a.d, 2 * a.k, 0, a.n, 0, dev)[:, :a.d].cpu().numpy()
cfg = skb.KMeansConfig(k=a.k, max_iters=10, sampling_fraction=a.frac, seed=0)
skb.fit(x[:100000], skb.KMeansConfig(k=256, max_iters=2, seed=0))  # warm-up
torch.cuda.synchronize()
t0 = time.perf_counter()
res = skb.fit(x, cfg)
t1 = time.perf_counter()
lab = skb.final_assign(x, res, cfg)
t2 = time.perf_counter()
rng = np.random.default_rng(1)
rows = rng.choice(a.n, 20000, replace=False)
xs = torch.tensor(x[rows], dtype=torch.float64, device=dev)
c = torch.tensor(res.centroids, dtype=torch.float64, device=dev)
dist = (xs * xs).sum(1, keepdim=True) - 2 * xs @ c.T + (c * c).sum(1)[None, :]
exact = dist.argmin(1).cpu().numpy()
agree = float(np.mean(exact == lab[rows]))
gap = dist.gather(1, torch.tensor(lab[rows], device=dev, dtype=torch.int64)[:, None])[:, 0] - dist.min(1).values
rel = float((gap / dist.min(1).values.clamp(min=1e-30)).max())
print(f"sampled fit: n={a.n} d={a.d} k={a.k} frac={a.frac} n_train={res.n_train} iters={len(res.stats)} "
      f"fit {t1 - t0:.2f}s phases { {k: round(v, 3) for k, v in res.phase_seconds.items()} }")
print(f"final_assign of {a.n} rows: {t2 - t1:.2f}s; agreement with exact fp64 argmin on 20000 rows {agree:.5f}, "
      f"max relative excess distance of the chosen centroid {rel:.2e}; labels in range {lab.min()}..{lab.max()}")

"""Randomised check of exact_work_stats=False against the exact-stats fit: every per-iteration
assignment and tau, d', survivors, n_changed, wcss, splits and the centroids must be bitwise
equal, for random shapes, generators, k, seeds and both GEMM backends."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

import paper_2603_20009_b200 as skb  # noqa: E402
from conftest import make_blobs, make_skewed_blobs  # noqa: E402
from paper_2603_20009_b200.config import KMeansConfig  # noqa: E402

rng = np.random.default_rng(int(os.environ.get("SEED", "2026")))
cases = int(os.environ.get("CASES", "24"))
bad = 0
for c in range(cases):
    d = int(rng.choice([64, 96, 128, 200, 256, 384, 512, 768, 1024, 1536]))
    n = int(rng.integers(20_000, 150_000))
    k = int(rng.choice([16, 50, 128, 300, 700, 1024, 2048]))
    k = min(k, n // 4)
    seed = int(rng.integers(0, 1000))
    gen = rng.choice(["blobs", "skew"])
    backend = "portable" if rng.random() < 0.2 else "auto"
    centers = int(rng.integers(max(2, k // 4), 4 * k))
    x = make_blobs(n, d, centers, seed=seed) if gen == "blobs" else make_skewed_blobs(n, d, centers, seed=seed)
    snaps = {}

    def grab(tag):
        def f(it, info):
            snaps[(tag, it)] = (info["assignments"], info["best_sq_dist"].view(np.uint32))
        return f

    iters = int(rng.integers(4, 9))
    base = dict(k=k, max_iters=iters, seed=seed, gemm_backend=backend)
    r0 = skb.fit(x, KMeansConfig(**base), inspect=grab(0))
    r1 = skb.fit(x, KMeansConfig(**base, exact_work_stats=False), inspect=grab(1))
    ok = len(r0.stats) == len(r1.stats)
    ok = ok and all((a.d_prime, a.survivors, a.n_changed, a.wcss, a.n_empty_splits) ==
                    (b.d_prime, b.survivors, b.n_changed, b.wcss, b.n_empty_splits) for a, b in zip(r0.stats, r1.stats))
    ok = ok and all(np.array_equal(snaps[(0, i)][0], snaps[(1, i)][0]) and np.array_equal(snaps[(0, i)][1], snaps[(1, i)][1])
                    for i in range(1, len(r0.stats) + 1))
    ok = ok and np.array_equal(r0.centroids.view(np.uint32), r1.centroids.view(np.uint32))
    saved = sum(a.tail_dims_touched for a in r0.stats) - sum(b.tail_dims_touched for b in r1.stats)
    bad += not ok
    print(f"case {c}: {gen} n={n} d={d} k={k} centers={centers} seed={seed} iters={iters} {backend}: "
          f"{'OK' if ok else 'MISMATCH'}; tail dims saved {saved / max(1, sum(a.tail_dims_touched for a in r0.stats)):.1%}",
          flush=True)
print(f"{cases - bad}/{cases} bitwise equal")
sys.exit(1 if bad else 0)

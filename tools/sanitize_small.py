"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck; initcheck takes > 18 min
once the ETR part runs): fit (pruned path with certification), sampled fit + final_assign,
hierarchical, ETR fit, IVF probe evaluation, a d = 8192 fit (one-warp scan)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

from conftest import make_skewed_blobs  # noqa: E402
import paper_2603_20009_b200 as skb  # noqa: E402

x = make_skewed_blobs(3000, 200, 40, 3)
r = skb.fit(x, skb.KMeansConfig(k=48, max_iters=4, seed=1))
cfg = skb.KMeansConfig(k=32, max_iters=3, seed=2, sampling_fraction=0.5)
r2 = skb.fit(x, cfg)
a = skb.final_assign(x, r2, cfg)
h = skb.hierarchical_fit(x, skb.HierarchicalConfig(k_total=60, seed=3))
# ETR: device ground truth (GEMM + radix top-k), probe tally every iteration
r3 = skb.fit(x, skb.KMeansConfig(k=40, max_iters=6, seed=4, etr=skb.EtrConfig(n_queries=200, top_k=10)))
# IVF probe evaluation (probe ranking + tally with explored sizes)
q = x[:100]
gt = skb.brute_force_topk(x, q, 10)
pe = skb.probe_eval(r.centroids, skb.build_cluster_lists(r.assignments, r.k), x, q, gt, 5, top_ks=(10,))
# exact_work_stats=False: full-d certificate (hi x hi extension) + deferred certified entries, flat
# and grouped paths included
r4 = skb.fit(x, skb.KMeansConfig(k=48, max_iters=4, seed=1, exact_work_stats=False))
h2 = skb.hierarchical_fit(x, skb.HierarchicalConfig(k_total=60, seed=3, exact_work_stats=False))
assert np.array_equal(r4.assignments, r.assignments) and np.array_equal(h2.assignments, h.assignments)
# long tail (d = 8192: 112+ tail blocks): the one-warp scan instantiation
xw = make_skewed_blobs(400, 8192, 12, 5)
r5 = skb.fit(xw, skb.KMeansConfig(k=16, max_iters=3, seed=1))
r6 = skb.fit(xw, skb.KMeansConfig(k=16, max_iters=3, seed=1, exact_work_stats=False))
assert np.array_equal(r5.assignments, r6.assignments)
print("ok", r.k, r2.k, int(a.max()), h.k, r3.terminated_by, round(pe["recall_at_10"], 3), "nowin ok")

"""Replay one pruned iteration of the device fit in the oracle from the device's own inputs
(rotated data, centroids used, previous assignments) to separate kernel bugs from trajectory
amplification."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

import paper_2603_20009_b200 as skb  # noqa: E402
from conftest import make_blobs  # noqa: E402
from oracle import skm_ref  # noqa: E402

x = make_blobs(100_000, 128, 256, seed=0)
snaps = []
res = skb.fit(x, skb.KMeansConfig(k=256, max_iters=6, seed=0), inspect=lambda it, c: snaps.append(c))
xr_dev = skb.apply_rotation(x, res.rotation)
for it in range(1, len(snaps)):
    s, prev = snaps[it], snaps[it - 1]
    dp = s["d_prime"]
    tau = np.empty(x.shape[0], np.float32)
    a = prev["assignments"].copy()
    p = skm_ref.Params(k=256)
    sv, td, ch = skm_ref.pruned_pass(np.ascontiguousarray(xr_dev), s["centroids_rotated"], dp, p, tau, a)
    dis = np.count_nonzero(a != s["assignments"])
    st = res.stats[it]
    print(f"it{it + 1} d'={dp}: oracle replay vs device: {dis} assignment diffs, survivors {sv} vs {st.survivors}, "
          f"tail {td} vs {st.tail_dims_touched}, tau equal {np.mean(tau == s['best_sq_dist']):.6f}")

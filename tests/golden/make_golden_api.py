"""Golden outputs of the reference's remaining public helpers (fit_lloyd, prune_and_assign,
initial_threshold, measure_prune_rate), produced by the REAL reference:
    PYTHONPATH=baseline/_ref python tests/golden/make_golden_api.py
Inputs are regenerated from seeds by the tests (tests/conftest.py generators)."""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from conftest import make_blobs  # noqa: E402

import superkmeans as skm  # noqa: E402
from superkmeans.distance import expand_to_sq_l2, matmul  # noqa: E402
from superkmeans.model import AssignmentState, pdxify  # noqa: E402
from superkmeans.preprocess import compute_norms  # noqa: E402


def main():
    out = {}
    x = make_blobs(5000, 96, 20, seed=3)
    r = skm.fit_lloyd(x, k=16, n_iters=8, seed=1, collect_assignments=True)
    out.update(lloyd_centroids=r.centroids, lloyd_assign=r.assignments, lloyd_wcss=np.array(r.wcss_history),
               lloyd_hist=np.stack(r.assignment_history), lloyd_term=np.array(r.terminated_by))
    # per-vector pruning twin on one bank
    rng = np.random.default_rng(8)
    x = make_blobs(300, 200, 12, seed=5)
    c = x[rng.choice(300, 40, replace=False)].copy()
    dp = 24
    bank = pdxify(c, dp)
    vals = expand_to_sq_l2(matmul(x, c, dp), compute_norms(x, dp), compute_norms(c, dp), partial=True)
    prev = rng.integers(0, 40, 300).astype(np.int32)
    tau = np.array([skm.initial_threshold(x[i], c[prev[i]]) for i in range(300)], np.float32)
    state = AssignmentState(assignment=prev.copy(), best_sq_dist=tau.copy())
    cfg = skm.KMeansConfig(k=40)
    outs = [skm.prune_and_assign(i, vals, bank, state, cfg, x[i]) for i in range(300)]
    out.update(pa_prev=prev, pa_tau0=tau, pa_assign=state.assignment, pa_tau=state.best_sq_dist,
               pa_surv=np.array([o.survivors_after_gemm for o in outs]),
               pa_dims=np.array([o.dims_touched for o in outs]),
               pa_rate=np.float64(skm.measure_prune_rate(outs, 40)))
    np.savez_compressed(os.path.join(HERE, "api.npz"), **out)


if __name__ == "__main__":
    main()

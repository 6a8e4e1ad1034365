"""The reference's remaining public helpers on the device, against the real reference's outputs
(tests/golden/make_golden_api.py): fit_lloyd (bitwise: exact full-distance argmin each
iteration), the per-vector pruning twin and its threshold / prune-rate helpers."""

import os

import numpy as np
import pytest

from conftest import make_blobs

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "api.npz")


def test_fit_lloyd_bitwise():
    import paper_2603_20009_b200 as skb
    g = np.load(GOLD)
    x = make_blobs(5000, 96, 20, seed=3)
    r = skb.fit_lloyd(x, k=16, n_iters=8, seed=1, collect_assignments=True)
    assert np.array_equal(np.stack(r.assignment_history), g["lloyd_hist"])
    assert r.wcss_history == g["lloyd_wcss"].tolist()
    assert np.array_equal(r.centroids, g["lloyd_centroids"])
    assert np.array_equal(r.assignments, g["lloyd_assign"])
    assert r.terminated_by == str(g["lloyd_term"])


def test_prune_and_assign_bitwise():
    import paper_2603_20009_b200 as skb
    from paper_2603_20009_b200.config import AssignmentState, pdxify
    from paper_2603_20009_b200.extras import compute_norms
    g = np.load(GOLD)
    rng = np.random.default_rng(8)
    x = make_blobs(300, 200, 12, seed=5)
    c = x[rng.choice(300, 40, replace=False)].copy()
    dp = 24
    prev = rng.integers(0, 40, 300).astype(np.int32)
    assert np.array_equal(prev, g["pa_prev"])
    tau = np.array([skb.initial_threshold(x[i], c[prev[i]]) for i in range(300)], np.float32)
    assert np.array_equal(tau, g["pa_tau0"])
    # the reference's partial distances (sgemm bits): the device chain GEMM + expansion
    import torch
    from paper_2603_20009_b200 import device
    from paper_2603_20009_b200.engine import chain_gemm
    X, Cm = device.to_device_matrix(x), device.to_device_matrix(c)
    D = torch.empty((300, 40), dtype=torch.float32, device="cuda")
    chain_gemm(X, Cm, 300, 40, dp, D, 0, 448, xsq=device.row_sq_norms(X, dp), ysq=device.row_sq_norms(Cm, dp))

    class Block:
        values = D.cpu().numpy()

    bank = pdxify(c, dp)
    state = AssignmentState(assignment=prev.copy(), best_sq_dist=tau.copy())
    cfg = skb.KMeansConfig(k=40)
    outs = [skb.prune_and_assign(i, Block, bank, state, cfg, x[i]) for i in range(300)]
    assert np.array_equal(state.assignment, g["pa_assign"])
    assert np.array_equal(state.best_sq_dist, g["pa_tau"])
    assert [o.survivors_after_gemm for o in outs] == g["pa_surv"].tolist()
    assert [o.dims_touched for o in outs] == g["pa_dims"].tolist()
    assert skb.measure_prune_rate(outs, 40) == float(g["pa_rate"])
    del compute_norms

"""Large-index regime (> 2^32 elements in the row matrix): duplication invariance.

The oracle cannot run at these sizes, so the property is size-independent: the matrix is a
shard stacked on itself (row i == row i + n).  Every per-row decision of the loop (GEMM argmin,
gate, pruning scan, Forgy/seed rows, hierarchical regrouping) sees identical inputs for both
copies, so their assignments must be identical in every phase; a 32-bit row-offset overflow in
any kernel (row * ld > 2^31 from row 2.1M on at d = 1024, > 2^32 from row 4.2M) breaks it.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

N_HALF = 2_200_000  # 2 x 2.2M rows x 1024 = 4.5e9 elements
D = 1024


@pytest.fixture(scope="module")
def doubled():
    from paper_2603_20009_b200.synth import make_shard_device
    dev = torch.device("cuda", 0)
    half = make_shard_device(N_HALF, D, 600, 0, N_HALF, 11, dev)
    return torch.cat([half, half]), dev


def test_fit_duplicated_rows_agree_past_int32(doubled):
    from paper_2603_20009_b200 import api
    from paper_2603_20009_b200.config import KMeansConfig
    from paper_2603_20009_b200.hostmath import generate_rotation
    x, dev = doubled
    cfg = KMeansConfig(k=512, max_iters=5, seed=1)
    r = api.fit_device(x.clone(), D, cfg, generate_rotation(D, 1), consume_input=True)
    a = r.loop.assignments
    assert a.shape[0] == 2 * N_HALF
    assert np.array_equal(a[:N_HALF], a[N_HALF:])
    assert any(s.d_prime is not None for s in r.loop.stats)  # the pruned scan ran
    assert len(np.unique(a)) > 256


def test_hierarchical_duplicated_rows_agree_past_int32(doubled):
    import paper_2603_20009_b200 as skb
    x, _ = doubled
    xh = x[:, :D].cpu().numpy()
    h = skb.hierarchical_fit(xh, skb.HierarchicalConfig(k_total=4096, seed=5))
    a = h.assignments
    assert np.array_equal(a[:N_HALF], a[N_HALF:])
    assert h.k > 1000

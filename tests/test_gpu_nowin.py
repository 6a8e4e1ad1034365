"""exact_work_stats = False (engine.cert_extension over all d columns): candidates whose full-d
distance interval lies above the seed tau skip the tail walk.  Everything the reference's loop decides --
every assignment, tau, survivors, the d' trajectory, n_changed, wcss, splits, the centroids --
must be bitwise the exact-stats fit; only tail_dims_touched may drop (it counts the walks made)."""

import numpy as np
import pytest

from conftest import make_blobs, make_skewed_blobs

pytestmark = pytest.mark.gpu

CASES = {
    "c1_shape": ("blobs", 100_000, 128, 256, 0, 256, 10),
    "skew768": ("skew", 200_000, 768, 2048, 0, 1024, 8),
    "skew1536": ("skew", 100_000, 1536, 1024, 1, 512, 6),
    "skew1024_small_k": ("skew", 300_000, 1024, 4096, 2, 64, 5),
    "skew768_portable": ("skew", 100_000, 768, 1024, 4, 256, 6, "portable"),
}


def _data(kind, n, d, centers, seed):
    return make_blobs(n, d, centers, seed=seed) if kind == "blobs" else make_skewed_blobs(n, d, centers, seed=seed)


@pytest.mark.parametrize("name", sorted(CASES))
def test_nowin_fit_matches_exact_stats(name):
    import paper_2603_20009_b200 as skb
    from paper_2603_20009_b200 import engine
    from paper_2603_20009_b200.config import KMeansConfig
    kind, n, d, centers, seed, k, iters = CASES[name][:7]
    backend = CASES[name][7] if len(CASES[name]) > 7 else "auto"
    x = _data(kind, n, d, centers, seed)
    snaps = {}

    def grab(tag):
        def f(it, info):
            snaps[(tag, it)] = (info["assignments"], info["best_sq_dist"])
        return f

    ref = skb.fit(x, KMeansConfig(k=k, max_iters=iters, seed=seed, gemm_backend=backend), inspect=grab("exact"))
    calls = []
    orig = engine.cert_extension

    def spy(data, cents, plan, *a, **kw):
        out = orig(data, cents, plan, *a, **kw)
        if out.get("nowin"):
            calls.append(1)
        return out

    engine.cert_extension = spy
    try:
        fast = skb.fit(x, KMeansConfig(k=k, max_iters=iters, seed=seed, gemm_backend=backend, exact_work_stats=False),
                       inspect=grab("fast"))
    finally:
        engine.cert_extension = orig
    assert calls, "the cannot-win certificate never ran"
    assert len(ref.stats) == len(fast.stats)
    for key in ("d_prime", "survivors", "n_changed", "wcss", "n_empty_splits", "prune_rate_after_gemm"):
        assert [getattr(s, key) for s in fast.stats] == [getattr(s, key) for s in ref.stats], key
    assert all(f.tail_dims_touched <= r.tail_dims_touched for f, r in zip(fast.stats, ref.stats))
    assert sum(f.tail_dims_touched for f in fast.stats) < sum(r.tail_dims_touched for r in ref.stats)
    for it in range(1, len(ref.stats) + 1):
        a0, t0 = snaps[("exact", it)]
        a1, t1 = snaps[("fast", it)]
        assert np.array_equal(a0, a1), it
        assert np.array_equal(t0.view(np.uint32), t1.view(np.uint32)), it
    assert np.array_equal(fast.assignments, ref.assignments)
    assert np.array_equal(fast.centroids.view(np.uint32), ref.centroids.view(np.uint32))
    assert fast.terminated_by == ref.terminated_by


def test_nowin_hierarchical_matches_exact_stats():
    import paper_2603_20009_b200 as skb
    x = make_skewed_blobs(200_000, 512, 4096, seed=3)
    a = skb.hierarchical_fit(x, skb.HierarchicalConfig(k_total=2048, seed=3))
    b = skb.hierarchical_fit(x, skb.HierarchicalConfig(k_total=2048, seed=3, exact_work_stats=False))
    assert a.k == b.k
    assert np.array_equal(a.assignments, b.assignments)
    assert np.array_equal(a.centroids.view(np.uint32), b.centroids.view(np.uint32))
    assert [s.survivors for s in a.stats] == [s.survivors for s in b.stats]


def _run_ws(rank, world, port, q, exact_work_stats):
    import os

    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_20009_b200 import api
        from paper_2603_20009_b200.config import KMeansConfig
        from paper_2603_20009_b200.engine import Comm
        from paper_2603_20009_b200.hostmath import generate_rotation
        torch.cuda.set_device(0)
        x = make_skewed_blobs(60_000, 256, 1024, seed=6)
        n, d = x.shape
        comm = Comm()
        lo, hi = comm.shard(n)
        xd = api._h2d(x[lo:hi], torch.device("cuda", 0))
        cfg = KMeansConfig(k=300, max_iters=6, seed=6, exact_work_stats=exact_work_stats)
        res = api.fit_device(xd, d, cfg, generate_rotation(d, 6), comm=comm, n_global=n, row_lo=lo)
        st = res.loop.stats
        q.put((rank, {"assign": res.loop.assignments, "lo": lo, "cent": res.centroids_dev[:, :d].cpu().numpy(),
                      "stats": [(s.d_prime, s.survivors, s.n_changed, s.wcss) for s in st],
                      "tail": [s.tail_dims_touched for s in st]}))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_nowin_two_ranks_match_single_rank_exact():
    """Row-sharded (2 ranks over gloo on one GPU): the option's decisions are per row and its
    policy reads the allreduced survivors, so the ranks agree and match the 1-GPU exact fit."""
    import os

    from test_gpu_multirank import _spawn
    port = 29900 + (os.getpid() % 400)
    one = _spawn(1, port, _run_ws, (True,))[0]
    two = _spawn(2, port + 1, _run_ws, (False,))
    a2 = np.concatenate([two[r]["assign"] for r in sorted(two, key=lambda r: two[r]["lo"])])
    assert np.array_equal(a2, one["assign"])
    for r in two:
        assert two[r]["stats"] == one["stats"]
        assert np.array_equal(two[r]["cent"], one["cent"])
        assert sum(two[r]["tail"]) < sum(one["tail"])

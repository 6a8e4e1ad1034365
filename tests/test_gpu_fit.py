"""Whole-fit parity on the B200 against golden trajectories produced by the real reference
(tests/golden/make_golden.py) -- the north-star bar:
  * per-iteration assignments agree on >= 99.9% of points, disagreements only at near-ties;
  * integer outputs (survivors, d' trajectory, n_changed, splits, termination) bit-exact
    whenever the assignments agree;
  * centroids within 1e-4 relative L2;
  * final_assign agrees like the loop does.
"""

import os

import numpy as np
import pytest

from conftest import make_blobs, make_skewed_blobs

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "fits.npz")
NEAR_TIE_REL = 1e-5


def _make(spec):
    kind, n, d, centers, seed = spec[:5]
    if kind != "blobs":
        return make_skewed_blobs(n, d, centers, seed=seed)
    return make_blobs(n, d, centers, seed=seed) if len(spec) == 5 else make_blobs(n, d, centers, seed=seed,
                                                                                 spread=spec[5])


def _cases():
    import importlib.util
    spec = importlib.util.spec_from_file_location("mg", os.path.join(os.path.dirname(GOLD), "make_golden.py"))
    # make_golden imports the reference at module level; read the case table textually instead
    src = open(os.path.join(os.path.dirname(GOLD), "make_golden.py")).read()
    start = src.index("FIT_CASES = {")
    end = src.index("}\n", start) + 1
    ns = {}
    exec(src[start:end], ns)
    return ns["FIT_CASES"]


CASES = _cases()


def _box_blas_is_reference() -> bool:
    """True when this box's NumPy/OpenBLAS reproduces the survey container's sgemm bits (the
    reference goldens' BLAS; tests/golden/blas_bits.npz): the oracle then computes the
    reference's exact arithmetic here and the device must equal it bit for bit."""
    import hashlib
    import importlib.util
    here = os.path.dirname(os.path.abspath(__file__))
    spec = importlib.util.spec_from_file_location("mbb", os.path.join(here, "golden", "make_blas_bits.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    g = np.load(os.path.join(here, "golden", "blas_bits.npz"))
    for (M, N, K, lay) in m.GEMM_CASES:
        a, b = m.gemm_inputs(M, N, K, lay, 0)
        out = a @ b.T if lay == "nt" else a @ b
        if hashlib.sha256(np.ascontiguousarray(out).tobytes()).hexdigest() != str(g[f"gemm_{M}_{N}_{K}_{lay}"]):
            return False
    return True


def _assert_bitwise_vs_oracle(res, snaps, ref):
    """The exact-arithmetic bar: d' trajectory, every assignment, survivors, dims touched,
    n_changed, wcss and the centroids equal the oracle's."""
    assert [s.d_prime for s in res.stats] == [s.d_prime for s in ref.stats]
    for it, (a, s) in enumerate(zip(snaps, ref.snapshots)):
        assert np.array_equal(a, s["assignments"]), it
    assert [s.survivors for s in res.stats] == [s.survivors for s in ref.stats]
    assert [s.tail_dims_touched for s in res.stats] == [s.tail_dims_touched for s in ref.stats]
    assert [s.n_changed for s in res.stats] == [s.n_changed for s in ref.stats]
    assert [s.wcss for s in res.stats] == [s.wcss for s in ref.stats]
    assert np.array_equal(res.centroids, ref.centroids)


def _rel_l2(a, b):
    return float(np.linalg.norm(a.astype(np.float64) - b) / max(np.linalg.norm(b.astype(np.float64)), 1e-30))


def _classify(xr, cents, a_ours, a_ref):
    """Relative distance gap of every disagreement (fp64, centroids of that iteration)."""
    idx = np.flatnonzero(a_ours != a_ref)
    if idx.size == 0:
        return np.zeros(0)
    x = xr[idx].astype(np.float64)
    da = np.sum((x - cents[a_ours[idx]]) ** 2, axis=1)
    db = np.sum((x - cents[a_ref[idx]]) ** 2, axis=1)
    return np.abs(da - db) / np.maximum(np.maximum(da, db), 1e-30)


@pytest.mark.parametrize("name", list(CASES))
def test_fit_matches_reference_trajectory(name):
    import paper_2603_20009_b200 as skb
    g = np.load(GOLD)
    spec, kw = CASES[name]
    x = _make(spec)
    if name.startswith("etr"):
        kw = dict(kw, etr=skb.EtrConfig(n_queries=300, top_k=10))
    cfg = skb.KMeansConfig(**kw)
    snaps = []
    res = skb.fit(x, cfg, inspect=lambda it, ctx: snaps.append(ctx))
    ref_assign = g[f"{name}_snap_assign"]
    assert np.array_equal(res.init_indices, g[f"{name}_init"])
    if f"{name}_rotation" in g.files:  # host QR contract
        assert np.array_equal(res.rotation.data, g[f"{name}_rotation"])
    else:
        import hashlib
        sha = hashlib.sha256(np.ascontiguousarray(res.rotation.data, dtype=np.float32).tobytes()).hexdigest()
        assert sha == str(g[f"{name}_rotation_sha256"])
    m = min(len(snaps), ref_assign.shape[0])
    all_equal = True
    xr = x if res.sample_indices is None else x[res.sample_indices]
    xr = xr.astype(np.float64) @ res.rotation.data.astype(np.float64)
    for it in range(m):
        a = snaps[it]["assignments"]
        agree = float(np.mean(a == ref_assign[it]))
        assert agree >= 0.999, (name, it, agree)
        if agree < 1.0:
            all_equal = False
            gaps = _classify(xr, g[f"{name}_snap_cent"][it].astype(np.float64), a, ref_assign[it])
            print(f"{name} it{it + 1}: {np.count_nonzero(a != ref_assign[it])} disagreements, max rel gap {gaps.max():.2e}")
    assert _rel_l2(res.centroids, g[f"{name}_centroids"]) <= 1e-4
    # the exact-arithmetic bar (the device reproduces the reference's rounding): every assignment,
    # the counters, wcss and the rotated centroids bit for bit; the final centroids come from a
    # tiny k x d un-rotation, where OpenBLAS takes its small-matrix kernel: last-ulp level
    assert all_equal, name
    assert np.array_equal(res.centroids_rotated, g[f"{name}_centroids_rot"]), name
    assert _rel_l2(res.centroids, g[f"{name}_centroids"]) <= 1e-6
    assert [s.survivors for s in res.stats] == g[f"{name}_surv"].tolist()
    assert [s.tail_dims_touched for s in res.stats] == g[f"{name}_tail"].tolist()
    assert [s.wcss for s in res.stats] == g[f"{name}_wcss"].tolist()
    if all_equal:
        st = res.stats
        assert np.array_equal(np.bincount(res.assignments, minlength=cfg.k),
                              np.bincount(g[f"{name}_assign"], minlength=cfg.k))
        assert [-1 if s.d_prime is None else s.d_prime for s in st] == g[f"{name}_dp"].tolist()
        assert [-1 if s.n_changed is None else s.n_changed for s in st] == g[f"{name}_changed"].tolist()
        assert [s.n_empty_splits for s in st] == g[f"{name}_splits"].tolist()
        assert res.terminated_by == str(g[f"{name}_term"])
        # ETR: recall history is an integer tally over the queries -> equal floats
        assert res.recall_history == g[f"{name}_recall"].tolist()
        # wcss sums expansion-based distances (cancellation-prone): GEMM-rounding level only
        np.testing.assert_allclose([s.wcss for s in st], g[f"{name}_wcss"], rtol=1e-4)
    fa = skb.final_assign(x, res, cfg)
    assert np.array_equal(fa, g[f"{name}_final"])
    # north star: final IVF recall@10 within 0.5 points of the reference's clustering
    from oracle import skm_ref
    xt = x if res.sample_indices is None else x[res.sample_indices]
    q = xt[np.random.default_rng(7).choice(xt.shape[0], 200, replace=False)]
    gi, gd = skm_ref.brute_force_topk(xt, q, 10)
    nprobe = max(1, int(np.ceil(0.05 * cfg.k)))
    ours = skb.probe_eval(res.centroids, skb.build_cluster_lists(res.assignments, cfg.k), xt, q,
                          skb.GroundTruth(indices=gi, distances=gd, k_gt=10), nprobe, top_ks=(10,))
    ref = skm_ref.probe_eval(g[f"{name}_centroids"], skm_ref.cluster_lists(g[f"{name}_assign"], cfg.k), xt, q, gi, 10,
                             nprobe, top_ks=(10,))
    assert abs(ours["recall_at_10"] - ref["recall_at_10"]) <= 0.005, (ours, ref)


def test_fit_c1_shape_vs_oracle():
    """Config-1 shape (100K x 128, k=256, 10 it) against the oracle (reference restatement):
    bitwise when this box's OpenBLAS is the reference's (checked against blas_bits.npz; the
    full-size goldens in test_gpu_full_size.py are bitwise on any box).  Otherwise:

    Disagreements come from distance near-ties and from ADSampling gate decisions whose
    partial distance sits within GEMM rounding of fl(tau*F) (the reference's own scan is not
    an exact argmin).  The d' controller is a knife edge on this config
    (iteration-4 prune rate 0.97020 vs the 0.97 band edge): when the two runs'
    prune rates straddle an edge the d' trajectories split and the runs legitimately diverge
    (different ADSampling false prunes).  The bar: >= 99.9% agreement on every iteration run
    at the same d'; a split must be explained by a prune rate within 1e-3 of a band edge;
    afterwards WCSS stays within the reference's Lloyd-equivalence bound (0.5%)."""
    import paper_2603_20009_b200 as skb
    from oracle import skm_ref
    x = make_blobs(100_000, 128, 256, seed=0)
    cfg = skb.KMeansConfig(k=256, max_iters=10, seed=0)
    snaps = []
    res = skb.fit(x, cfg, inspect=lambda it, ctx: snaps.append(ctx["assignments"]))
    ref = skm_ref.fit(x, skm_ref.Params(k=256, max_iters=10, seed=0))
    if _box_blas_is_reference():
        _assert_bitwise_vs_oracle(res, snaps, ref)
        return
    # another CPU's OpenBLAS kernel: the oracle is no longer the reference's exact arithmetic
    xr = x.astype(np.float64) @ ref.rotation.astype(np.float64)
    ours_dp = [s.d_prime for s in res.stats]
    ref_dp = [s.d_prime for s in ref.stats]
    print("d' ours", ours_dp, "ref", ref_dp)
    print("prune ours", [s.prune_rate_after_gemm for s in res.stats])
    print("prune ref ", [s.prune_rate_after_gemm for s in ref.stats])
    split_at = None
    for it, (a, s) in enumerate(zip(snaps, ref.snapshots)):
        agree = float(np.mean(a == s["assignments"]))
        gaps = _classify(xr, s["centroids_rotated"].astype(np.float64), a, s["assignments"])
        near = int(np.count_nonzero(gaps <= NEAR_TIE_REL))
        print(f"c1 it{it + 1}: d' {ours_dp[it]}/{ref_dp[it]} agree {agree:.6f}, {gaps.size} disagreements "
              f"({near} near-ties <= 1e-5)")
        if split_at is None and ours_dp[it] != ref_dp[it]:
            split_at = it
        if split_at is None:
            assert agree >= 0.999, (it, agree)
    if split_at is not None:
        rate = ref.stats[split_at - 1].prune_rate_after_gemm
        edge = min(abs(rate - cfg.prune_target_low), abs(rate - cfg.prune_target_high))
        print(f"d' split at iteration {split_at + 1}: reference prune rate {rate:.5f} is {edge:.2e} from a band edge")
        assert edge <= 1e-3
    w_ours, w_ref = res.stats[-1].wcss, ref.stats[-1].wcss
    assert abs(w_ours - w_ref) / w_ref <= 0.005
    rel = _rel_l2(res.centroids, ref.centroids)
    print("c1 centroid rel-L2", rel)
    if split_at is None:
        assert rel <= 2e-3


def test_fit_c2_shape_vs_oracle():
    """Config-2 dimensionality and k (d = 1536, k = 4096, 10 iterations, skewed blobs of the
    reference's prune-band fixture) on a 62 500-row sample, against the oracle: the same bar as
    the c1 test, plus final IVF recall@10 within 0.5 points."""
    import paper_2603_20009_b200 as skb
    from conftest import make_skewed_blobs
    from oracle import skm_ref
    x = make_skewed_blobs(62_500, 1536, 8192, seed=0)
    cfg = skb.KMeansConfig(k=4096, max_iters=10, seed=0)
    snaps = []
    res = skb.fit(x, cfg, inspect=lambda it, ctx: snaps.append(ctx["assignments"]))
    ref = skm_ref.fit(x, skm_ref.Params(k=4096, max_iters=10, seed=0))
    if _box_blas_is_reference():
        _assert_bitwise_vs_oracle(res, snaps, ref)
    ours_dp = [s.d_prime for s in res.stats]
    ref_dp = [s.d_prime for s in ref.stats]
    print("c2-shape d' ours", ours_dp, "ref", ref_dp)
    split_at = None
    for it, (a, s) in enumerate(zip(snaps, ref.snapshots)):
        agree = float(np.mean(a == s["assignments"]))
        print(f"c2-shape it{it + 1}: d' {ours_dp[it]}/{ref_dp[it]} agree {agree:.6f} "
              f"surv {res.stats[it].survivors}/{ref.stats[it].survivors}")
        if split_at is None and ours_dp[it] != ref_dp[it]:
            split_at = it
        if split_at is None:
            assert agree >= 0.999, (it, agree)
    if split_at is not None:
        rate = ref.stats[split_at - 1].prune_rate_after_gemm
        edge = min(abs(rate - cfg.prune_target_low), abs(rate - cfg.prune_target_high))
        assert edge <= 1e-3, (split_at, rate)
    else:
        assert _rel_l2(res.centroids, ref.centroids) <= 1e-4
    assert abs(res.stats[-1].wcss - ref.stats[-1].wcss) / ref.stats[-1].wcss <= 0.005
    q = x[np.random.default_rng(7).choice(x.shape[0], 500, replace=False)]
    gi, gd = skm_ref.brute_force_topk(x, q, 10)
    nprobe = int(np.ceil(0.01 * cfg.k))
    ours = skb.probe_eval(res.centroids, skb.build_cluster_lists(res.assignments, cfg.k), x, q,
                          skb.GroundTruth(indices=gi, distances=gd, k_gt=10), nprobe, top_ks=(10,))
    theirs = skm_ref.probe_eval(ref.centroids, skm_ref.cluster_lists(ref.assignments, cfg.k), x, q, gi, 10, nprobe,
                                top_ks=(10,))
    print("c2-shape recall@10 ours", ours["recall_at_10"], "ref", theirs["recall_at_10"])
    assert abs(ours["recall_at_10"] - theirs["recall_at_10"]) <= 0.005


def test_nonfinite_input_rejected_on_device():
    """validate_vector_set's NaN/Inf contract (model.py:84-87) is checked on the device after the
    copy: same exception, same first (row, col) in row-major order, for fit (with and without
    sampling), hierarchical_fit and final_assign (checked per batch)."""
    import paper_2603_20009_b200 as skb
    x = make_blobs(3000, 96, 8, seed=1)
    bad = x.copy()
    bad[1700, 90] = np.inf
    bad[2200, 3] = np.nan
    bad[1700, 5] = np.nan
    for cfg in (skb.KMeansConfig(k=8, max_iters=2), skb.KMeansConfig(k=8, max_iters=2, sampling_fraction=0.5)):
        with pytest.raises(skb.NonFiniteValue) as e:
            skb.fit(bad, cfg)
        assert (e.value.row, e.value.col) == (1700, 5)
    with pytest.raises(skb.NonFiniteValue) as e:
        skb.hierarchical_fit(bad, skb.HierarchicalConfig(k_total=16, seed=0))
    assert (e.value.row, e.value.col) == (1700, 5)
    cfg = skb.KMeansConfig(k=8, max_iters=2)
    res = skb.fit(x, cfg)
    with pytest.raises(skb.NonFiniteValue) as e:
        skb.final_assign(bad, res, cfg, batch_rows=1000)
    assert (e.value.row, e.value.col) == (1700, 5)


@pytest.mark.parametrize("d", [96, 256])
def test_fit_exact_duplicates_vs_oracle(d):
    """Degenerate data: 60 distinct points each repeated 50 times, k = 80, so Forgy draws
    duplicate rows -> identical centroid rows -> exact distance ties, which must go to the lowest
    index (bitwise-identical distances, independent of GEMM rounding): iteration 1 must agree
    100 % and the empty duplicate clusters must produce the same number of splits.  After a
    split every member of a duplicated point is exactly equidistant (in exact arithmetic) from
    the pair r +- delta, so later assignments hinge on ulp-level rounding of the rotated
    coordinates (3xTF32 vs sgemm) and whole groups of 50 duplicates may legitimately flip, after
    which the split-heavy dynamics of this data take the two runs to different local optima
    (observed final WCSS 4002 here vs 5088 for the oracle): only the rounding-independent
    outcomes are compared."""
    import paper_2603_20009_b200 as skb
    from oracle import skm_ref
    base = make_blobs(60, d, 12, seed=40 + d)
    x = np.ascontiguousarray(np.repeat(base, 50, axis=0)[np.random.default_rng(d).permutation(3000)])
    cfg = skb.KMeansConfig(k=80, max_iters=6, seed=9)
    snaps = []
    res = skb.fit(x, cfg, inspect=lambda it, ctx: snaps.append(ctx["assignments"]))
    ref = skm_ref.fit(x, skm_ref.Params(k=80, max_iters=6, seed=9))
    assert np.array_equal(snaps[0], ref.snapshots[0]["assignments"])
    assert res.stats[0].n_empty_splits == ref.stats[0].n_empty_splits > 0
    assert np.isfinite(res.stats[-1].wcss) and len(np.unique(res.assignments)) <= cfg.k


@pytest.mark.parametrize("n,d,k", [(2000, 96, 1), (300, 128, 300), (257, 70, 256)])
def test_fit_edge_shapes_vs_oracle(n, d, k):
    """k = 1 (everything in one cluster), n == k (each row its own Forgy centroid: exact zero
    distances) and n = k + 1: assignments and centroids as the oracle's."""
    import paper_2603_20009_b200 as skb
    from oracle import skm_ref
    x = make_blobs(n, d, max(2, min(k, 40)), seed=n + k)
    cfg = skb.KMeansConfig(k=k, max_iters=4, seed=2)
    res = skb.fit(x, cfg)
    ref = skm_ref.fit(x, skm_ref.Params(k=k, max_iters=4, seed=2))
    assert float(np.mean(res.assignments == ref.assignments)) >= 0.999
    assert _rel_l2(res.centroids, ref.centroids) <= 1e-4
    assert res.terminated_by == ref.terminated_by
    if k == 1:
        assert not res.assignments.any()


@pytest.mark.parametrize("d", [3072, 4096, 8192])
def test_fit_large_d_vs_oracle(d):
    """Embedding sizes beyond c2 (d' = 384 / 512, 42 / 56 tail blocks: the scan's shared-memory
    staging sized at run time; d = 8192: 112-118 tail blocks, the one-warp scan) against the oracle: same d' trajectory, >= 99.9% assignment
    agreement every iteration, centroids within 1e-4."""
    import paper_2603_20009_b200 as skb
    from conftest import make_skewed_blobs
    from oracle import skm_ref
    x = make_skewed_blobs(3000, d, 60, seed=d)
    cfg = skb.KMeansConfig(k=48, max_iters=5, seed=1)
    snaps = []
    res = skb.fit(x, cfg, inspect=lambda it, ctx: snaps.append(ctx["assignments"]))
    ref = skm_ref.fit(x, skm_ref.Params(k=48, max_iters=5, seed=1))
    assert [s.d_prime for s in res.stats] == [s.d_prime for s in ref.stats]
    for it, (a, s) in enumerate(zip(snaps, ref.snapshots)):
        assert float(np.mean(a == s["assignments"])) >= 0.999, it
    assert _rel_l2(res.centroids, ref.centroids) <= 1e-4
    labels = skb.final_assign(x, res, cfg)
    assert float(np.mean(labels == res.assignments)) >= 0.999


@pytest.mark.parametrize("name", ["skewed", "low_d", "wide"])
def test_fit_portable_backend_bitwise(name):
    """gemm_backend="portable": every distance decision is settled with the reference's mul+add
    chain (no K blocking) instead of OpenBLAS's fma chain; the whole trajectory equals the real
    reference run with the same backend (tests/golden/make_golden_portable.py) bit for bit."""
    import importlib.util
    import paper_2603_20009_b200 as skb
    from conftest import make_blobs, make_skewed_blobs
    here = os.path.dirname(os.path.abspath(__file__))
    spec = importlib.util.spec_from_file_location("mgp", os.path.join(here, "golden", "make_golden_portable.py"))
    src = open(os.path.join(here, "golden", "make_golden_portable.py")).read()
    ns = {}
    exec(src[src.index("CASES = {"):src.index("}\n", src.index("CASES = {")) + 1], ns)
    gen, args, kw = ns["CASES"][name]
    g = np.load(os.path.join(here, "golden", "portable.npz"))
    x = make_blobs(*args) if gen == "blobs" else make_skewed_blobs(*args)
    snaps = []
    r = skb.fit(x, skb.KMeansConfig(gemm_backend="portable", **kw),
                inspect=lambda it, ctx: snaps.append(ctx["assignments"].copy()))
    assert [-1 if s.d_prime is None else s.d_prime for s in r.stats] == g[f"{name}_dp"].tolist()
    assert np.array_equal(np.stack(snaps), g[f"{name}_assign"])
    assert [s.survivors for s in r.stats] == g[f"{name}_surv"].tolist()
    assert [s.tail_dims_touched for s in r.stats] == g[f"{name}_tail"].tolist()
    assert [s.wcss for s in r.stats] == g[f"{name}_wcss"].tolist()
    assert np.array_equal(r.centroids_rotated, g[f"{name}_centroids_rotated"])
    # un-rotation of a tiny k x d matrix: OpenBLAS takes its small-matrix kernel there (another
    # summation order than the blocked driver the chain reproduces), so the last ulp may differ
    assert _rel_l2(r.centroids, g[f"{name}_centroids"]) <= 1e-6

"""CPU: pin the oracle (tests/ + bench infrastructure) against the golden fixtures produced by
the real reference (tests/golden/make_golden.py), and -- when the reference tree is present in
this container -- against the live reference package itself."""

import os
import sys

import numpy as np
import pytest

from conftest import make_blobs, make_skewed_blobs
from oracle import kernels_np as O
from oracle import skm_ref

HERE = os.path.dirname(os.path.abspath(__file__))
K = np.load(os.path.join(HERE, "golden", "kernels.npz"))
F = np.load(os.path.join(HERE, "golden", "fits.npz"))


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("sentinel", [0, 1])
def test_oracle_scan_and_seed_bitwise(seed, sentinel):
    from paper_2603_20009_b200.config import pdxify
    key = f"scan_s{seed}_{sentinel}"
    x, c, prev, vals, f = (K[key + s] for s in ("_x", "_c", "_prev", "_vals", "_f"))
    tau = np.empty(x.shape[0], np.float32)
    O.seed_thresholds(x, c, prev, tau)
    assert np.array_equal(tau, K[key + "_seedtau"])
    if sentinel:
        tau[:] = np.inf
    a = prev.copy()
    bank = pdxify(c, 25)
    sv, td = O.scan_bank(vals, x, bank.tail, bank.block_offsets, bank.block_dims, f, 25, 0, tau, a, bool(sentinel))
    assert np.array_equal(a, K[key + "_assign"])
    assert np.array_equal(tau, K[key + "_tau"])
    assert [sv, td] == K[key + "_counts"].tolist()


def test_oracle_accumulate_bitwise():
    sums = np.zeros((12, 64))
    counts = np.zeros(12, np.int64)
    O.accumulate_centroid_sums(K["acc_x"], K["acc_a"], sums, counts)
    assert np.array_equal(sums, K["acc_sums"])
    assert np.array_equal(counts, K["acc_counts"])


def _cases():
    src = open(os.path.join(HERE, "golden", "make_golden.py")).read()
    start = src.index("FIT_CASES = {")
    ns = {}
    exec(src[start:src.index("}\n", start) + 1], ns)
    return ns["FIT_CASES"]


def _make(spec):
    kind, n, d, centers, seed = spec[:5]
    if kind != "blobs":
        return make_skewed_blobs(n, d, centers, seed=seed)
    return make_blobs(n, d, centers, seed=seed) if len(spec) == 5 else make_blobs(n, d, centers, seed=seed,
                                                                                 spread=spec[5])


CASES = _cases()


@pytest.mark.parametrize("name", list(CASES))
def test_oracle_fit_reproduces_reference_trajectory(name):
    """Same NumPy/OpenBLAS GEMMs as the reference -> identical trajectory (this container)."""
    spec, kw = CASES[name]
    x = _make(spec)
    extra = {}
    if name.startswith("etr"):
        extra["etr"] = {"n_queries": 300, "top_k": 10}
    p = skm_ref.Params(**{k: v for k, v in kw.items()}, **extra)
    out = skm_ref.fit(x, p)
    snaps = np.stack([s["assignments"] for s in out.snapshots])
    assert np.array_equal(snaps, F[f"{name}_snap_assign"])
    assert np.array_equal(out.centroids, F[f"{name}_centroids"])
    assert [s.survivors for s in out.stats] == F[f"{name}_surv"].tolist()
    assert [s.tail_dims_touched for s in out.stats] == F[f"{name}_tail"].tolist()
    assert out.terminated_by == str(F[f"{name}_term"])
    assert out.recall_history == F[f"{name}_recall"].tolist()
    fa = skm_ref.final_assign(x, out, p)
    assert np.array_equal(fa, F[f"{name}_final"])


def test_oracle_hierarchical_matches_reference():
    x = make_blobs(6000, 128, 50, seed=31, spread=5.0, noise=0.8)
    cent, _, ga, _, plans = skm_ref.hierarchical_fit(x, 120, seed=2)
    assert cent.shape[0] == int(F["hier_k"])
    assert np.array_equal(ga, F["hier_assign"])
    assert np.array_equal(cent, F["hier_centroids"])


REF_SRC = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference tree not mounted")
def test_oracle_matches_live_reference_random_case():
    sys.path.insert(0, REF_SRC)
    os.environ.setdefault("SUPERKMEANS_KERNELS", "python")
    try:
        import superkmeans as ref
    finally:
        sys.path.remove(REF_SRC)
    x = make_skewed_blobs(3000, 160, 40, seed=99)
    snaps = []
    r = ref.fit(x, ref.KMeansConfig(k=20, max_iters=5, seed=4), inspect=lambda it, c: snaps.append(c["assignments"]))
    o = skm_ref.fit(x, skm_ref.Params(k=20, max_iters=5, seed=4))
    assert np.array_equal(np.stack(snaps), np.stack([s["assignments"] for s in o.snapshots]))
    assert np.array_equal(r.centroids, o.centroids)


def test_c_oracle_kernels_bitwise_equal_numpy_oracle():
    from oracle import kernels_c
    from paper_2603_20009_b200.config import pdxify
    if not kernels_c.available():
        pytest.skip("make -C oracle not run")
    for seed in range(3):
        for sentinel in (0, 1):
            key = f"scan_s{seed}_{sentinel}"
            x, c, prev, vals, f = (K[key + s] for s in ("_x", "_c", "_prev", "_vals", "_f"))
            tau = np.empty(x.shape[0], np.float32)
            kernels_c.seed_thresholds(x, c, prev, tau, 3)
            assert np.array_equal(tau, K[key + "_seedtau"])
            if sentinel:
                tau[:] = np.inf
            a = prev.copy()
            bank = pdxify(c, 25)
            sv, td = kernels_c.scan_bank(vals, x, bank.tail, bank.block_offsets, bank.block_dims, f, 25, 0, tau, a,
                                         bool(sentinel), 3)
            assert np.array_equal(a, K[key + "_assign"]) and np.array_equal(tau, K[key + "_tau"])
            assert [sv, td] == K[key + "_counts"].tolist()
    sums = np.zeros((12, 64))
    counts = np.zeros(12, np.int64)
    kernels_c.accumulate_centroid_sums(K["acc_x"], K["acc_a"], sums, counts)
    assert np.array_equal(sums, K["acc_sums"]) and np.array_equal(counts, K["acc_counts"])


PROBE_CASES = [(0, 12000, 48, 40, 64, 3), (1, 6000, 130, 25, 37, 4)]


@pytest.mark.parametrize("case,n,d,centers,k,seed", PROBE_CASES)
def test_oracle_probe_eval_matches_reference(case, n, d, centers, k, seed):
    """Oracle IVF probe evaluation == the reference's probe_eval / ivf_probe_search outputs
    (golden fixture), bitwise on this container's OpenBLAS."""
    P = np.load(os.path.join(HERE, "golden", "probes.npz"))
    key = f"p{case}"
    x = make_blobs(n, d, centers, seed=seed)
    lists = skm_ref.cluster_lists(P[key + "_assign"], k)
    for nprobe in (1, 3, 8):
        r = skm_ref.probe_eval(P[key + "_centroids"], lists, x, P[key + "_queries"], P[key + "_gt_idx"], 100, nprobe)
        assert r["recall_at_10"] == float(P[f"{key}_np{nprobe}_r10"])
        assert r["recall_at_100"] == float(P[f"{key}_np{nprobe}_r100"])
        assert r["vectors_explored_mean"] == float(P[f"{key}_np{nprobe}_explored"])
    for qi in range(5):
        ids, dist, ex = skm_ref.ivf_probe_search(P[key + "_centroids"], lists, x, P[key + "_queries"][qi], 3, 20)
        assert np.array_equal(ids, P[f"{key}_s{qi}_ids"])
        assert np.array_equal(dist, P[f"{key}_s{qi}_dist"])
        assert ex == int(P[f"{key}_s{qi}_ex"])
    # the tally formulation used on the device gives the same recall here
    hits = skm_ref.etr_hits(P[key + "_centroids"], x, P[key + "_assign"], P[key + "_queries"],
                            P[key + "_gt_idx"], 3, 10)
    assert skm_ref.recall_from_hits(hits, 10) == float(P[f"{key}_np3_r10"])

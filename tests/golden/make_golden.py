"""Generate the golden fixtures in tests/golden/ by running the REAL reference package.

Run here (the container that has /root/reference):
    PYTHONPATH=/root/reference/pkg/src SUPERKMEANS_KERNELS=python python tests/golden/make_golden.py

The reference is imported read-only; nothing under /root/reference is copied.  The fixtures
pin (a) the bit-exact kernel protocol outputs (scan/seed/accumulate/portable matmul) for
fixed inputs, (b) whole-fit trajectories (assignments, centroids, d', survivors, wcss,
prune rates, ETR recall, hierarchical plans) on seeded synthetic data, and (c) host math
(rotation, factors, cutoff controller).  GPU runs compare against these with the
north-star tolerances; CPU tests pin oracle/ against them bitwise where bits are
CPU-independent.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))  # tests/ for conftest generators
from conftest import make_blobs, make_skewed_blobs  # noqa: E402

import superkmeans as skm  # noqa: E402  (the reference, from PYTHONPATH)
from superkmeans import _kernels_py as RK  # noqa: E402
from superkmeans.distance import expand_to_sq_l2, matmul  # noqa: E402
from superkmeans.model import pdxify, tail_block_layout  # noqa: E402
from superkmeans.preprocess import compute_norms  # noqa: E402
from superkmeans.pruning import threshold_factors  # noqa: E402


def kernels():
    out = {}
    for seed in range(3):
        rng = np.random.default_rng(seed)
        n, k, d, dp = 123, 77, 200, 25
        x = rng.standard_normal((n, d)).astype(np.float32)
        c = rng.standard_normal((k, d)).astype(np.float32)
        prev = rng.integers(0, k, n).astype(np.int32)
        bank = pdxify(c, dp)
        vals = expand_to_sq_l2(matmul(x, c, dp), compute_norms(x, dp), compute_norms(c, dp), partial=True).values
        dims, bounds = tail_block_layout(d, dp)
        f = threshold_factors(d, dp, bounds, 2.1)
        for sentinel in (False, True):
            tau = np.empty(n, np.float32)
            RK.seed_thresholds(x, c, prev, tau, 1)
            seed_tau = tau.copy()
            if sentinel:
                tau[:] = np.inf
            a = prev.copy()
            sv, td = RK.scan_bank(vals, x, bank.tail, bank.block_offsets, bank.block_dims, f, dp, 0, tau, a,
                                  sentinel, 1)
            key = f"scan_s{seed}_{int(sentinel)}"
            out[key + "_x"] = x
            out[key + "_c"] = c
            out[key + "_prev"] = prev
            out[key + "_vals"] = vals
            out[key + "_f"] = f
            out[key + "_seedtau"] = seed_tau
            out[key + "_tau"] = tau
            out[key + "_assign"] = a
            out[key + "_counts"] = np.array([sv, td], np.int64)
    rng = np.random.default_rng(3)
    x = rng.standard_normal((500, 64)).astype(np.float32)
    a = rng.integers(0, 12, 500).astype(np.int32)
    sums = np.zeros((12, 64))
    counts = np.zeros(12, np.int64)
    RK.accumulate_centroid_sums(x, a, sums, counts)
    out.update(acc_x=x, acc_a=a, acc_sums=sums, acc_counts=counts)
    return out


def fit_case(name, x, cfg, out):
    snaps = []
    res = skm.fit(x, cfg, inspect=lambda it, ctx: snaps.append(ctx))
    out[f"{name}_centroids"] = res.centroids
    out[f"{name}_centroids_rot"] = res.centroids_rotated
    out[f"{name}_assign"] = res.assignments
    out[f"{name}_init"] = res.init_indices
    out[f"{name}_term"] = np.array(res.terminated_by)
    out[f"{name}_dpf"] = np.array(-1 if res.d_prime_final is None else res.d_prime_final)
    st = res.stats
    out[f"{name}_wcss"] = np.array([s.wcss for s in st])
    out[f"{name}_surv"] = np.array([s.survivors for s in st], np.int64)
    out[f"{name}_tail"] = np.array([s.tail_dims_touched for s in st], np.int64)
    out[f"{name}_dp"] = np.array([-1 if s.d_prime is None else s.d_prime for s in st], np.int64)
    out[f"{name}_rate"] = np.array([np.nan if s.prune_rate_after_gemm is None else s.prune_rate_after_gemm for s in st])
    out[f"{name}_changed"] = np.array([-1 if s.n_changed is None else s.n_changed for s in st], np.int64)
    out[f"{name}_splits"] = np.array([s.n_empty_splits for s in st], np.int64)
    out[f"{name}_recall"] = np.array(res.recall_history)
    out[f"{name}_snap_assign"] = np.stack([s["assignments"] for s in snaps])
    out[f"{name}_snap_cent"] = np.stack([s["centroids_rotated"] for s in snaps])
    if res.rotation.dim >= 512:  # large R: pinned by the SHA-256 of its float32 bytes
        import hashlib
        out[f"{name}_rotation_sha256"] = np.array(
            hashlib.sha256(np.ascontiguousarray(res.rotation.data, dtype=np.float32).tobytes()).hexdigest())
    else:
        out[f"{name}_rotation"] = res.rotation.data
    if res.sample_indices is not None:
        out[f"{name}_sidx"] = res.sample_indices
    fa = skm.final_assign(x, res, cfg)
    out[f"{name}_final"] = fa
    return res


FIT_CASES = {
    # name: (generator args, config kwargs)
    "blobs": (("blobs", 3000, 128, 32, 4), dict(k=24, max_iters=6, seed=5)),
    "sentinel": (("blobs", 2000, 96, 16, 6), dict(k=12, max_iters=5, seed=7, pruning_sentinel=True)),
    "smalld": (("blobs", 1500, 48, 8, 3), dict(k=8, max_iters=6, seed=1)),
    "skewed": (("skewed", 6000, 256, 128, 11), dict(k=64, max_iters=6, seed=5)),
    "ragged": (("blobs", 2500, 200, 20, 9), dict(k=30, max_iters=6, seed=2)),
    "sampled": (("blobs", 3000, 128, 24, 12), dict(k=16, max_iters=5, seed=3, sampling_fraction=0.5)),
    "etr": (("blobs", 4000, 128, 60, 21), dict(k=40, max_iters=12, seed=1)),
    "split": (("blobs", 1200, 96, 4, 13), dict(k=40, max_iters=5, seed=0)),
    "etr2": (("blobs", 12000, 128, 200, 3, 4.0), dict(k=100, max_iters=25, seed=1)),
    # the c2 dimensionality: 24 tail blocks of 64 after d' = 192, R from a 1536 x 1536 QR
    "wide": (("skewed", 8000, 1536, 128, 17), dict(k=64, max_iters=5, seed=3)),
    # the c3 family: d = 1024 with early termination by recall
    "etr_wide": (("skewed", 10000, 1024, 256, 23), dict(k=128, max_iters=10, seed=4)),
    # the c4 family: d = 768 (ragged last tail block after d' = 96: 10 x 64 + 32)
    "mid": (("skewed", 8000, 768, 160, 19), dict(k=96, max_iters=6, seed=8)),
    # sampling at d = 1024 (sample drawn before rotation, final_assign over all rows)
    "sampled_wide": (("skewed", 12000, 1024, 200, 27), dict(k=64, max_iters=6, seed=11, sampling_fraction=0.25)),
    # sentinel pruning (no seed thresholds) at d = 768
    "sentinel_wide": (("skewed", 6000, 768, 120, 31), dict(k=48, max_iters=5, seed=12, pruning_sentinel=True)),
}


def make_x(spec):
    kind, n, d, centers, seed = spec[:5]
    spread = spec[5] if len(spec) > 5 else None
    if kind == "blobs":
        return make_blobs(n, d, centers, seed=seed) if spread is None else \
            make_blobs(n, d, centers, seed=seed, spread=spread)
    return make_skewed_blobs(n, d, centers, seed=seed)


def fits():
    out = {}
    for name, (spec, kw) in FIT_CASES.items():
        x = make_x(spec)
        if name.startswith("etr"):
            kw = dict(kw, etr=skm.EtrConfig(n_queries=300, top_k=10))
        fit_case(name, x, skm.KMeansConfig(**kw), out)
    # hierarchical
    x = make_blobs(6000, 128, 50, seed=31, spread=5.0, noise=0.8)
    h = skm.hierarchical_fit(x, skm.HierarchicalConfig(k_total=120, seed=2))
    out["hier_centroids"] = h.centroids
    out["hier_assign"] = h.assignments
    out["hier_k"] = np.array(h.k)
    out["hier_meso_assign_snap"] = np.array(0)
    out.update(hier_wide())
    return out


def hier_wide():
    """Hierarchical at the c5 dimensionality (d = 1024, skewed blobs)."""
    x = make_skewed_blobs(*HIER_WIDE[0])
    h = skm.hierarchical_fit(x, skm.HierarchicalConfig(**HIER_WIDE[1]))
    return {"hierw_centroids": h.centroids, "hierw_assign": h.assignments, "hierw_k": np.array(h.k)}


HIER_WIDE = ((20000, 1024, 300, 29), dict(k_total=400, seed=6))


def hostmath():
    out = {}
    for d, s in ((64, 3), (200, 0), (96, 7)):
        out[f"rot_{d}_{s}"] = skm.generate_rotation(d, s).data
    from superkmeans.core import adjust_d_prime
    cfg = skm.KMeansConfig(k=4)
    cases = [(192, 0.96, 1536), (192, 0.99, 1536), (96, 0.90, 1536), (18, 0.999, 1536), (1400, 0.5, 1536),
             (25, 0.90, 200), (24, 0.98, 128), (32, 0.9476, 128), (24, 0.9713, 128)]
    out["adjust_in"] = np.array([[a, r, d] for a, r, d in cases])
    out["adjust_out"] = np.array([adjust_d_prime(a, r, cfg, d) for a, r, d in cases])
    dims, bounds = tail_block_layout(1536, 192)
    out["factors_1536_192"] = threshold_factors(1536, 192, bounds, 2.1)
    dims, bounds = tail_block_layout(200, 25)
    out["factors_200_25"] = threshold_factors(200, 25, bounds, 2.1)
    return out


def probes():
    """IVF probe evaluation (evaluation.py:86-105, 173-203) on a reference fit: inputs are
    regenerated from seeds by the tests; centroids, lists, GT and outputs are stored."""
    from superkmeans.evaluation import build_cluster_lists, ivf_probe_search, probe_eval
    out = {}
    for case, (n, d, centers, k, seed) in enumerate([(12000, 48, 40, 64, 3), (6000, 130, 25, 37, 4)]):
        x = make_blobs(n, d, centers, seed=seed)
        res = skm.fit(x, skm.KMeansConfig(k=k, max_iters=6, seed=seed))
        rng = np.random.default_rng([seed, 99])
        q_idx = rng.choice(n, size=150, replace=False)
        queries = (x[q_idx] + rng.standard_normal((150, d)).astype(np.float32) * 0.3).astype(np.float32)
        gt = skm.brute_force_topk(x, queries, 100)
        lists = build_cluster_lists(res.assignments, k)
        key = f"p{case}"
        out[key + "_centroids"] = res.centroids
        out[key + "_assign"] = res.assignments
        out[key + "_q_idx"] = q_idx
        out[key + "_queries"] = queries
        out[key + "_gt_idx"] = gt.indices
        out[key + "_gt_dist"] = gt.distances
        for nprobe in (1, 3, 8):
            r = probe_eval(res.centroids, lists, x, queries, gt, nprobe, top_ks=(10, 100))
            out[f"{key}_np{nprobe}_r10"] = np.float64(r["recall_at_10"])
            out[f"{key}_np{nprobe}_r100"] = np.float64(r["recall_at_100"])
            out[f"{key}_np{nprobe}_explored"] = np.float64(r["vectors_explored_mean"])
        for qi in range(5):
            ids, dist, ex = ivf_probe_search(res.centroids, lists, x, queries[qi], 3, 20)
            out[f"{key}_s{qi}_ids"] = ids
            out[f"{key}_s{qi}_dist"] = dist
            out[f"{key}_s{qi}_ex"] = np.int64(ex)
    return out


DATAIO_CASES = {
    # name: (format, n, d, mutations) -- files are rebuilt by tests/dataio_cases.py
    "fvecs_ok": ("fvecs", 9000, 37, []),
    "fbin_ok": ("fbin", 9000, 37, []),
    "fvecs_nan_row": ("fvecs", 9000, 20, [("val", 5000, 3, "nan")]),
    "fvecs_inf_first_chunk": ("fvecs", 9000, 20, [("val", 4095, 19, "inf"), ("dim", 4097, 0, 21)]),
    "fvecs_dim_vs_nan_same_chunk": ("fvecs", 9000, 20, [("val", 100, 2, "nan"), ("dim", 2000, 0, 7)]),
    "fbin_nan_two": ("fbin", 5000, 16, [("val", 4200, 15, "-inf"), ("val", 4100, 0, "nan")]),
    "fvecs_trailing_match": ("fvecs", 100, 8, [("trail", 4, 0, 8)]),
    "fvecs_trailing_mismatch": ("fvecs", 100, 8, [("trail", 12, 0, 9)]),
    "fvecs_trailing_short": ("fvecs", 100, 8, [("trail", 3, 0, 0)]),
    "fbin_truncated": ("fbin", 100, 8, [("truncate", 30, 0, 0)]),
    "fbin_bad_header": ("fbin", 10, 4, [("header", -1, 4, 0)]),
    "fvecs_bad_header": ("fvecs", 10, 4, [("header", 0, 0, 0)]),
}


def dataio_golden():
    """Reference outcomes of load_vectors on generated (valid and malformed) files, and the
    reference's SKMC / SKGT bytes for small models."""
    import tempfile
    sys.path.insert(0, os.path.dirname(HERE))
    from dataio_cases import build_case  # tests/dataio_cases.py
    from superkmeans import dataio as rdio
    from superkmeans.evaluation import GroundTruth as RGT
    out = {}
    with tempfile.TemporaryDirectory() as td:
        for name, spec in DATAIO_CASES.items():
            path = build_case(td, name, spec)
            try:
                x = rdio.load_vectors(path)
                out[f"{name}_outcome"] = np.array("ok")
                out[f"{name}_sum"] = np.float64(x.astype(np.float64).sum())
                out[f"{name}_shape"] = np.array(x.shape)
            except Exception as e:  # noqa: BLE001
                out[f"{name}_outcome"] = np.array(type(e).__name__)
                out[f"{name}_msg"] = np.array(str(e).replace(td, "<dir>"))
                out[f"{name}_rowcol"] = np.array([getattr(e, "row", -1), getattr(e, "col", -1)])
        rng = np.random.default_rng(5)
        c = rng.standard_normal((7, 5)).astype(np.float32)
        rdio.save_centroids(os.path.join(td, "m0.skmc"), c, 42)
        rdio.save_centroids(os.path.join(td, "m1.skmc"), c, 7, cluster_lists=[np.arange(i) for i in range(7)])
        gt = RGT(indices=rng.integers(0, 100, (3, 4)), distances=rng.random((3, 4)).astype(np.float32), k_gt=4)
        rdio.save_ground_truth(os.path.join(td, "g.skgt"), gt)
        out["model_centroids"] = c
        out["gt_indices"] = gt.indices
        out["gt_distances"] = gt.distances
        for f in ("m0.skmc", "m1.skmc", "g.skgt"):
            out["bytes_" + f.replace(".", "_")] = np.frombuffer(open(os.path.join(td, f), "rb").read(), np.uint8)
    return out


def cli_golden():
    """The reference CLI's fit / gt / eval reports on a small fbin dataset."""
    import json
    import tempfile
    from superkmeans import dataio as rdio
    from superkmeans.cli import main as rmain
    out = {}
    with tempfile.TemporaryDirectory() as td:
        x = make_blobs(2000, 48, 12, seed=8)
        path = os.path.join(td, "d.fbin")
        rdio.write_fbin(path, x)
        rep = os.path.join(td, "fit.json")
        model = os.path.join(td, "m.skmc")
        assert rmain(["fit", "--input", path, "--k", "12", "--iters", "4", "--seed", "9", "--eval-queries", "50",
                      "--out-centroids", model, "--report", rep]) == 0
        out["fit_report"] = np.array(json.dumps(rdio.RunReport.load(rep).comparable(), sort_keys=True))
        gtp = os.path.join(td, "g.skgt")
        assert rmain(["gt", "--input", path, "--n-queries", "40", "--topk", "20", "--seed", "3", "--out", gtp]) == 0
        out["gt_bytes"] = np.frombuffer(open(gtp, "rb").read(), np.uint8)
        rep2 = os.path.join(td, "eval.json")
        assert rmain(["eval", "--centroids", model, "--input", path, "--gt", gtp, "--n-queries", "40", "--seed", "3",
                      "--topk", "20", "--report", rep2]) == 0
        out["eval_report"] = np.array(json.dumps(rdio.RunReport.load(rep2).comparable(), sort_keys=True))
        out["model_bytes"] = np.frombuffer(open(model, "rb").read(), np.uint8)
    return out


def main():
    if "--only-fit" in sys.argv:  # (re)generate one FIT_CASES entry, keep the rest of fits.npz
        name = sys.argv[sys.argv.index("--only-fit") + 1]
        path = os.path.join(HERE, "fits.npz")
        out = {k: v for k, v in np.load(path).items() if not k.startswith(name + "_")}
        spec, kw = FIT_CASES[name]
        if name.startswith("etr"):
            kw = dict(kw, etr=skm.EtrConfig(n_queries=300, top_k=10))
        fit_case(name, make_x(spec), skm.KMeansConfig(**kw), out)
        np.savez_compressed(path, **out)
        return
    if "--only-hier-wide" in sys.argv:
        path = os.path.join(HERE, "fits.npz")
        out = {k: v for k, v in np.load(path).items() if not k.startswith("hierw_")}
        out.update(hier_wide())
        np.savez_compressed(path, **out)
        return
    if "--only-cli" in sys.argv:
        np.savez_compressed(os.path.join(HERE, "cli.npz"), **cli_golden())
        return
    if "--only-dataio" in sys.argv:
        np.savez_compressed(os.path.join(HERE, "dataio.npz"), **dataio_golden())
        return
    if "--only-probes" in sys.argv:
        np.savez_compressed(os.path.join(HERE, "probes.npz"), **probes())
        return
    np.savez_compressed(os.path.join(HERE, "probes.npz"), **probes())
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **kernels())
    np.savez_compressed(os.path.join(HERE, "hostmath.npz"), **hostmath())
    np.savez_compressed(os.path.join(HERE, "fits.npz"), **fits())
    for f in ("kernels.npz", "hostmath.npz", "fits.npz"):
        print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()

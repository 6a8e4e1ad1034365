"""Full-size golden trajectories for BASELINE configs c1 and c2, produced by the REAL reference.

Run here (the container that has the reference; the compiled Cython kernels are the reference's
own default backend):
    PYTHONPATH=baseline/_ref python tests/golden/make_golden_full.py c1 [c2 ...]

``baseline/_ref`` is the reference package installed from /root/reference/pkg with its own
setup.py (pip --target, compiled `_kernels` extension); nothing under /root/reference is copied
into the repository.  Inputs are regenerated from seeds with the reference's own generators
(tests/conftest.py restates pkg/tests/conftest.py:7-20), so the GPU box rebuilds the identical
matrix and only the outputs are stored:

* per iteration: d', survivors, tail dims touched, n_changed, wcss, prune rate, splits,
  cluster sizes (exact), and the assignments of every ``ROW_STRIDE``-th row;
* the final assignments (all rows), ``final_assign`` of all rows, init indices, rotation SHA-256;
* every ``CENT_STRIDE``-th final centroid (original space), plus f64 norms of all of them;
* the reference's wall clock and phase split (documents the CPU baseline of SURVEY 8d).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))  # tests/ for conftest generators
from conftest import make_blobs, make_skewed_blobs  # noqa: E402

import superkmeans as skm  # noqa: E402  (the reference, from PYTHONPATH)

# name: (generator, args, KMeansConfig kwargs, row stride, centroid stride)
FULL_CASES = {
    "c1": ("blobs", (100_000, 128, 256, 0), dict(k=256, max_iters=10, seed=0), 1, 1),
    "c2": ("skewed", (1_000_000, 1536, 8192, 0), dict(k=4096, max_iters=10, seed=0), 10, 8),
    "c4k1024": ("skewed", (1_000_000, 768, 2048, 0), dict(k=1024, max_iters=10, seed=0), 10, 4),
    "c4k4096": ("skewed", (1_000_000, 768, 8192, 0), dict(k=4096, max_iters=10, seed=0), 10, 8),
    "c4k16384": ("skewed", (1_000_000, 768, 32768, 0), dict(k=16384, max_iters=10, seed=0), 10, 16),
    # BASELINE c3: ETR on 1000 queries, recall@10; "etr" = (n_queries, top_k)
    "c3": ("skewed", (1_000_000, 1024, 32768, 0), dict(k=16384, max_iters=25, seed=0, etr=(1000, 10)), 10, 16),
}


def make_config(kw):
    kw = dict(kw)
    if "etr" in kw:
        nq, top_k = kw.pop("etr")
        kw["etr"] = skm.EtrConfig(n_queries=nq, top_k=top_k)
    return skm.KMeansConfig(**kw)


def make_input(name):
    gen, args, _, _, _ = FULL_CASES[name]
    return make_blobs(*args) if gen == "blobs" else make_skewed_blobs(*args)


def run(name):
    gen, args, kw, rs, cs = FULL_CASES[name]
    t0 = time.perf_counter()
    x = make_input(name)
    t_gen = time.perf_counter() - t0
    cfg = make_config(kw)
    snaps = []

    def inspect(it, ctx):
        a = ctx["assignments"]
        snaps.append(dict(sub=a[::rs].copy(), counts=np.bincount(a, minlength=cfg.k).astype(np.int64),
                          tau_sum=float(np.sum(ctx["best_sq_dist"], dtype=np.float64))))

    t0 = time.perf_counter()
    res = skm.fit(x, cfg, inspect=inspect)
    t_fit = time.perf_counter() - t0
    t0 = time.perf_counter()
    fa = skm.final_assign(x, res, cfg)
    t_fa = time.perf_counter() - t0
    st = res.stats
    adt = np.uint8 if cfg.k <= 256 else np.uint16
    out = dict(
        init=res.init_indices,
        rotation_sha256=np.array(hashlib.sha256(np.ascontiguousarray(res.rotation.data, np.float32).tobytes())
                                 .hexdigest()),
        term=np.array(res.terminated_by),
        dp=np.array([-1 if s.d_prime is None else s.d_prime for s in st], np.int64),
        surv=np.array([s.survivors for s in st], np.int64),
        tail=np.array([s.tail_dims_touched for s in st], np.int64),
        changed=np.array([-1 if s.n_changed is None else s.n_changed for s in st], np.int64),
        wcss=np.array([s.wcss for s in st]),
        rate=np.array([np.nan if s.prune_rate_after_gemm is None else s.prune_rate_after_gemm for s in st]),
        splits=np.array([s.n_empty_splits for s in st], np.int64),
        snap_sub=np.stack([s["sub"] for s in snaps]).astype(adt),
        snap_counts=np.stack([s["counts"] for s in snaps]),
        snap_tau_sum=np.array([s["tau_sum"] for s in snaps]),
        row_stride=np.int64(rs),
        assign=res.assignments.astype(adt),
        final=fa.astype(adt),
        cent_stride=np.int64(cs),
        cent_sub=res.centroids[::cs].copy(),
        cent_norms=np.linalg.norm(res.centroids.astype(np.float64), axis=1),
        cent_sum=res.centroids.astype(np.float64).sum(axis=0),
        dpf=np.int64(-1 if res.d_prime_final is None else res.d_prime_final),
        recall=np.array(res.recall_history),
    )
    import threadpoolctl
    meta = dict(case=name, generator=gen, args=args, config=kw, cpu_count=os.cpu_count(),
                numpy=np.__version__, blas=[{k: v for k, v in i.items() if k in ("internal_api", "version",
                                                                                  "num_threads")}
                                            for i in threadpoolctl.threadpool_info()],
                kernels=str(skm.__dict__.get("HAS_COMPILED", "")), gen_s=t_gen, fit_s=t_fit,
                final_assign_s=t_fa, phase_seconds=res.phase_seconds,
                iter_seconds=[dict(s.timings) for s in st], d_prime=out["dp"].tolist(),
                survivors=out["surv"].tolist(), n_changed=out["changed"].tolist(),
                prune_rate=out["rate"].tolist(), tail_dims=out["tail"].tolist())
    out["meta"] = np.array(json.dumps(meta))
    path = os.path.join(HERE, f"full_{name}.npz")
    np.savez_compressed(path, **out)
    print(json.dumps(meta, indent=1))
    print(path, os.path.getsize(path))


if __name__ == "__main__":
    from superkmeans import kernels as K
    assert K.HAS_COMPILED, "build the reference's compiled kernels first (baseline/_ref)"
    for name in sys.argv[1:]:
        run(name)

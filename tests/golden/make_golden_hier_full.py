"""Full-size hierarchical golden (c5's shape scaled to one host: 1M x 1024 skewed blobs,
k_total = 4096) produced by the REAL reference:
    PYTHONPATH=baseline/_ref python tests/golden/make_golden_hier_full.py
Stores the achieved k, every assignment (uint16), every 8th final centroid, all centroid norms
and the reference's wall clock.  The input is regenerated from the seeded generator."""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from conftest import make_skewed_blobs  # noqa: E402

import superkmeans as skm  # noqa: E402

N, D, K_TOTAL, SEED = 1_000_000, 1024, 4096, 0


def main():
    x = make_skewed_blobs(N, D, 2 * K_TOTAL, SEED)
    cfg = skm.HierarchicalConfig(k_total=K_TOTAL, seed=SEED)
    t0 = time.perf_counter()
    r = skm.hierarchical_fit(x, cfg)
    fit_s = time.perf_counter() - t0
    out = dict(k=np.int64(r.k), assign=r.assignments.astype(np.uint16), cent_sub=r.centroids[::8].copy(),
               cent_norms=np.linalg.norm(r.centroids.astype(np.float64), axis=1),
               meta=np.array(json.dumps(dict(n=N, d=D, k_total=K_TOTAL, seed=SEED, fit_s=fit_s,
                                             cpu_count=os.cpu_count(), meso_k=cfg.meso_k))))
    path = os.path.join(HERE, "full_hier.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), "k", r.k, "fit_s", round(fit_s, 1))


if __name__ == "__main__":
    main()

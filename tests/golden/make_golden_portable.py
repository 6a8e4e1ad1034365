"""Whole-fit trajectories of the REAL reference with gemm_backend="portable" (the Cython
mul+add chain, _kernels.pyx:122-142, instead of OpenBLAS sgemm for every distance GEMM):
    PYTHONPATH=baseline/_ref python tests/golden/make_golden_portable.py"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from conftest import make_blobs, make_skewed_blobs  # noqa: E402

import superkmeans as skm  # noqa: E402

CASES = {
    "skewed": ("skewed", (4000, 256, 40, 3), dict(k=32, max_iters=6, seed=2)),
    "low_d": ("blobs", (3000, 48, 30, 5), dict(k=24, max_iters=5, seed=4)),
    "wide": ("skewed", (2500, 768, 60, 7), dict(k=48, max_iters=6, seed=9)),
}


def main():
    out = {}
    for name, (gen, args, kw) in CASES.items():
        x = make_blobs(*args) if gen == "blobs" else make_skewed_blobs(*args)
        snaps = []
        r = skm.fit(x, skm.KMeansConfig(gemm_backend="portable", **kw),
                    inspect=lambda it, ctx: snaps.append(ctx["assignments"].copy()))
        out[f"{name}_assign"] = np.stack(snaps).astype(np.int32)
        out[f"{name}_centroids"] = r.centroids
        out[f"{name}_centroids_rotated"] = r.centroids_rotated
        out[f"{name}_dp"] = np.array([-1 if s.d_prime is None else s.d_prime for s in r.stats])
        out[f"{name}_surv"] = np.array([s.survivors for s in r.stats])
        out[f"{name}_tail"] = np.array([s.tail_dims_touched for s in r.stats])
        out[f"{name}_wcss"] = np.array([s.wcss for s in r.stats])
    np.savez_compressed(os.path.join(HERE, "portable.npz"), **out)
    print("ok", sorted(out))


if __name__ == "__main__":
    main()

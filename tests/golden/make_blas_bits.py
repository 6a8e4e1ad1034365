"""Golden bits of the reference's contraction backends on the survey container.

The reference multiplies with NumPy ``@`` (OpenBLAS 0.3.30 sgemm, SkylakeX kernel, threaded
driver on 8 cores) and reduces squared norms with ``np.einsum(..., dtype=float64)``
(preprocess.py:95-101).  This script records the SHA-256 of those outputs for seeded inputs so
the device's exact-chain GEMM (csrc/sgemm_chain.cuh) and einsum-order norms can be checked
bitwise on the GPU box, whose CPU may pick a different OpenBLAS kernel.  Run here:
    python tests/golden/make_blas_bits.py
"""

import hashlib
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

# (M, N, K, layout): "nt" = a @ b.T (distance.py:58-59), "nn" = a @ r (preprocess.py:43)
GEMM_CASES = [(300, 200, 16, "nt"), (300, 200, 130, "nt"), (300, 200, 448, "nt"), (300, 200, 449, "nt"),
              (300, 200, 1000, "nt"), (257, 384, 1536, "nt"), (500, 768, 768, "nn"), (400, 1024, 1024, "nn"),
              (300, 1536, 1536, "nn"), (64, 1536, 1536, "nt")]
NORM_CASES = [(3000, 7), (3000, 128), (3000, 130), (2000, 1536), (2000, 1023)]


def gemm_inputs(M, N, K, layout, seed):
    rng = np.random.default_rng([seed, M, N, K])
    a = (rng.standard_normal((M, K)) * rng.uniform(0.1, 10.0, (1, K))).astype(np.float32)
    b = rng.standard_normal((N, K) if layout == "nt" else (K, N)).astype(np.float32)
    return a, b


def norm_input(n, d, seed):
    rng = np.random.default_rng([seed, n, d])
    return (rng.standard_normal((n, d)) * rng.uniform(0.1, 100.0, (1, d))).astype(np.float32)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    out = {}
    for (M, N, K, lay) in GEMM_CASES:
        a, b = gemm_inputs(M, N, K, lay, 0)
        c = a @ b.T if lay == "nt" else a @ b
        out[f"gemm_{M}_{N}_{K}_{lay}"] = np.array(sha(c.astype(np.float32)))
    for (n, d) in NORM_CASES:
        m = norm_input(n, d, 0)
        for dims in (d, max(1, d // 3 + 1)):
            v = np.einsum("ij,ij->i", m[:, :dims], m[:, :dims], dtype=np.float64).astype(np.float32)
            out[f"norm_{n}_{d}_{dims}"] = np.array(sha(v))
    np.savez(os.path.join(HERE, "blas_bits.npz"), **out)
    print(len(out), "hashes")


if __name__ == "__main__":
    main()

"""One exact-chain rotation GEMM at the c2 shape (k-major R) for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_20009_b200.engine import chain_gemm  # noqa: E402

m, n, k = 1 << 20, 1536, 1536
a = torch.randn((m, k), device="cuda")
b = torch.randn((k, n), device="cuda")
out = torch.empty((m, n), device="cuda")
for _ in range(2):
    chain_gemm(a, b, m, n, k, out, 0, 448, b_kmajor=True)
torch.cuda.synchronize()

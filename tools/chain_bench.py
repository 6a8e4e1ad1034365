"""Throughput of the exact-chain GEMM (csrc/sgemm_chain.cuh) at the rotation shape."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_20009_b200.engine import chain_gemm  # noqa: E402

for (m, n, k) in ((1 << 20, 1536, 1536), (1 << 20, 1024, 1024), (1 << 20, 768, 768), (1 << 18, 4096, 192)):
    a = torch.randn((m, k), device="cuda")
    b = torch.randn((n, k), device="cuda")
    bk = b.t().contiguous()
    out = torch.empty((m, n), device="cuda")
    for kmaj in (False, True):
        bb = bk if kmaj else b
        for _ in range(2):
            chain_gemm(a, bb, m, n, k, out, 0, 448, b_kmajor=kmaj)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            chain_gemm(a, bb, m, n, k, out, 0, 448, b_kmajor=kmaj)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"chain gemm {m}x{n}x{k} kmajor={kmaj}: {ms:.2f} ms, {2.0 * m * n * k / ms / 1e9:.1f} TFLOP/s "
              f"(FFMA peak ~74)", flush=True)

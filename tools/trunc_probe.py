"""Is raw fp32 fed to tcgen05 kind::tf32 bit-identical to its explicit truncation (x & 0xFFFFE000)?
Compares GEMM_STORE(A_raw, 0, B_raw, 0) with GEMM_STORE(trunc(A), 0, trunc(B), 0) on random data,
and the full 3xTF32 product with hi = raw vs hi = truncated."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_20009_b200 import native  # noqa: E402
from paper_2603_20009_b200.api import _split  # noqa: E402
from paper_2603_20009_b200.engine import _gemm  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
for (m, n, k) in ((1000, 512, 256), (4096, 1024, 1536)):
    a = torch.randn((m, k), generator=g, device=dev) * torch.exp(torch.randn((m, k), generator=g, device=dev))
    b = torch.randn((n, k), generator=g, device=dev)
    a_hi, a_lo = _split(a, k)
    b_hi, b_lo = _split(b, k)
    z_a, z_b = torch.zeros_like(a), torch.zeros_like(b)
    o1 = torch.empty((m, n), device=dev)
    o2 = torch.empty((m, n), device=dev)
    _gemm(a, z_a, b, z_b, m, n, k, native.GEMM_STORE, out=o1)
    _gemm(a_hi, z_a, b_hi, z_b, m, n, k, native.GEMM_STORE, out=o2)
    same1 = torch.equal(o1, o2)
    _gemm(a, a_lo, b, b_lo, m, n, k, native.GEMM_STORE, out=o1)
    _gemm(a_hi, a_lo, b_hi, b_lo, m, n, k, native.GEMM_STORE, out=o2)
    same3 = torch.equal(o1, o2)
    print(f"{m}x{n}x{k}: hi-only raw==trunc {same1}; 3xTF32 raw-hi==trunc-hi {same3}", flush=True)

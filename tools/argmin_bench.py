"""Fixed-shape timing of the full-argmin GEMM (iteration 1) at the c2 shape.  python tools/argmin_bench.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_20009_b200 import native  # noqa: E402
from paper_2603_20009_b200.api import _split  # noqa: E402
from paper_2603_20009_b200.engine import _gemm  # noqa: E402

m, k, d = 1 << 20, 4096, 1536
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
x = torch.randn((m, d), generator=g, device=dev)
c = x[:k].clone() + 0.1
x_hi, x_lo = _split(x, d)
c_hi, c_lo = _split(c, d)
xs = (x.double() ** 2).sum(1).float()
ys = (c.double() ** 2).sum(1).float()
assign = torch.empty(m, dtype=torch.int32, device=dev)
tau = torch.empty(m, dtype=torch.float32, device=dev)
for rep in range(2):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        _gemm(x_hi, x_lo, c_hi, c_lo, m, k, d, native.GEMM_ARGMIN, xsq=xs, ysq=ys, assign=assign, tau=tau)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{os.environ.get('TAG', '')} argmin {m}x{k}x{d}: {ms:.2f} ms  {6.0 * m * k * d / ms / 1e9:.0f} TFLOP/s (tf32 MMA)  "
          f"checksum {int(assign.long().sum())}", flush=True)

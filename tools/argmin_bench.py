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
keys = torch.empty(m, dtype=torch.int64, device=dev)
ref = None
for split in (1, 4, 8, 16):
    def run():
        if split == 1:
            _gemm(x_hi, x_lo, c_hi, c_lo, m, k, d, native.GEMM_ARGMIN, xsq=xs, ysq=ys, assign=assign, tau=tau)
        else:
            keys.fill_(-1)
            _gemm(x_hi, x_lo, c_hi, c_lo, m, k, d, native.GEMM_ARGMIN, xsq=xs, ysq=ys, keys=keys, n_split=split)
            native.call("skm_decode_argmin_keys", keys.data_ptr(), m, assign.data_ptr(), tau.data_ptr(), None)
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    got = (assign.clone(), tau.clone())
    same = ref is None or (torch.equal(ref[0], got[0]) and torch.equal(ref[1], got[1]))
    ref = ref or got
    print(f"argmin split={split}: {ms:.2f} ms  {6.0 * m * k * d / ms / 1e9:.0f} TFLOP/s  identical={same}", flush=True)
out = torch.empty((m, d), dtype=torch.float32, device=dev)
for split in (1, 2, 3, 6):
    _gemm(x_hi, x_lo, c_hi[:d] if False else x_hi[:d], x_lo[:d], m, d, d, native.GEMM_STORE, out=out, n_split=split)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        _gemm(x_hi, x_lo, x_hi[:d], x_lo[:d], m, d, d, native.GEMM_STORE, out=out, n_split=split)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"store {m}x{d}x{d} split={split}: {ms:.2f} ms  {6.0 * m * d * d / ms / 1e9:.0f} TFLOP/s  "
          f"checksum {float(out[::4097].double().sum()):.6e}", flush=True)
for rep in range(0):
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

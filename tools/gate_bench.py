"""Fixed-shape timing of the gate GEMM (GEMM_GATE) at the c2 batch shape.
python tools/gate_bench.py [--dbg 1]   (SKM_GEMM_DBG is read once per process by the library)"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_20009_b200.synth import make_shard_device  # noqa: E402
from paper_2603_20009_b200 import native  # noqa: E402
from paper_2603_20009_b200.api import _split  # noqa: E402
from paper_2603_20009_b200.engine import _gemm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=132608)
ap.add_argument("--k", type=int, default=4096)
ap.add_argument("--d", type=int, default=1536)
ap.add_argument("--pass-frac", type=float, default=0.1)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
dev = torch.device("cuda", 0)
x = make_shard_device(a.m, a.d, 8192, 0, a.m, 0, dev)
c = x[torch.randperm(a.m, device=dev)[:a.k]].clone()
x_hi, x_lo = _split(x, a.d)
c_hi, c_lo = _split(c, a.d)
cap = a.k
cand = torch.empty((a.m, cap, 2), dtype=torch.int32, device=dev)
cand_cnt = torch.empty(a.m, dtype=torch.int32, device=dev)
for dp in (128, 192, 256, 384):
    for ext in (0, 64):
        xs = (x[:, :dp].double() ** 2).sum(1).float()
        ys = (c[:, :dp].double() ** 2).sum(1).float()
        xe = (x[:, dp:dp + ext].double() ** 2).sum(1).float()
        ye = (c[:, dp:dp + ext].double() ** 2).sum(1).float()
        dist = (xs[:256, None] + ys[None, :] - 2 * x[:256, :dp] @ c[:, :dp].T)
        thr = torch.full((a.m,), float(dist.flatten().kthvalue(int(a.pass_frac * dist.numel())).values), device=dev)
        thr1 = thr * (1.0 + ext / dp)
        kw = dict(xsq=xs, ysq=ys, thr=thr, cand=cand, cand_cnt=cand_cnt, cand_cap=cap)
        if ext:
            kw.update(ext_k=ext, xsq_ext=xe, ysq_ext=ye, thr1=thr1, cert_eps=3e-5)
        _gemm(x_hi, x_lo, c_hi, c_lo, a.m, a.k, dp, native.GEMM_GATE, **kw)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            _gemm(x_hi, x_lo, c_hi, c_lo, a.m, a.k, dp, native.GEMM_GATE, **kw)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        tf = 2.0 * 3 * a.m * a.k * (dp + ext) / ms / 1e9
        print(f"dbg={os.environ.get('SKM_GEMM_DBG', '0')} d'={dp:4d} ext={ext:2d}: {ms:.3f} ms  "
              f"{tf:.0f} TFLOP/s (tf32 MMA)  pass/row={float(cand_cnt.float().mean()):.0f}", flush=True)

"""ETR ground-truth pass at the c3 shape (1000 queries x 1M rows x 1024, top-10): fused chain
top-k kernel vs chain distance blocks + radix top-k."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_20009_b200 import etr  # noqa: E402

nq, n, d, k = 1000, 1_000_000, 1024, 10
x = torch.randn((n, d), device="cuda")
q = x[:nq].clone()
xs = (x.double() ** 2).sum(1).float()
qs = xs[:nq].clone()
for fused in (True, False):
    etr.FUSED_GT = fused
    for _ in range(2):
        etr.device_topk_distances(q, None, None, qs, x, None, None, xs, d, k)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        etr.device_topk_distances(q, None, None, qs, x, None, None, xs, d, k)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"fused={fused}: {ms:.1f} ms, {2.0 * nq * n * d / ms / 1e9:.1f} TFLOP/s", flush=True)

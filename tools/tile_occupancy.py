"""Diagnostic: after the gate GEMM of a steady-state iteration, what fraction of
(128-row M tile, 256-centroid N tile) pairs hold at least one gate survivor?  Rows in
cluster order (as the engine batches them).  python tools/tile_occupancy.py --n 200000"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_20009_b200.synth import make_shard_device  # noqa: E402
from paper_2603_20009_b200 import api, engine  # noqa: E402
from paper_2603_20009_b200.config import KMeansConfig  # noqa: E402
from paper_2603_20009_b200.hostmath import generate_rotation  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=200000)
ap.add_argument("--iters", type=int, default=5)
a = ap.parse_args()
dev = torch.device("cuda", 0)
x = make_shard_device(a.n, 1536, 8192, 0, a.n, 0, dev)
captured = {}
orig = engine.pruned_assign_pass


def spy(data, cents, ws, plan, order=None, **kw):
    orig(data, cents, ws, plan, order=order, **kw)
    bn = min(ws.batch, data.n)
    cnt = ws.cand_cnt[:bn].clone()
    idx = ws.cand[:bn, :, 0].clone()
    captured.setdefault("it", []).append((cnt, idx, ws.cap, cents.k, plan.d_prime))


engine.pruned_assign_pass = spy
api.fit_device(x, 1536, KMeansConfig(k=4096, max_iters=a.iters, seed=0), generate_rotation(1536, 0))
for it, (cnt, idx, cap, k, dp) in enumerate(captured["it"], start=2):
    n = cnt.numel()
    mt = (n + 127) // 128
    nt = (k + 255) // 256
    occ = torch.zeros(mt, nt, dtype=torch.bool, device=dev)
    uni = torch.zeros(mt, k, dtype=torch.bool, device=dev)
    valid = torch.arange(cap, device=dev)[None, :] < cnt.clamp(max=cap)[:, None]
    rows = torch.arange(n, device=dev)[:, None].expand(-1, cap)
    r, c = rows[valid], idx[valid].long()
    occ[r // 128, c // 256] = True
    uni[r // 128, c] = True
    geff = []
    for G in (2, 4, 8, 16):
        ng = n // G
        ug = torch.zeros(ng, k, dtype=torch.bool, device=dev)
        rr = r // G
        keep = rr < ng
        ug[rr[keep], c[keep]] = True
        geff.append(f"G{G}:{(cnt[:ng * G].clamp(max=cap).sum() / ug.sum()).item():.2f}")
    print(f"iter {it} sharing (pairs per union column) " + " ".join(geff))
    print(f"iter {it} d'={dp}: surv/row {cnt.float().mean():.1f}  alive N-tiles per M-tile "
          f"{occ.float().sum(1).mean():.2f}/{nt} ({100 * occ.float().mean():.1f}%)  union cols per M-tile "
          f"{uni.float().sum(1).mean():.0f}/{k}")

"""Diagnostic: histogram of the exact scan's survivors by the tail block where they are
pruned (last bin = completed), per pruned iteration.  python tools/prune_hist.py --n 200000"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

os.environ.setdefault("SKM_DIAG", "1")  # scan diagnostics read back per iteration

from paper_2603_20009_b200.synth import make_shard_device  # noqa: E402
from paper_2603_20009_b200 import api, engine  # noqa: E402
from paper_2603_20009_b200.config import KMeansConfig  # noqa: E402
from paper_2603_20009_b200.hostmath import generate_rotation  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=200000)
ap.add_argument("--iters", type=int, default=8)
a = ap.parse_args()
dev = torch.device("cuda", 0)
x = make_shard_device(a.n, 1536, 8192, 0, a.n, 0, dev)
engine.PRUNE_HIST = torch.zeros(48, dtype=torch.int64, device=dev)
orig = engine.pruned_assign_pass


def spy(*args, **kw):
    engine.PRUNE_HIST.zero_()
    orig(*args, **kw)
    h = engine.PRUNE_HIST.cpu().tolist()
    tot = sum(h)
    nz = [i for i, v in enumerate(h) if v]
    last = max(nz) if nz else 0
    print(f"survivors {tot}: " + " ".join(f"b{i}:{100 * h[i] / tot:.1f}%" for i in range(last + 1)))


engine.pruned_assign_pass = spy
api.fit_device(x, 1536, KMeansConfig(k=4096, max_iters=a.iters, seed=0), generate_rotation(1536, 0))

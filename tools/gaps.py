"""GPU idle gaps between consecutive native launches of one c2 fit (device-resident), from the
KernelTimer's CUDA events.  python tools/gaps.py --n 1000000"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_20009_b200.synth import make_shard_device  # noqa: E402
from paper_2603_20009_b200 import api, profiling  # noqa: E402
from paper_2603_20009_b200.config import KMeansConfig  # noqa: E402
from paper_2603_20009_b200.hostmath import generate_rotation  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
a = ap.parse_args()
dev = torch.device("cuda", 0)
x = make_shard_device(a.n, 1536, 8192, 0, a.n, 0, dev)
cfg = KMeansConfig(k=4096, max_iters=10, seed=0)
rot = generate_rotation(1536, 0)
api.fit_device(x, 1536, cfg, rot)  # warm
torch.cuda.synchronize()
prof = profiling.KernelTimer()
start = torch.cuda.Event(enable_timing=True)
stop = torch.cuda.Event(enable_timing=True)
start.record()
with profiling.active(prof):
    api.fit_device(x, 1536, cfg, rot)
stop.record()
torch.cuda.synchronize()
recs = prof.records
total = start.elapsed_time(stop)
busy = sum(a_.elapsed_time(b_) for _, a_, b_, _, _ in recs)
gaps = []
prev_name, prev_end = "start", start
for name, a_, b_, _, _ in recs:
    gaps.append((prev_end.elapsed_time(a_), prev_name, name))
    prev_name, prev_end = name, b_
gaps.append((prev_end.elapsed_time(stop), prev_name, "stop"))
print(f"fit {total:.1f} ms, launches {len(recs)}, in-launch {busy:.1f} ms, gaps {sum(g for g, _, _ in gaps):.1f} ms")
agg = {}
for g, p, n_ in gaps:
    key = f"{p} -> {n_}"
    s = agg.setdefault(key, [0, 0.0])
    s[0] += 1
    s[1] += g
for k_, (c, g) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:15]:
    print(f"  {g:7.2f} ms over {c:3d} gaps  {k_}")

"""SURVEY 8f-2/8f-3 at the c2 scale: write a 1M x 1536 .fbin (6 GB), then run the CLI
`fit` on it (file -> pinned double buffer -> device ingest + validation -> fit -> SKMC model +
report) and time each part.  python tools/run_cli_scale.py --dir /tmp/skm"""
import argparse
import json
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_20009_b200.synth import make_shard_device  # noqa: E402
from paper_2603_20009_b200.dataio import write_fbin  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dir", default="/tmp/skm_cli")
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--d", type=int, default=1536)
ap.add_argument("--k", type=int, default=4096)
a = ap.parse_args()
os.makedirs(a.dir, exist_ok=True)
path = os.path.join(a.dir, "base.fbin")
x = make_shard_device(a.n, a.d, 8192, 0, a.n, 0, torch.device("cuda", 0))[:, :a.d].cpu().numpy()
t0 = time.perf_counter()
write_fbin(path, x)
print(f"wrote {path}: {os.path.getsize(path) / 1e9:.2f} GB in {time.perf_counter() - t0:.2f}s", flush=True)
del x
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cmd = [sys.executable, "-m", "paper_2603_20009_b200", "fit", "--input", path, "--k", str(a.k), "--iters", "10",
       "--seed", "0", "--eval-queries", "1000", "--out-centroids", os.path.join(a.dir, "m.skmc"),
       "--report", os.path.join(a.dir, "fit.json")]
t0 = time.perf_counter()
r = subprocess.run(cmd, cwd=root, capture_output=True, text=True)
wall = time.perf_counter() - t0
print("cli rc", r.returncode, f"wall {wall:.2f}s (includes interpreter start and CUDA context)")
if r.returncode:
    print(r.stderr[-2000:])
else:
    rep = json.load(open(os.path.join(a.dir, "fit.json")))
    print("report keys", sorted(rep)[:12])
    print("final metrics", rep.get("final_metrics"))
    print("phases", {k: round(v, 3) for k, v in rep.get("phase_seconds", {}).items()} if "phase_seconds" in rep else "")

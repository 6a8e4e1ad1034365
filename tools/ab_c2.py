"""A/B timing of one library build (SKM_LIB=...) on the c2 shape: device-generated rows of the
c2 distribution (1M x 1536, k = 4096, 10 iterations), 1 warm-up + 3 timed device-resident fits.
Prints the median fit time, the per-phase split and a hash of the final assignments (builds of
the same ABI must agree bitwise).
   SKM_LIB=build_variants/x.so python tools/ab_c2.py"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_20009_b200 import api, profiling  # noqa: E402
from paper_2603_20009_b200.config import KMeansConfig  # noqa: E402
from paper_2603_20009_b200.hostmath import generate_rotation  # noqa: E402
from paper_2603_20009_b200.synth import make_shard_device  # noqa: E402

dev = torch.device("cuda", 0)
n, d, k = 1_000_000, 1536, 4096
x = make_shard_device(n, d, 8192, 0, n, 0, dev)
rot = generate_rotation(d, 0)
cfg = KMeansConfig(k=k, max_iters=10, seed=0)
times, phase, h = [], None, None
REPS = int(os.environ.get('AB_REPS', '4'))
for rep in range(REPS):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    mode = os.environ.get("AB_PROF", "0")  # 0: no kernel timer, 1: timer, 2: timer with a pooled reserve
    timer = profiling.KernelTimer(reserve=1600 if mode == "2" else 0)
    ctx = profiling.active(timer) if mode != "0" else profiling.active(None)
    with ctx:
        e0.record()
        res = api.fit_device(x, d, cfg, rot)
        e1.record()
    torch.cuda.synchronize()
    if rep:
        times.append(e0.elapsed_time(e1))
    phase = res.phase
    if os.environ.get("AB_VERBOSE"):
        ms = torch.cuda.memory_stats()
        print(f"rep {rep}: {e0.elapsed_time(e1):.1f} ms {[(kk, round(1e3 * v, 1)) for kk, v in phase.items()]} "
              f"cudaMalloc calls so far {ms.get('num_device_alloc')} frees {ms.get('num_device_free')}", flush=True)
    h = hashlib.sha1(res.loop.assign_dev.cpu().numpy().tobytes()).hexdigest()[:12] \
        if hasattr(res.loop, "assign_dev") else None
times.sort()
print(f"prof={os.environ.get('AB_PROF', '0')} lib={os.environ.get('SKM_LIB', 'default')} median_ms={times[len(times) // 2]:.1f} all={['%.1f' % t for t in times]} "
      f"phase_ms={ {kk: round(1e3 * v, 1) for kk, v in phase.items()} } assign_sha={h}", flush=True)

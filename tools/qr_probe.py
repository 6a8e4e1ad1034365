"""Host QR (generate_rotation) cost on this machine.  python tools/qr_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2603_20009_b200.hostmath import generate_rotation  # noqa: E402

print("cpus", os.cpu_count(), "OPENBLAS_NUM_THREADS", os.environ.get("OPENBLAS_NUM_THREADS"))
for d in (1024, 1536):
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        g = np.random.default_rng(0).standard_normal((d, d))
        t1 = time.perf_counter()
        q, r = np.linalg.qr(g)
        t2 = time.perf_counter()
        generate_rotation(d, 0)
        ts.append((1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (time.perf_counter() - t2)))
    print(d, "rng/qr/total ms", [tuple(round(v) for v in t) for t in ts])

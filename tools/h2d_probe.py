"""Host->device bandwidth options for a pageable numpy matrix.  python tools/h2d_probe.py --gb 4"""
import argparse
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

ap = argparse.ArgumentParser()
ap.add_argument("--gb", type=float, default=4.0)
ap.add_argument("--d", type=int, default=1024)
a = ap.parse_args()
n = int(a.gb * 2**30 / (4 * a.d))
x = np.random.default_rng(0).standard_normal((n, a.d), dtype=np.float32)
dev = torch.device("cuda", 0)
out = torch.empty((n, a.d), dtype=torch.float32, device=dev)
gb = x.nbytes / 1e9


def timed(name, fn, reps=2):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"{name:40s} {best * 1e3:8.1f} ms  {gb / best:6.1f} GB/s", flush=True)


timed("pageable copy_", lambda: out.copy_(torch.from_numpy(x)))
pin = torch.empty((n, a.d), dtype=torch.float32, pin_memory=True)
timed("pinned copy_ (DMA only)", lambda: out.copy_(pin, non_blocking=True))
timed("host memcpy 1 thread into pinned", lambda: np.copyto(pin.numpy(), x))
for th in (4, 8, 16):
    pool = ThreadPoolExecutor(th)
    pv = pin.numpy()

    def par():
        step = (n + th - 1) // th
        list(pool.map(lambda i: np.copyto(pv[i:i + step], x[i:i + step]), range(0, n, step)))
    timed(f"host memcpy {th} threads into pinned", par)

    for chunk_mb in (64, 256):
        rows = max(1, (chunk_mb << 20) // (4 * a.d))
        bufs = [torch.empty((rows, a.d), dtype=torch.float32, pin_memory=True) for _ in range(3)]
        evs = [None] * 3
        s = torch.cuda.Stream()

        def staged():
            for i, r0 in enumerate(range(0, n, rows)):
                b = i % 3
                if evs[b] is not None:
                    evs[b].synchronize()
                nb = min(rows, n - r0)
                bv = bufs[b].numpy()
                step = (nb + th - 1) // th
                list(pool.map(lambda j: np.copyto(bv[j:j + step], x[r0 + j:r0 + j + step]), range(0, nb, step)))
                with torch.cuda.stream(s):
                    out[r0:r0 + nb].copy_(bufs[b][:nb], non_blocking=True)
                    e = torch.cuda.Event()
                    e.record(s)
                    evs[b] = e
            torch.cuda.current_stream().wait_stream(s)
        timed(f"staged {th} thr {chunk_mb} MB x3", staged)
print("cpus", __import__("os").cpu_count())

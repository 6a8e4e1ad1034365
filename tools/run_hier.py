"""Time hierarchical_fit on device-generated skewed blobs.
   python tools/run_hier.py --n 10000000 --d 1024 --k 65536             (1 GPU, host NumPy entry)
   torchrun --nproc-per-node 8 --master-addr 127.0.0.1 tools/run_hier.py --n 10000000 --d 1024 --k 65536
   (rows sharded over the ranks, device-resident entry hierarchical_fit_device, NCCL)"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_20009_b200.synth import make_shard_device  # noqa: E402
from paper_2603_20009_b200 import profiling  # noqa: E402
from paper_2603_20009_b200.engine import Comm  # noqa: E402
from paper_2603_20009_b200.hierarchical import HierarchicalConfig, hierarchical_fit, hierarchical_fit_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--d", type=int, default=1024)
ap.add_argument("--k", type=int, default=16384)
ap.add_argument("--meso-k", type=int, default=None)
ap.add_argument("--device", action="store_true", help="device-resident entry even on one GPU")
a = ap.parse_args()
world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
if world > 1:
    import torch.distributed as dist
    dist.init_process_group("nccl", device_id=dev)
comm = Comm()
kw = dict(k_total=a.k, seed=0) | ({"meso_k": a.meso_k} if a.meso_k else {})
cfg = HierarchicalConfig(**kw)
device_entry = a.device or world > 1
lo, hi = comm.shard(a.n)
x = make_shard_device(a.n, a.d, 2 * a.k, lo, hi, 0, dev)
if device_entry:
    w = min(20000, hi - lo)  # warm-up on a small shard of every rank
    hierarchical_fit_device(x[:w].clone(), a.d, HierarchicalConfig(k_total=256, seed=0), comm=comm,
                            n_global=w * world, row_lo=rank * w)
else:
    x = x[:, :a.d].cpu().numpy()
    hierarchical_fit(x[:50000], HierarchicalConfig(k_total=256, seed=0))
torch.cuda.synchronize()
if world > 1:
    dist.barrier()
t0 = time.perf_counter()
prof = profiling.KernelTimer()
prof_host = None
if os.environ.get("SKM_CPROFILE"):
    import cProfile
    prof_host = cProfile.Profile()
    prof_host.enable()
with profiling.active(prof):
    if device_entry:
        r = hierarchical_fit_device(x, a.d, cfg, comm=comm, n_global=a.n, row_lo=lo)
    else:
        r = hierarchical_fit(x, cfg)
if prof_host is not None:
    prof_host.disable()
torch.cuda.synchronize()
wall = time.perf_counter() - t0
if world > 1:
    t = torch.tensor([wall], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    wall = float(t.item())
if rank == 0:
    print("kernels ms:", {kk: round(v["ms"], 1) for kk, v in sorted(prof.summary().items(), key=lambda kv: -kv[1]["ms"])})
    print(f"hierarchical n={a.n} d={a.d} k_total={a.k} ranks={world} entry={'device' if device_entry else 'host'}: "
          f"achieved k={r.k} wall={wall:.3f}s phase={ {k: round(v, 3) for k, v in r.phase_seconds.items()} }")
if prof_host is not None and rank == 0:
    import pstats
    pstats.Stats(prof_host).sort_stats("tottime").print_stats(30)
if world > 1:
    dist.destroy_process_group()

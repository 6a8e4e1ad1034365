"""Row-sharded data-parallel fit on the real device path with world size 2.

Only one GPU is available to this build, so both ranks share cuda:0 and talk over gloo
(which accepts CUDA tensors for collectives; point-to-point sends are staged through the host);
the device kernels, the sharded update (rank-ordered chained f64 sums or per-rank partials, then
the iteration's one packed allreduce -> finalize), the Forgy-row / ETR-query assembly, the sharded
ETR ground truth (per-rank top-k -> allgather -> stable merge) and the integer hit tally all run
exactly as under NCCL.  With the default exact_reduce the result is bitwise the single-process fit
(assignments, every per-iteration stat incl. wcss, centroids); with exact_reduce=False the integer
outputs must still match and the centroids equal up to the f64 association of the reduction."""

import os

import numpy as np
import pytest

from conftest import make_blobs

pytestmark = pytest.mark.gpu


def _run(rank, world, port, q, etr, exact, public):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2603_20009_b200 as skb
        from paper_2603_20009_b200 import api
        from paper_2603_20009_b200.config import EtrConfig, KMeansConfig
        from paper_2603_20009_b200.engine import Comm
        from paper_2603_20009_b200.hostmath import generate_rotation
        torch.cuda.set_device(0)
        x = make_blobs(40000, 128, 200, seed=3, spread=4.0)
        n, d = x.shape
        cfg = KMeansConfig(k=100, max_iters=8, seed=1, exact_reduce=exact,
                           etr=EtrConfig(n_queries=300, top_k=10) if etr else None)
        if public:  # the drop-in entry under an initialised process group shards by itself
            res = skb.fit(x, cfg)
            st = res.stats
            q.put((rank, {"assign": res.assignments, "lo": 0, "cent": res.centroids,
                          "dp": [s.d_prime for s in st], "changed": [s.n_changed for s in st],
                          "surv": [s.survivors for s in st], "wcss": [s.wcss for s in st],
                          "recall": res.recall_history, "term": res.terminated_by}))
            return
        comm = Comm()
        lo, hi = comm.shard(n)
        xd = api._h2d(x[lo:hi], torch.device("cuda", 0))
        res = api.fit_device(xd, d, cfg, generate_rotation(d, 1), comm=comm, n_global=n, row_lo=lo)
        st = res.loop.stats
        q.put((rank, {"assign": res.loop.assignments, "lo": lo,
                      "cent": res.centroids_dev[:, :d].cpu().numpy(),
                      "dp": [s.d_prime for s in st], "changed": [s.n_changed for s in st],
                      "surv": [s.survivors for s in st], "wcss": [s.wcss for s in st],
                      "recall": res.loop.recall_history, "term": res.loop.terminated_by}))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _spawn(world, port, fn, args):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=fn, args=(r, world, port, q) + args) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in ps:
        p.join(timeout=120)
    for r, v in res.items():
        assert isinstance(v, dict), v
    return res


@pytest.mark.parametrize("etr,exact,public", [(False, True, False), (True, True, False), (False, False, False),
                                              (False, True, True)])
def test_two_ranks_match_single_rank(etr, exact, public):
    outs = {}
    for world in (1, 2):
        port = 29600 + world + (os.getpid() % 400) + (100 if etr else 0) + (30 if exact else 0) + (60 if public else 0)
        outs[world] = _spawn(world, port, _run, (etr, exact, public))
    one = outs[1][0]
    two = outs[2]
    if public:
        for r in two:
            assert np.array_equal(two[r]["assign"], one["assign"])
    else:
        a2 = np.concatenate([two[r]["assign"] for r in sorted(two, key=lambda r: two[r]["lo"])])
        assert np.array_equal(a2, one["assign"])
    for r in two:
        for key in ("dp", "changed", "surv", "recall", "term"):
            assert two[r][key] == one[key], key
        if exact:  # rank-ordered sums + buffer-aligned shards: the 1-GPU result bit for bit
            assert two[r]["wcss"] == one["wcss"]
            assert np.array_equal(two[r]["cent"], one["cent"])
        else:
            rel = np.linalg.norm(two[r]["cent"] - one["cent"]) / np.linalg.norm(one["cent"])
            assert rel <= 1e-6, rel
    assert np.array_equal(two[0]["cent"], two[1]["cent"])  # replicas stay identical


def _run_hier(rank, world, port, q, layout, mode="owner"):
    import torch
    import torch.distributed as dist
    os.environ["SKM_HIER_FINE"] = mode  # read at import
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2603_20009_b200 as skb
        from paper_2603_20009_b200.engine import Comm
        torch.cuda.set_device(0)
        x = make_blobs(16000, 96, 150, seed=5, spread=4.0)
        if layout == "sorted":  # spatially coherent shards: many groups live on one rank only
            x = np.ascontiguousarray(x[np.argsort(x[:, 0], kind="stable")])
        res = skb.hierarchical_fit(x, skb.HierarchicalConfig(k_total=400, seed=7), comm=Comm())
        q.put((rank, {"assign": res.assignments, "cent": res.centroids_rotated, "k": res.k,
                      "dp": [s.d_prime for s in res.stats], "work": res.work}))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("layout,ranks,mode", [("shuffled", 2, "owner"), ("sorted", 3, "owner"),
                                               ("sorted", 2, "sharded"), ("shuffled", 3, "sharded")])
def test_hierarchical_two_ranks_match_single_rank(layout, ranks, mode):
    """Multi-rank hierarchical fit (2 and 3 ranks: uneven shards; fine phase by group owner after
    one all-to-all, or as sharded loops) (BASELINE c5's data-sharded form): meso loop sharded,
    every group fitted as a sharded loop over its members' rank-local rows.  Integer outputs
    equal the single-process fit, centroids up to the cross-rank f64 summation order, replicas
    identical."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    outs = {}
    for world in (1, ranks):
        q = ctx.Queue()
        port = 29900 + world + (os.getpid() % 400) + (50 if layout == "sorted" else 0) + 10 * ranks + \
            (100 if mode == "owner" else 0)
        ps = [ctx.Process(target=_run_hier, args=(r, world, port, q, layout, mode)) for r in range(world)]
        for p in ps:
            p.start()
        res = dict(q.get(timeout=600) for _ in range(world))
        for p in ps:
            p.join(timeout=120)
        for r, v in res.items():
            assert isinstance(v, dict), v
        outs[world] = res
    one = outs[1][0]
    for r, two in outs[ranks].items():
        assert two["k"] == one["k"]
        assert two["dp"] == one["dp"]
        assert np.array_equal(two["assign"], one["assign"])
        assert two["work"] == one["work"]
        rel = np.linalg.norm(two["cent"] - one["cent"]) / np.linalg.norm(one["cent"])
        assert rel <= 1e-6, rel
        # owner: every group fitted on one rank exactly as on one GPU; sharded: the batched fine
        # loop chains each centroid's f64 member sums in rank order (exact_reduce) -- both bitwise
        assert np.array_equal(two["cent"], one["cent"])
    for r in range(1, ranks):
        assert np.array_equal(outs[ranks][0]["cent"], outs[ranks][r]["cent"])


def test_bench_two_ranks_runs():
    """bench.py's sharded path end to end under torchrun (2 ranks sharing cuda:0 over gloo):
    one JSON line from rank 0 with the whole-job metric, e2e and roofline objects."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SKM_BENCH_DEVICE="0", SKM_DIST_BACKEND="gloo")
    port = 29700 + os.getpid() % 200
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", "bench.py", "--gpus", "2", "--steps", "1",
           "--warmup", "3", "--no-cpu-baseline", "--rows", "60000", "--k", "256"]
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0 and d["roofline"]["achieved"] > 0

"""CPU, world_size 2 over gloo: the host side of the row-sharded data-parallel path.

Covers what the N>1 device run relies on: contiguous shards that tile [0, n), one packed
allreduce of [ordered f64 sums | counts] per iteration reproducing the single-process update,
the Forgy-row assembly by allreduce, the ETR integer tally summing across shards, and the
packed scalar reduction (wcss, n_changed, survivors, tail dims)."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import make_blobs


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import kernels_np as O
        from oracle import skm_ref
        from paper_2603_20009_b200.engine import Comm
        comm = Comm()
        assert (comm.rank, comm.world) == (rank, world)
        n, d, k = 3001, 24, 13
        x = make_blobs(n, d, 7, seed=1)
        a = np.random.default_rng(2).integers(0, k, n).astype(np.int32)
        lo, hi = comm.shard(n)
        # 1. shards tile [0, n)
        bounds = torch.tensor([lo, hi], dtype=torch.int64)
        allb = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allb, bounds)
        spans = sorted(tuple(b.tolist()) for b in allb)
        assert spans[0][0] == 0 and spans[-1][1] == n
        assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
        # 2. packed [sums | counts] allreduce == global update (up to f64 summation order)
        sums = np.zeros((k, d))
        counts = np.zeros(k, np.int64)
        O.accumulate_centroid_sums(x[lo:hi], a[lo:hi], sums, counts)
        packed = torch.tensor(np.concatenate([sums.ravel(), counts.astype(np.float64)]))
        comm.allreduce_(packed)
        g_sums = packed[: k * d].numpy().reshape(k, d)
        g_counts = packed[k * d:].round().to(torch.int64).numpy()
        ref_c, ref_n = skm_ref.update(x, a, k, np.zeros((k, d), np.float32))
        assert np.array_equal(g_counts, ref_n)
        cent = np.where(g_counts[:, None] > 0, (g_sums / np.maximum(g_counts, 1)[:, None]).astype(np.float32), 0)
        assert np.max(np.abs(cent - ref_c)) <= 1e-6 * max(1.0, np.abs(ref_c).max())
        # 3. Forgy rows assembled by allreduce of owner-filled rows
        init = np.random.default_rng([0, 2]).choice(n, size=k, replace=False)
        rows = torch.zeros((k, d))
        mine = np.flatnonzero((init >= lo) & (init < hi))
        rows[mine] = torch.from_numpy(x[init[mine]])
        comm.allreduce_(rows)
        assert np.array_equal(rows.numpy(), x[init])
        # 4. ETR: per-shard integer hits sum to the global tally
        c = x[init].copy()
        assign = np.argmin(((x[:, None, :] - c[None]) ** 2).sum(-1), axis=1).astype(np.int32)
        qs = x[:40].copy()
        gi, _ = skm_ref.brute_force_topk(x, qs, 5)
        probe = np.argsort(((qs[:, None, :] - c[None]) ** 2).sum(-1), axis=1, kind="stable")[:, :3]
        local = np.array([sum(1 for g in gi[i] if lo <= g < hi and assign[g] in probe[i]) for i in range(40)])
        h = torch.tensor(local, dtype=torch.int64)
        comm.allreduce_(h)
        glob = np.array([sum(1 for g in gi[i] if assign[g] in probe[i]) for i in range(40)])
        assert np.array_equal(h.numpy(), glob)
        # 5. packed scalars
        tau = np.random.default_rng(5).random(n).astype(np.float32)
        s = torch.tensor([float(np.sum(tau[lo:hi], dtype=np.float64)), 3.0, 7.0, 11.0], dtype=torch.float64)
        comm.allreduce_(s)
        assert s[1:].tolist() == [3.0 * world, 7.0 * world, 11.0 * world]
        assert abs(s[0].item() - float(np.sum(tau, dtype=np.float64))) <= 1e-9 * n
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_row_sharded_host_path_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(msg == "ok" for _, msg in res), res

"""Host logic of the sharded hierarchical fine phase (hierarchical.group_plans), no GPU.

Rows are split into contiguous rank shards; each rank's stable cluster sort gives its local
member lists.  The plans must (1) agree on every rank about group sizes, k_i and centroid
offsets, and (2) place each rank's members so that concatenating them in rank order is the
reference's member list np.flatnonzero(meso_assign == g) (hierarchical.py:118-141,
build_cluster_lists evaluation.py:78-83)."""

import numpy as np
import pytest

from paper_2603_20009_b200.hierarchical import _fine_k, group_plans


def _rank_state(assign, mk, lo, hi):
    a = assign[lo:hi]
    order = np.argsort(a, kind="stable")  # the device cluster sort is stable
    counts = np.bincount(a, minlength=mk)
    offsets = np.concatenate(([0], np.cumsum(counts)[:-1]))
    return order, counts, offsets


@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("layout", ["random", "sorted", "empty_groups"])
def test_group_plans_rebuild_reference_member_lists(world, layout):
    rng = np.random.default_rng(world * 10 + len(layout))
    n, mk = 5003, 37
    assign = rng.integers(0, mk, n)
    if layout == "sorted":
        assign = np.sort(assign)  # groups concentrated on single ranks
    if layout == "empty_groups":
        assign[(assign % 5) == 0] = 1  # some groups empty everywhere
        assign[7] = 35                # a singleton group
        assign[assign == 35] = 36
        assign[7] = 35
    per = (n + world - 1) // world
    shards = [(min(n, r * per), min(n, (r + 1) * per)) for r in range(world)]
    states = [_rank_state(assign, mk, lo, hi) for lo, hi in shards]
    table = np.stack([s[1] for s in states])
    all_plans = [group_plans(table, r, states[r][2]) for r in range(world)]
    # (1) identical global view on every rank
    glob = [[(p[0], p[3], p[5], p[6]) for p in plans] for plans, _ in all_plans]
    assert all(g == glob[0] for g in glob)
    assert all(t == all_plans[0][1] for _, t in all_plans)
    ref_groups = [g for g in range(mk) if np.any(assign == g)]
    assert [p[0] for p in all_plans[0][0]] == ref_groups
    off = 0
    for gi, n_i, k_i, o_cent in glob[0]:
        assert n_i == int(np.sum(assign == gi)) and k_i == _fine_k(n_i) and o_cent == off
        off += k_i
    assert all_plans[0][1] == off
    # (2) rank-local members, concatenated in rank order, are the reference member list
    for idx in range(len(ref_groups)):
        gi = ref_groups[idx]
        members = []
        for r, (lo, _) in enumerate(shards):
            p = all_plans[r][0][idx]
            assert p[4] == len(members)  # this rank's first member index inside the group
            order = states[r][0]
            members.extend((lo + order[p[1]:p[1] + p[2]]).tolist())
        assert members == np.flatnonzero(assign == gi).tolist()


def test_group_owners_lpt_deterministic():
    from paper_2603_20009_b200.hierarchical import group_owners
    sizes = np.array([5, 1, 9, 3, 0, 7])
    assert group_owners(sizes, 2).tolist() == [1, 0, 0, 0, 1, 1]
    rng = np.random.default_rng(0)
    sizes = rng.integers(0, 1000, 300)
    for world in (2, 3, 8):
        own = group_owners(sizes, world)
        loads = np.bincount(own, weights=sizes, minlength=world)
        assert loads.max() - loads.min() <= sizes.max()  # LPT bound


def _exchange_worker(rank, world, port, q):
    import os
    import types
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_20009_b200.engine import Comm
        from paper_2603_20009_b200.hierarchical import _exchange_groups, group_owners
        rng = np.random.default_rng(42)
        n, mk, ld = 997, 23, 8
        assign = rng.integers(0, mk, n)
        assign[assign == 4] = 5  # an empty group
        x = torch.arange(n * ld, dtype=torch.float32).reshape(n, ld)  # row r holds r*ld..
        comm = Comm()
        lo, hi = comm.shard(n)
        a_l = assign[lo:hi]
        order = torch.as_tensor(np.argsort(a_l, kind="stable").astype(np.int32))
        counts = np.bincount(a_l, minlength=mk)
        offs = np.concatenate(([0], np.cumsum(counts)[:-1]))
        from paper_2603_20009_b200.engine import shard_bounds
        table = np.stack([np.bincount(assign[slice(*shard_bounds(n, world, r))], minlength=mk) for r in range(world)])
        owner = group_owners(table.sum(axis=0), world)
        data = types.SimpleNamespace(x=x[lo:hi], n=hi - lo, ld=ld)
        rows, gids, goff = _exchange_groups(data, order, offs, table, owner, comm, lo)
        q.put((rank, {"rows": rows.numpy(), "gids": gids.numpy(), "goff": goff, "owner": owner, "assign": assign,
                      "x": x.numpy()}))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_groups_gives_owners_their_groups_in_row_order(world):
    import os
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + world + os.getpid() % 300
    ps = [ctx.Process(target=_exchange_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    seen = []
    for r, v in res.items():
        assert isinstance(v, dict), v
        assign, owner, x = v["assign"], v["owner"], v["x"]
        mine = [g for g in range(len(owner)) if owner[g] == r and np.any(assign == g)]
        assert sorted(v["goff"]) == mine
        for g in mine:
            members = np.flatnonzero(assign == g)
            o = v["goff"][g]
            assert np.array_equal(v["gids"][o:o + members.size], members)
            assert np.array_equal(v["rows"][o:o + members.size], x[members])
        seen.extend(v["gids"].tolist())
    assert sorted(seen) == list(range(len(res[0]["assign"])))  # every row moved exactly once


def test_grouped_tile_ranges_and_layout():
    """grouped.py host helpers: each 128-row tile's N range is the union of its rows' group
    column ranges (ragged last tile included); the layout's per-row ranges follow the groups."""
    import numpy as np
    import torch
    from paper_2603_20009_b200.grouped import GroupLayout, tile_ranges
    sizes = np.array([5, 300, 2, 129, 1000, 64], dtype=np.int64)
    ks = np.array([2, 17, 1, 11, 32, 8], dtype=np.int64)
    lay = GroupLayout(sizes, ks, torch.device("cpu"))
    assert lay.n == sizes.sum() and lay.k_total == ks.sum()
    g = np.repeat(np.arange(len(sizes)), sizes)
    c0 = np.concatenate(([0], np.cumsum(ks)[:-1]))
    want = np.stack([c0[g], c0[g] + ks[g]], 1)
    assert np.array_equal(lay.row_crange.numpy(), want)
    assert np.array_equal(lay.row_group.numpy(), g)
    tr = tile_ranges(lay.row_crange).numpy()
    assert tr.shape == ((lay.n + 127) // 128, 2)
    for t in range(tr.shape[0]):
        rows = want[t * 128:(t + 1) * 128]
        assert tr[t, 0] == rows[:, 0].min() and tr[t, 1] == rows[:, 1].max()
    # a subset of rows (a d' class) keeps the same contract
    sub = lay.row_crange[torch.arange(3, 700, 3)]
    trs = tile_ranges(sub.contiguous()).numpy()
    s = sub.numpy()
    for t in range(trs.shape[0]):
        rows = s[t * 128:(t + 1) * 128]
        assert trs[t, 0] == rows[:, 0].min() and trs[t, 1] == rows[:, 1].max()

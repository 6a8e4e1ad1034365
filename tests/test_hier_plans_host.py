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

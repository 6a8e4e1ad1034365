"""Group-batched Lloyd loops: the hierarchical fine phase as ONE device loop over every group.

The reference fits every meso group with its own ``_fit_rotated`` (hierarchical.py:129-147):
round(sqrt(n_i)) centroids, ``fine_iters`` iterations, seed ``SeedSequence([seed, 5, gi])``, its own
d' controller, split RNG and convergence test.  Here all groups advance together, one launch per
kernel per iteration ("batched K2/K3/K4 over groups"):

  * rows are laid out group by group (the meso phase's stable cluster order), centroids are one
    concatenated matrix, group g owning columns [c0_g, c0_g + k_g);
  * iteration 1 is ONE tensor-core ARGMIN over all rows in which row i only sees its group's
    columns (``row_crange``) and each 128-row tile walks only the N tiles its rows' groups cover
    (``tile_nrange``); the exact settle of near-ties runs on the same grouped ranges;
  * pruned iterations run one grouped GATE GEMM + scan per distinct d' among the active groups
    (every group starts at the same d' and the controller moves each by +-20 %, so there are a
    few classes); the scan adds each row's survivors / dims touched / changed into its group's
    counters;
  * the update is the ordinary stable cluster sort + ordered member sums over all centroids;
    a group that stops (converged, or its last iteration) has its centroids frozen at that
    point, exactly where its own loop would have left them, and its rows leave the passes;
    splits and d' are decided per group on the host from one readback per iteration.

Every per-row operation is the single-group loop's (engine.py), so each group's centroids and
assignments are bitwise those of its own fit -- and of the reference.  Row-sharded
every rank runs the same loop on its members, with one packed allreduce per iteration.
"""

from __future__ import annotations

import numpy as np
import torch

from . import native
from .config import KMeansConfig, WorkCounters, initial_d_prime, pruning_supported
from .device import padded_ld, ptr, stream_handle
from .engine import (
    DEFER_CERT,
    FLAT_MAX_CHANGED,
    GATE_KPAIR,
    NOWIN_SURV_FRAC,
    SCAN_FLAT,
    Centroids,
    DeviceData,
    PrunePlan,
    Workspace,
    _gemm,
    cert_extension,
    chained_cluster_sums,
    tc_kappa,
)
from .hostmath import SPLIT_EPS, adjust_d_prime, init_indices, plan_splits, prune_rate_from_totals


def tile_ranges(crange: torch.Tensor) -> torch.Tensor:
    """[ceil(m / 128), 2] int32: the union of the column ranges of each 128-row tile."""
    m = crange.shape[0]
    tiles = (m + 127) // 128
    pad = tiles * 128 - m
    cr = crange if pad == 0 else torch.cat([crange, crange[-1:].expand(pad, 2)], 0)
    cr = cr.view(tiles, 128, 2)
    return torch.stack([cr[:, :, 0].amin(1), cr[:, :, 1].amax(1)], 1).to(torch.int32).contiguous()


class GroupLayout:
    """Groups of a row-contiguous layout: group g = rows [starts[g], starts[g] + sizes[g]),
    centroid columns [c0[g], c0[g] + ks[g])."""

    def __init__(self, sizes: np.ndarray, ks: np.ndarray, dev):
        self.sizes = np.asarray(sizes, dtype=np.int64)
        self.ks = np.asarray(ks, dtype=np.int64)
        self.G = len(self.sizes)
        self.starts = np.concatenate(([0], np.cumsum(self.sizes)[:-1])).astype(np.int64)
        self.c0 = np.concatenate(([0], np.cumsum(self.ks)[:-1])).astype(np.int64)
        self.n = int(self.sizes.sum())
        self.k_total = int(self.ks.sum())
        grange = np.stack([self.c0, self.c0 + self.ks], 1).astype(np.int32)
        self.grange = torch.from_numpy(grange).to(dev)
        self.row_group = torch.repeat_interleave(torch.arange(self.G, dtype=torch.int32, device=dev),
                                                 torch.from_numpy(self.sizes).to(dev))
        self.row_crange = self.grange[self.row_group.long()].contiguous()


def _grouped_full_assign(data: DeviceData, cents: Centroids, ws: Workspace, lay: GroupLayout, r0: int, r1: int) -> None:
    """Exact argmin of rows [r0, r1) over their own groups' centroids (engine.full_assign_pass
    with grouped column ranges)."""
    n = r1 - r0
    if n <= 0:
        return
    d = data.d
    st = stream_handle()
    xsq = data.norms(d)[r0:r1]
    crange = lay.row_crange[r0:r1]
    top = ws.top_records(n)
    _gemm(data.hi[r0:r1], data.lo[r0:r1], cents.hi, cents.lo, n, cents.k, d, native.GEMM_ARGMIN,
          xsq=xsq, ysq=cents.ysq, top=top, n_split=1, row_crange=crange, tile_nrange=tile_ranges(crange))
    assign, tau = ws.assign[r0:r1], ws.tau[r0:r1]
    ws.amb_count.zero_()
    native.call("skm_argmin_merge", ptr(top), 1, n, ptr(xsq), ptr(cents.ysq_max), float(tc_kappa(d, GATE_KPAIR)),
                ptr(assign), ptr(tau), ptr(ws.amb_rows), ptr(ws.amb_count), st)
    native.call("skm_exact_pair_dist", ptr(data.x[r0:r1]), data.ld, ptr(cents.c), cents.ld, ptr(assign), n, d,
                ptr(xsq), ptr(cents.ysq), ws.chain_flavour, ws.chain_q, ptr(tau), st, nbytes=4.0 * n * d)
    n_amb = int(ws.amb_count.item())
    if not n_amb:
        return
    # near-ties: every column of the row's group whose exact distance may tie or beat the best,
    # then the reference's chain distance of each (rows sorted so tiles stay inside few groups)
    glob_all = (torch.sort(ws.amb_rows[:n_amb]).values + r0).to(torch.int32)
    xsq_all = data.norms(d)
    kap = tc_kappa(d, GATE_KPAIR)
    for c0 in range(0, n_amb, ws.batch):
        glob = glob_all[c0:c0 + ws.batch].contiguous()
        m = int(glob.numel())
        thr, xs = ws.bthr[:m], ws.bx[:m]
        native.call("skm_argmin_candidates", ptr(glob), m, ptr(ws.tau), ptr(xsq_all), ptr(cents.ysq_max),
                    float(kap), ptr(thr), ptr(xs), st)
        xa_hi = torch.empty((m, data.ld), dtype=torch.float32, device=data.x.device)
        xa_lo = torch.empty_like(xa_hi)
        native.call("skm_gather_rows_i32", ptr(data.hi), data.ld, ptr(glob), m, data.ld, ptr(xa_hi), data.ld, st)
        native.call("skm_gather_rows_i32", ptr(data.lo), data.ld, ptr(glob), m, data.ld, ptr(xa_lo), data.ld, st)
        cr = lay.row_crange[glob.long()].contiguous()
        _gemm(xa_hi, xa_lo, cents.hi, cents.lo, m, cents.k, d, native.GEMM_GATE, xsq=xs, ysq=cents.ysq, thr=thr,
              cand=ws.cand, cand_cnt=ws.cand_cnt, cand_cap=ws.cap, row_crange=cr, tile_nrange=tile_ranges(cr))
        native.call("skm_cand_exact_argmin", ptr(glob), m, ptr(ws.cand), ptr(ws.cand_cnt), ws.cap, ptr(data.x),
                    data.ld, ptr(cents.c), cents.ld, d, ptr(xsq_all), ptr(cents.ysq), ws.chain_flavour,
                    ws.chain_q, ptr(ws.assign), ptr(ws.tau), st)
        if bool((ws.cand_cnt[:m] > ws.cap).any()):  # cap >= every group's k: cannot happen
            raise RuntimeError("grouped argmin: candidate slab overflow")


def _grouped_pruned_pass(data: DeviceData, cents: Centroids, ws: Workspace, plan: PrunePlan, lay: GroupLayout,
                         rmap: torch.Tensor, gcount: torch.Tensor) -> None:
    """engine.pruned_assign_pass (ordered branch) over the rows ``rmap`` of one d' class:
    tau was seeded for every row; gate threshold, grouped GATE GEMM, scan into group counters."""
    n = int(rmap.numel())
    if n == 0:
        return
    d, dp = data.d, plan.d_prime
    st = stream_handle()
    xsq = data.norms(dp)
    kap = tc_kappa(dp, GATE_KPAIR)
    native.call("skm_gate_threshold", ptr(ws.tau), data.n, float(plan.gate[0]), int(plan.sentinel), ptr(ws.thr),
                ptr(xsq), ptr(cents.ysq_max), float(kap), st)
    cx = cert_extension(data, cents, plan, ws.tau, ws.thr1, data.n, ws.nowin)
    ext = cx.get("ext_k", 0)
    xsq_ext = cx.get("xsq_ext")
    defer = DEFER_CERT and cx.get("nowin", False) and not ws.flat
    if defer:
        tau_seed, skip, imp, imp_cnt = ws.defer_buffers()
        tau_seed.copy_(ws.tau)
    fld = padded_ld(dp + ext)
    ga_hi, ga_lo = ws.front_buffers(fld)
    k = cents.k
    for b0 in range(0, n, ws.batch):
        bn = min(ws.batch, n - b0)
        rm = rmap[b0:b0 + bn]
        native.call("skm_gather_front", ptr(data.hi), ptr(data.lo), data.ld, ptr(rm), bn, dp + ext, ptr(ga_hi),
                    ptr(ga_lo), ga_hi.stride(0), ptr(xsq), ptr(ws.thr), ptr(ws.bx), ptr(ws.bthr),
                    ptr(xsq_ext) if ext else None, ptr(ws.thr1) if ext else None,
                    ptr(ws.bx_ext) if ext else None, ptr(ws.bthr1) if ext else None, st,
                    nbytes=16.0 * bn * (dp + ext) + 24.0 * bn)
        cr = lay.row_crange[rm.long()].contiguous()
        cert = dict(cx, xsq_ext=ws.bx_ext[:bn], thr1=ws.bthr1[:bn]) if ext else {}
        _gemm(ga_hi[:bn], ga_lo[:bn], cents.hi, cents.lo, bn, k, dp, native.GEMM_GATE, xsq=ws.bx[:bn],
              ysq=cents.ysq, thr=ws.bthr[:bn], cand=ws.cand, cand_cnt=ws.cand_cnt, cand_cap=ws.cap,
              row_crange=cr, tile_nrange=tile_ranges(cr), **cert)
        sp = native.ScanParams()
        sp.cand, sp.cand_cnt, sp.cap = ws.cand.data_ptr(), ws.cand_cnt.data_ptr(), ws.cap
        sp.k, sp.n_rows, sp.row0 = k, bn, 0
        sp.row_map = rm.data_ptr()
        sp.work = ws.work.data_ptr()
        sp.x, sp.ldx = data.x.data_ptr(), data.ld
        sp.tails, sp.nb, sp.d_prime = cents.tails.data_ptr(), plan.nb, dp
        sp.theta, sp.block_dims = plan.theta.data_ptr(), plan.bdims.data_ptr()
        sp.tau, sp.assign, sp.counters = ws.tau.data_ptr(), ws.assign.data_ptr(), ws.counters.data_ptr()
        sp.kap = kap
        sp.xsq, sp.ysq, sp.ysq_max = xsq.data_ptr(), cents.ysq.data_ptr(), cents.ysq_max.data_ptr()
        sp.cent, sp.ldc = cents.c.data_ptr(), cents.ld
        sp.chain_flavour, sp.chain_q = ws.chain_flavour, ws.chain_q
        sp.row_group, sp.group_counters = lay.row_group.data_ptr(), gcount.data_ptr()
        if SCAN_FLAT and ws.flat and not plan.sentinel:
            sp.flat, sp.fb_rows, sp.fb_count = 1, ws.fb_rows.data_ptr(), ws.fb_count.data_ptr()
        if defer:
            native.call("skm_defer_cert_flags", ptr(ws.cand), ptr(ws.cand_cnt), ws.cap, bn, ptr(skip), st)
            sp.skip_cert, sp.imp, sp.imp_cnt = skip.data_ptr(), imp.data_ptr(), imp_cnt.data_ptr()
        native.call("skm_pruned_scan", ctypes_ref(sp), st, tag="pruned_scan", nbytes=4.0 * bn * (d - dp) + 16.0 * bn)
        if defer:
            native.call("skm_deferred_cert_count", ctypes_ref(sp), ptr(tau_seed), st)


def ctypes_ref(obj):
    import ctypes
    return ctypes.byref(obj)


def fit_groups_device(data: DeviceData, sizes: np.ndarray, ks: np.ndarray, seeds: list[int], cfg: KMeansConfig,
                      max_iters: int, comm=None, sizes_global: np.ndarray | None = None,
                      lo_in_group: np.ndarray | None = None) -> tuple[torch.Tensor, torch.Tensor, WorkCounters]:
    """Fit every group of ``data`` (rows laid out group by group, ``sizes[g]`` rows each) into
    ``ks[g]`` centroids with seed ``seeds[g]``, ``max_iters`` iterations each, exactly as
    independent ``fit_rotated_device`` calls would.  Returns (centroids (sum ks, ld) with group g
    at rows [c0_g, c0_g + k_g), assignments as global centroid rows, merged work counters).

    Row-sharded (``comm`` with world > 1): this rank holds members
    [lo_in_group[g], lo_in_group[g] + sizes[g]) of group g's ``sizes_global[g]`` (ranks hold
    ascending row ranges, so the concatenation over ranks is the group's member list).  The Forgy
    rows are assembled by one allreduce, and every iteration does ONE allreduce of the packed
    [centroid sums (f64, chained in rank order with cfg.exact_reduce) | counts | per-group
    survivors, dims touched, changed] -- the groups' d', convergence and splits are decided on
    identical global numbers on every rank, so the result is the one-GPU batched result."""
    dev = data.x.device
    d = data.d
    lay = GroupLayout(sizes, ks, dev)
    G, n = lay.G, lay.n
    sharded = comm is not None and comm.world > 1
    nglob = np.asarray(sizes_global if sharded else lay.sizes, dtype=np.int64)
    lo_g = np.asarray(lo_in_group if sharded else np.zeros(G), dtype=np.int64)
    assert n == data.n and G > 0 and int(nglob.min()) >= 2
    st = stream_handle()
    # Forgy rows of every group from its own stream ([seed_g, 2]), gathered in one launch
    # (sharded: each rank gathers the members it holds, one allreduce assembles the rest)
    c = torch.zeros((lay.k_total, data.ld), dtype=torch.float32, device=dev)
    src_rows, dst_rows = [], []
    for g in range(G):
        idx_g = init_indices(int(nglob[g]), int(lay.ks[g]), [seeds[g], 2])
        mine = np.flatnonzero((idx_g >= lo_g[g]) & (idx_g < lo_g[g] + lay.sizes[g]))
        src_rows.append(idx_g[mine] - lo_g[g] + lay.starts[g])
        dst_rows.append(mine + lay.c0[g])
    src = np.concatenate(src_rows).astype(np.int64)
    dst = np.concatenate(dst_rows).astype(np.int64)
    if src.size:
        tmp = torch.empty((src.size, data.ld), dtype=torch.float32, device=dev)
        native.call("skm_gather_rows", ptr(data.x), data.ld, ptr(torch.from_numpy(src).to(dev)), int(src.size),
                    data.ld, ptr(tmp), data.ld, st)
        c.index_copy_(0, torch.from_numpy(dst).to(dev), tmp)
    if sharded:
        comm.allreduce_(c)  # every Forgy row is held by exactly one rank
    cents = Centroids(c, d)
    kmax = int(lay.ks.max())
    wcfg = KMeansConfig(k=lay.k_total, max_iters=max_iters, seed=cfg.seed, gemm_backend=cfg.gemm_backend,
                        cand_cap=max(32, (kmax + 31) // 32 * 32), x_batch_device=cfg.x_batch_device)
    ws = Workspace(dev, n, lay.k_total, d, wcfg)
    assert ws.cap >= kmax
    gcount = torch.zeros((G, 3), dtype=torch.int64, device=dev)
    rngs = [np.random.default_rng([seeds[g], 3]) for g in range(G)]
    pruned_mode = pruning_supported(d)
    dprime = np.full(G, initial_d_prime(d, cfg.d_prime_init_fraction) if pruned_mode else 0, dtype=np.int64)
    active = np.ones(G, dtype=bool)
    work = WorkCounters()
    final_c = torch.zeros_like(c)  # each group's centroids as its own loop ends
    pin_g = torch.empty((G, 3), dtype=torch.int64, pin_memory=True)
    pin_counts = torch.empty(lay.k_total, dtype=torch.int32, pin_memory=True)
    nk = nglob * lay.ks
    last_changed = None
    last_surv = None
    if sharded:
        K = lay.k_total
        red = torch.zeros(K * d + K + 3 * G, dtype=torch.float64, device=dev)
        pin_red = torch.empty(K + 3 * G, dtype=torch.float64, pin_memory=True)
        counts64 = torch.empty(K, dtype=torch.int64, device=dev)

    for it in range(1, max_iters + 1):
        act = np.flatnonzero(active)
        if act.size == 0:
            break
        pruned_iter = pruned_mode and it > 1
        gcount.zero_()
        if not pruned_iter:
            if it > 1:
                prev = ws.assign[:n].clone()
            cents.refresh(d, None)
            # contiguous runs of active groups
            runs = np.split(act, np.flatnonzero(np.diff(act) != 1) + 1)
            for run in runs:
                r0 = int(lay.starts[run[0]])
                r1 = int(lay.starts[run[-1]] + lay.sizes[run[-1]])
                _grouped_full_assign(data, cents, ws, lay, r0, r1)
            if it > 1:
                ch = (ws.assign[:n] != prev).to(torch.int64)
                gcount[:, 2] = torch.zeros(G, dtype=torch.int64, device=dev).index_add_(0, lay.row_group.long(), ch)
            work.full_pair_dims += int((nk[act] * d).sum())
        else:
            native.call("skm_seed_thresholds", ptr(data.x), data.ld, ptr(cents.c), cents.ld, ptr(ws.assign), n, d,
                        ptr(ws.tau), st, nbytes=4.0 * n * d + 8.0 * n)
            ws.flat = last_changed is not None and last_changed <= FLAT_MAX_CHANGED * int(nglob[act].sum())
            ws.nowin = (not cfg.exact_work_stats and not cfg.pruning_sentinel and not ws.flat
                        and (last_surv is None or last_surv > NOWIN_SURV_FRAC * int(nk[act].sum())))
            for dp in np.unique(dprime[act]):
                cls = act[dprime[act] == dp]
                plan = PrunePlan(d, int(dp), cfg.epsilon0, cfg.pruning_sentinel, dev)
                cents.refresh(int(dp), int(dp))
                if cls.size == G:
                    rmap = ws.order[:n]
                else:  # the class's groups' segments of the cluster order (= their row ranges)
                    segs = [ws.order[int(lay.starts[g]):int(lay.starts[g] + lay.sizes[g])] for g in cls]
                    rmap = torch.cat(segs) if len(segs) > 1 else segs[0]
                if plan.sentinel:
                    for g in cls:
                        ws.tau[int(lay.starts[g]):int(lay.starts[g] + lay.sizes[g])].fill_(float("inf"))
                _grouped_pruned_pass(data, cents, ws, plan, lay, rmap.contiguous(), gcount)
                work.front_pair_dims += int((nk[cls] * dp).sum())
                if not cfg.pruning_sentinel:
                    work.seed_dims += int((nglob[cls] * d).sum())
        # stable cluster sort of every row (groups own disjoint column ranges, so the order is
        # group by group, members ascending) + one readback of counts and group counters
        if n:
            native.call("skm_cluster_sort", ptr(ws.assign), n, lay.k_total, ptr(ws.order), ptr(ws.counts),
                        ptr(ws.offsets), ptr(ws.sort_ws), ws.sort_ws.numel(), st, nbytes=32.0 * n)
        else:
            ws.counts.zero_()
            ws.offsets.zero_()
        if sharded:
            # the iteration's one collective: [sums | counts | group counters], sums chained in
            # rank order (exact) or per-rank partials added by the allreduce
            K = lay.k_total
            sums = red[:K * d]
            if cfg.exact_reduce:
                chained_cluster_sums(comm, data, ws, sums, K, d)
            else:
                native.call("skm_cluster_sums", ptr(data.x), data.ld, ptr(ws.order), ptr(ws.offsets),
                            ptr(ws.counts), K, d, ptr(sums), 0, None, 0, 1, st, nbytes=4.0 * n * d)
            red[K * d:K * d + K].copy_(ws.counts.to(torch.float64))
            red[K * d + K:].copy_(gcount.view(-1).to(torch.float64))
            comm.allreduce_(red)
            pin_red.copy_(red[K * d:], non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()
            h = pin_red.numpy()
            counts = np.rint(h[:K]).astype(np.int64)
            gc = np.rint(h[K:]).astype(np.int64).reshape(G, 3)
        else:
            pin_g.copy_(gcount, non_blocking=True)
            pin_counts.copy_(ws.counts, non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()
            gc = pin_g.numpy().copy()
            counts = pin_counts.numpy().astype(np.int64)
        last_changed = int(gc[act, 2].sum()) if it > 1 else None
        if pruned_iter:
            last_surv = int(gc[act, 0].sum())  # survivors of the active groups (exact_work_stats policy)
        stop_now = np.zeros(G, dtype=bool)
        if it > 1:
            stop_now[act] = gc[act, 2] == 0  # converged: no update, no split (core.py:358-363)
        if pruned_iter:
            work.tail_dims += int(gc[act, 1].sum())
        # a converged group ends before the update (its centroids may differ from its members'
        # means after earlier splits): keep them as they are now
        _freeze(final_c, cents.c, lay, np.flatnonzero(stop_now))
        # update of every centroid (the groups that stopped are not read again)
        if sharded:
            counts64.copy_(torch.from_numpy(counts))
            native.call("skm_finalize_centroids", ptr(red), ptr(counts64), lay.k_total, d, ptr(cents.c), cents.ld, st)
        else:
            native.call("skm_cluster_sums", ptr(data.x), data.ld, ptr(ws.order), ptr(ws.offsets), ptr(ws.counts),
                        lay.k_total, d, None, 0, ptr(cents.c), cents.ld, 0, st,
                        nbytes=4.0 * n * d + 4.0 * lay.k_total * d)
        empties, donors = [], []
        # groups with an empty cluster (only they draw from their split RNG, core.py:103-128)
        has_empty = np.minimum.reduceat(counts, lay.c0) == 0 if cfg.split_empty else np.zeros(G, dtype=bool)
        for g in act:
            if stop_now[g]:
                continue
            if has_empty[g]:
                c0, k = int(lay.c0[g]), int(lay.ks[g])
                e, dn = plan_splits(counts[c0:c0 + k].copy(), rngs[g])
                empties += [c0 + v for v in e]
                donors += [c0 + v for v in dn]
            if pruned_iter:
                rate = prune_rate_from_totals(int(gc[g, 0]), int(nglob[g]), int(lay.ks[g]))
                dprime[g] = adjust_d_prime(int(dprime[g]), rate, cfg, d)
        if empties:
            e_t = torch.tensor(empties, dtype=torch.int32, device=dev)
            d_t = torch.tensor(donors, dtype=torch.int32, device=dev)
            native.call("skm_apply_splits", ptr(cents.c), cents.ld, d, ptr(e_t), ptr(d_t), len(empties),
                        float(SPLIT_EPS), st)
        active &= ~stop_now
        if it == max_iters:
            _freeze(final_c, cents.c, lay, np.flatnonzero(active))
    return final_c, ws.assign[:n], work


def _freeze(dst: torch.Tensor, src: torch.Tensor, lay: GroupLayout, groups: np.ndarray) -> None:
    if groups.size == 0:
        return
    rows = np.concatenate([np.arange(lay.c0[g], lay.c0[g] + lay.ks[g]) for g in groups])
    idx = torch.from_numpy(rows.astype(np.int64)).to(dst.device)
    dst.index_copy_(0, idx, src.index_select(0, idx))

"""ORACLE -- test infrastructure only (imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py; never by the product package).

A plain NumPy restatement of the reference SuperKMeans loop, written to reproduce its
arithmetic exactly given the same GEMM (NumPy/OpenBLAS sgemm):

  fit                  pkg/src/superkmeans/core.py:417-460
  _fit_rotated         core.py:284-414
  _full_assign_pass    core.py:169-192
  _pruned_assign_pass  core.py:195-267 (scan/seed kernels: oracle/kernels_np.py)
  update/split/adjust  core.py:79-154
  final_assign         core.py:463-541
  ETR                  evaluation.py:53-75, 116-170
  IVF probe evaluation evaluation.py:78-105, 173-203
  hierarchical_fit     hierarchical.py:91-171

It is pinned against the real reference (tests/test_oracle_*.py compare it with the imported
reference package here, and with committed golden fixtures everywhere else).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import kernels_c as _KC
from . import kernels_np as _KN

# the C/OpenMP restatement when built (same bits, reference-compiled speed), else NumPy
K = _KC if _KC.available() else _KN


def use_numpy_kernels(flag: bool = True) -> None:
    global K
    K = _KN if flag or not _KC.available() else _KC

PDX_BLOCK, MAX_BANK, D_MIN, D_ALIGN = 64, 1024, 16, 8
SPLIT_EPS = np.float32(1.0 / 1024.0)


@dataclass
class Params:
    """The subset of KMeansConfig the loop reads (same names/defaults)."""
    k: int
    max_iters: int = 25
    x_batch: int = 4096
    y_batch: int = 1024
    d_prime_init_fraction: float = 0.125
    epsilon0: float = 2.1
    prune_target_low: float = 0.95
    prune_target_high: float = 0.97
    d_prime_adjust_factor: float = 0.20
    sampling_fraction: float = 1.0
    seed: int = 0
    split_empty: bool = True
    pruning_sentinel: bool = False
    etr: dict | None = None  # {"tolerance", "patience_iters", "n_queries", "top_k", "nprobe_fraction"}


@dataclass
class Stat:
    iter_index: int
    wcss: float
    n_empty_splits: int = 0
    prune_rate_after_gemm: float | None = None
    recall: float | None = None
    d_prime: int | None = None
    survivors: int = 0
    tail_dims_touched: int = 0
    n_changed: int | None = None


@dataclass
class Out:
    centroids: np.ndarray
    centroids_rotated: np.ndarray
    assignments: np.ndarray
    stats: list
    terminated_by: str
    d_prime_final: int | None
    init_indices: np.ndarray
    rotation: np.ndarray
    sample_indices: np.ndarray | None
    recall_history: list = field(default_factory=list)
    snapshots: list = field(default_factory=list)
    tail_dims: int = 0


# ------------------------------------------------------------------ host math
def rotation(d, seed):
    # BLAS pinned to 4 threads (= the single-threaded bits): OpenBLAS's QR bits depend on the
    # thread count (see paper_2603_20009_b200/hostmath.py blas_threads)
    from threadpoolctl import threadpool_limits
    with threadpool_limits(4, user_api="blas"):
        q, r = np.linalg.qr(np.random.default_rng(seed).standard_normal((d, d)))
    s = np.sign(np.diag(r))
    s[s == 0] = 1.0
    return (q * s[None, :]).astype(np.float32)


def sq_norms(m, dims=None):
    v = m if dims is None else m[:, :dims]
    return np.einsum("ij,ij->i", v, v, dtype=np.float64).astype(np.float32)


def expand(inner, xs, ys):
    v = inner * np.float32(-2.0)
    v += xs[:, None]
    v += ys[None, :]
    np.maximum(v, np.float32(0.0), out=v)
    return v


def layout(d, dp):
    nf, rest = divmod(d - dp, PDX_BLOCK)
    w = np.array([PDX_BLOCK] * nf + ([rest] if rest else []), dtype=np.int32)
    return w, dp + np.cumsum(w, dtype=np.int64)


def factors(d, dp, bounds, eps0):
    m = np.concatenate(([dp], bounds)).astype(np.int64)
    g = 1.0 + eps0 / np.sqrt(m.astype(np.float64))
    f = (m / d) * g * g
    f[m == d] = 1.0
    return f.astype(np.float32)


def pdx_bank(c, dp):
    kb, d = c.shape
    w, ends = layout(d, dp)
    starts = np.concatenate(([dp], ends[:-1]))
    offs = np.concatenate(([0], np.cumsum(w[:-1], dtype=np.int64))) * kb
    tail = np.concatenate([np.ascontiguousarray(c[:, s:e].T).ravel() for s, e in zip(starts, ends)])
    return np.ascontiguousarray(c[:, :dp]), tail.astype(np.float32), w, offs.astype(np.int64)


def adjust(dp, rate, p: Params, d):
    lo, hi = D_MIN, d - PDX_BLOCK
    if rate > p.prune_target_high:
        new, up = int(np.floor(dp * (1.0 - p.d_prime_adjust_factor))), False
    elif rate < p.prune_target_low:
        new, up = int(np.ceil(dp * (1.0 + p.d_prime_adjust_factor))), True
    else:
        return dp
    new = min(hi, max(lo, new))
    new = -(-new // D_ALIGN) * D_ALIGN if up else (new // D_ALIGN) * D_ALIGN
    return min(hi, max(lo, new))


def update(x, assign, k, prev):
    sums = np.zeros((k, x.shape[1]), np.float64)
    counts = np.zeros(k, np.int64)
    K.accumulate_centroid_sums(x, assign, sums, counts)
    c = prev.copy()
    ne = counts > 0
    c[ne] = (sums[ne] / counts[ne, None]).astype(np.float32)
    return c, counts


def split(c, counts, rng):
    empties = np.flatnonzero(counts == 0)
    k, d = c.shape
    signs = np.where(np.arange(d) % 2 == 0, 1.0, -1.0).astype(np.float32)
    for e in empties:
        donor = int(rng.choice(k, p=counts / counts.sum()))
        row = c[donor].copy()
        delta = row * SPLIT_EPS * signs
        c[e] = row + delta
        c[donor] = row - delta
        moved = counts[donor] // 2
        counts[e] = counts[donor] - moved
        counts[donor] = moved
    return len(empties)


# ------------------------------------------------------------------ passes
def full_pass(xr, c, p: Params, tau, assign):
    n, d = xr.shape
    k = c.shape[0]
    xs, ys = sq_norms(xr), sq_norms(c)
    tau[:] = np.inf
    for s0 in range(0, n, p.x_batch):
        e0 = min(n, s0 + p.x_batch)
        for s1 in range(0, k, p.y_batch):
            e1 = min(k, s1 + p.y_batch)
            v = expand(xr[s0:e0] @ c[s1:e1].T, xs[s0:e0], ys[s1:e1])
            loc = np.argmin(v, axis=1)
            best = v[np.arange(e0 - s0), loc]
            better = best < tau[s0:e0]
            assign[s0:e0][better] = (s1 + loc[better]).astype(np.int32)
            tau[s0:e0][better] = best[better]


def pruned_pass(xr, c, dp, p: Params, tau, assign):
    n, d = xr.shape
    k = c.shape[0]
    w, bounds = layout(d, dp)
    f = factors(d, dp, bounds, p.epsilon0)
    banks = [(s1, pdx_bank(c[s1:s1 + p.y_batch], dp)) for s1 in range(0, k, p.y_batch)]
    xs, ys = sq_norms(xr, dp), sq_norms(c, dp)
    surv = touched = changed = 0
    for s0 in range(0, n, p.x_batch):
        e0 = min(n, s0 + p.x_batch)
        xb, ab, tb = xr[s0:e0], assign[s0:e0], tau[s0:e0]
        prev = ab.copy()
        if p.pruning_sentinel:
            tb[:] = np.inf
        else:
            K.seed_thresholds(xb, c, ab, tb)
        front = np.ascontiguousarray(xb[:, :dp])
        for s1, (bf, tail, bw, boff) in banks:
            v = expand(front @ bf.T, xs[s0:e0], ys[s1:s1 + bf.shape[0]])
            sv, td = K.scan_bank(np.ascontiguousarray(v), xb, tail, boff, bw, f, dp, s1, tb, ab, p.pruning_sentinel)
            surv += sv
            touched += td
        changed += int(np.count_nonzero(prev != ab))
    return surv, touched, changed


# ------------------------------------------------------------------ ETR
def brute_force_topk(x, q, k_gt, qb=128):
    xs = sq_norms(x)
    idx = np.empty((q.shape[0], k_gt), np.int64)
    dst = np.empty((q.shape[0], k_gt), np.float32)
    for s in range(0, q.shape[0], qb):
        e = min(q.shape[0], s + qb)
        d2 = expand(q[s:e] @ x.T, sq_norms(q[s:e]), xs)
        o = np.argsort(d2, axis=1, kind="stable")[:, :k_gt]
        idx[s:e] = o
        dst[s:e] = np.take_along_axis(d2, o, axis=1)
    return idx, dst


def etr_hits(c, xr, assign, q, gt_idx, nprobe, top_k):
    """Per-query hit counts of the reference's probe (evaluation.py:142-170)."""
    k = c.shape[0]
    nprobe = min(max(1, nprobe), k)
    order = np.argsort(assign, kind="stable")
    bounds = np.cumsum(np.bincount(assign, minlength=k))[:-1]
    lists = np.split(order, bounds)
    cs, xs = sq_norms(c), sq_norms(xr)
    hits = np.zeros(q.shape[0], np.int64)
    for s in range(0, q.shape[0], 256):
        e = min(q.shape[0], s + 256)
        probe = np.argsort(expand(q[s:e] @ c.T, sq_norms(q[s:e]), cs), axis=1, kind="stable")[:, :nprobe]
        for qi in range(e - s):
            cand = np.concatenate([lists[j] for j in probe[qi]])
            d2 = expand(q[s + qi:s + qi + 1] @ xr[cand].T, sq_norms(q[s + qi:s + qi + 1]), xs[cand])[0]
            take = min(top_k, cand.size)
            top = cand[np.lexsort((cand, d2))[:take]]
            hits[s + qi] = int(np.isin(top, gt_idx[s + qi, :top_k], assume_unique=True).sum())
    return hits


def cluster_lists(assign, k):
    """build_cluster_lists (evaluation.py:78-83)."""
    order = np.argsort(assign, kind="stable")
    return np.split(order, np.cumsum(np.bincount(assign, minlength=k))[:-1])


def ivf_probe_search(c, lists, x, q, nprobe, top_k):
    """evaluation.py:86-105."""
    nprobe = min(nprobe, c.shape[0])
    q2 = q.reshape(1, -1).astype(np.float32)
    probe = np.argsort(expand(q2 @ c.T, sq_norms(q2), sq_norms(c))[0], kind="stable")[:nprobe]
    cand = np.concatenate([lists[j] for j in probe])
    if cand.size == 0:
        return np.empty(0, np.int64), np.empty(0, np.float32), 0
    d2 = expand(q2 @ x[cand].T, sq_norms(q2), sq_norms(x[cand]))[0]
    o = np.lexsort((cand, d2))[:top_k]
    return cand[o].astype(np.int64), d2[o], int(cand.size)


def probe_eval(c, lists, x, q, gt_idx, k_gt, nprobe, top_ks=(10, 100)):
    """evaluation.py:173-203: recall@t per t <= k_gt and mean vectors explored."""
    nprobe = min(max(1, nprobe), c.shape[0])
    top_ks = sorted({t for t in top_ks if t <= k_gt})
    cs, xs = sq_norms(c), sq_norms(x)
    nq = q.shape[0]
    rec = {t: 0.0 for t in top_ks}
    explored = 0
    for s in range(0, nq, 256):
        e = min(nq, s + 256)
        probe = np.argsort(expand(q[s:e] @ c.T, sq_norms(q[s:e]), cs), axis=1, kind="stable")[:, :nprobe]
        for qi in range(e - s):
            cand = np.concatenate([lists[j] for j in probe[qi]])
            explored += cand.size
            d2 = expand(q[s + qi:s + qi + 1] @ x[cand].T, sq_norms(q[s + qi:s + qi + 1]), xs[cand])[0]
            found = cand[np.lexsort((cand, d2))]
            for t in top_ks:
                take = min(t, found.size)
                rec[t] += int(np.isin(found[:take], gt_idx[s + qi, :t], assume_unique=True).sum()) / t
    out = {f"recall_at_{t}": rec[t] / nq for t in top_ks}
    out["vectors_explored_mean"] = explored / nq
    return out


def recall_from_hits(hits, top_k):
    total = 0.0
    for h in hits:
        total += int(h) / top_k
    return total / len(hits)


def etr_should_stop(v, tol, patience):
    if len(v) < patience + 1:
        return False
    w = v[-(patience + 1):]
    if max(w[1:]) - w[0] > tol:
        return False
    return all(b - a <= tol for a, b in zip(w[1:], w[2:]))


# ------------------------------------------------------------------ loop
def fit_rotated(xr, p: Params, inspect=True):
    n, d = xr.shape
    k = p.k
    init = np.random.default_rng([p.seed, 2]).choice(n, size=k, replace=False)
    c = xr[init].copy()
    assign = np.zeros(n, np.int32)
    tau = np.full(n, np.inf, np.float32)
    rng_split = np.random.default_rng([p.seed, 3])
    pruned_mode = d - PDX_BLOCK >= D_MIN
    dp = max(D_MIN, min(d - PDX_BLOCK, int(d * p.d_prime_init_fraction))) if pruned_mode else None
    etr = None
    if p.etr is not None:
        nq = min(p.etr.get("n_queries", 1000), n)
        qidx = np.random.default_rng([p.seed, 4]).choice(n, size=nq, replace=False)
        q = xr[qidx].copy()
        top_k = p.etr.get("top_k", 100)
        gt_idx, _ = brute_force_topk(xr, q, top_k)
        nprobe = int(np.ceil(p.etr.get("nprobe_fraction", 0.01) * k))
        etr = (q, gt_idx, nprobe, top_k)
    stats, recalls, snaps = [], [], []
    term = "max_iters"
    tail_total = 0
    for it in range(1, p.max_iters + 1):
        pruned_iter = pruned_mode and it > 1
        surv = touched = 0
        rate = None
        changed = None
        if not pruned_iter:
            prev = assign.copy() if it > 1 else None
            full_pass(xr, c, p, tau, assign)
            if prev is not None:
                changed = int(np.count_nonzero(prev != assign))
        else:
            surv, touched, changed = pruned_pass(xr, c, dp, p, tau, assign)
            rate = 1.0 - surv / (n * k)
            tail_total += touched
        wcss = float(np.sum(tau, dtype=np.float64))
        if inspect:
            snaps.append({"assignments": assign.copy(), "best_sq_dist": tau.copy(), "centroids_rotated": c.copy(),
                          "d_prime": dp if pruned_iter else None, "prune_rate": rate})
        if changed == 0:
            stats.append(Stat(it, wcss, 0, rate, None, dp if pruned_iter else None, surv, touched, changed))
            term = "converged"
            break
        c, counts = update(xr, assign, k, c)
        ns = split(c, counts, rng_split) if p.split_empty else 0
        d_used = dp if pruned_iter else None
        if pruned_iter:
            dp = adjust(dp, rate, p, d)
        rec = None
        if etr is not None:
            q, gt_idx, nprobe, top_k = etr
            rec = recall_from_hits(etr_hits(c, xr, assign, q, gt_idx, nprobe, top_k), top_k)
            recalls.append(rec)
        stats.append(Stat(it, wcss, ns, rate, rec, d_used, surv, touched, changed))
        if etr is not None and etr_should_stop(recalls, p.etr.get("tolerance", 0.005), p.etr.get("patience_iters", 2)):
            term = "etr"
            break
    return c, assign, tau, stats, term, dp, init, recalls, snaps, tail_total


def fit(x, p: Params, inspect=True) -> Out:
    x = np.ascontiguousarray(x, dtype=np.float32)
    n, d = x.shape
    sidx = None
    xs = x
    if p.sampling_fraction != 1.0:
        m = int(np.ceil(p.sampling_fraction * n))
        sidx = np.random.default_rng([p.seed, 1]).choice(n, size=m, replace=False)
        sidx.sort()
        xs = x[sidx]
    r = rotation(d, p.seed)
    xr = np.ascontiguousarray(xs @ r, dtype=np.float32)
    c, a, tau, stats, term, dp, init, recalls, snaps, tail_total = fit_rotated(xr, p, inspect)
    return Out(centroids=np.ascontiguousarray(c @ r.T, dtype=np.float32), centroids_rotated=c, assignments=a,
               stats=stats, terminated_by=term, d_prime_final=dp, init_indices=init, rotation=r,
               sample_indices=sidx, recall_history=recalls, snapshots=snaps, tail_dims=tail_total)


def final_assign(x_full, out: Out, p: Params):
    x_full = np.ascontiguousarray(x_full, dtype=np.float32)
    n, d = x_full.shape
    c = out.centroids_rotated
    k = c.shape[0]
    assign = np.zeros(n, np.int32)
    if out.sample_indices is not None:
        assign[out.sample_indices] = out.assignments
    elif out.assignments.shape[0] == n:
        assign[:] = out.assignments
    pruned_mode = (d - PDX_BLOCK >= D_MIN) and out.d_prime_final is not None
    tau = np.empty(p.x_batch, np.float32)
    for s0 in range(0, n, p.x_batch):
        e0 = min(n, s0 + p.x_batch)
        xb = np.ascontiguousarray(x_full[s0:e0] @ out.rotation, dtype=np.float32)
        ab, tb = assign[s0:e0], tau[: e0 - s0]
        q = Params(**{**p.__dict__, "pruning_sentinel": False})
        if pruned_mode:
            pruned_pass(xb, c, out.d_prime_final, q, tb, ab)
        else:
            full_pass(xb, c, q, tb, ab)
    return assign


def sub_seed(seed, tag):
    return int(np.random.SeedSequence([seed, 5, tag]).generate_state(1)[0])


def hierarchical_fit(x, k_total, meso_k=None, meso_iters=3, fine_iters=5, seed=0, **kw):
    x = np.ascontiguousarray(x, dtype=np.float32)
    n, d = x.shape
    if meso_k is None:
        meso_k = int(np.ceil(np.sqrt(k_total)))
    r = rotation(d, seed)
    xr = np.ascontiguousarray(x @ r, dtype=np.float32)
    base = dict(kw)
    meso = fit_rotated(xr, Params(k=meso_k, max_iters=meso_iters, seed=seed, **base), inspect=False)
    massign = meso[1]
    order = np.argsort(massign, kind="stable")
    groups = np.split(order, np.cumsum(np.bincount(massign, minlength=meso_k))[:-1])
    plans, off = [], 0
    for gi, idx in enumerate(groups):
        if idx.size == 0:
            continue
        ki = 1 if idx.size == 1 else max(1, round(np.sqrt(idx.size)))
        plans.append((gi, idx, ki, off))
        off += ki
    cent = np.empty((off, d), np.float32)
    gassign = np.empty(n, np.int32)
    for gi, idx, ki, o in plans:
        if idx.size == 1:
            cent[o] = xr[idx[0]]
            gassign[idx] = o
            continue
        res = fit_rotated(np.ascontiguousarray(xr[idx]), Params(k=ki, max_iters=fine_iters, seed=sub_seed(seed, gi),
                                                                  **base), inspect=False)
        cent[o:o + ki] = res[0]
        gassign[idx] = o + res[1]
    return np.ascontiguousarray(cent @ r.T, dtype=np.float32), cent, gassign, meso, plans

"""Early Termination by Recall on the device.

Setup (once per fit, core.py:305-316):
  q_idx = default_rng([seed, 4]).choice(n, nq)   (host RNG -> device gather)
  GT    = exact top_k of every query over all rows: distance GEMM (tcgen05 3xTF32, DIST
          epilogue) + exact per-row radix top-k with lowest-index ties
          (brute_force_topk, evaluation.py:53-75).  Row-sharded: per-rank top-k + merge.
Per iteration (after update + split, core.py:380-387):
  probe = top-nprobe post-update centroids per query (GEMM + top-k, stable ties)
  hits_q = #{g in GT_q : assign[g] in probe_q}        (integer tally, allreduced)
  recall = (sum_q hits_q / top_k) / nq               (host f64, query order)
The tally equals the reference's per-query recall (evaluation.py:142-170): a GT member that
is a candidate always ranks within top_k among the candidates.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import native
from .device import on_device, padded_ld, ptr, require_cuda, stream_handle
from .hostmath import etr_should_stop


@dataclass
class GroundTruth:
    indices: np.ndarray   # (n_queries, k_gt) int64
    distances: np.ndarray  # (n_queries, k_gt) float32
    k_gt: int
    metric: str = "l2"


@dataclass
class RecallHistory:
    values: list = field(default_factory=list)
    tolerance: float = 0.005
    patience: int = 2

    def append(self, value: float) -> None:
        self.values.append(float(value))

    def should_stop(self) -> bool:
        return etr_should_stop(self.values, self.tolerance, self.patience)


def _split(x: torch.Tensor, cols: int):
    hi = torch.empty_like(x)
    lo = torch.empty_like(x)
    if x.shape[0]:
        native.call("skm_split_hilo", ptr(x), x.shape[1], x.shape[0], cols, ptr(hi), ptr(lo), x.shape[1],
                    stream_handle())
    return hi, lo


def _norms(x: torch.Tensor, dims: int) -> torch.Tensor:
    out = torch.empty(max(x.shape[0], 1), dtype=torch.float32, device=x.device)
    if x.shape[0]:
        native.call("skm_row_sq_norms", ptr(x), x.shape[1], x.shape[0], dims, ptr(out), stream_handle())
    return out


TOPK_MAX = 2048  # csrc/topk.cuh


def merge_topk_shards(all_i: torch.Tensor, all_v: torch.Tensor, shards: int, kk: int, nq: int, k_out: int):
    """Stable (distance, index) merge of per-shard sorted top-k lists [shard][query][kk]; the
    device merge takes up to 8 lists at a time, so more shards merge in rounds."""
    dev = all_i.device
    while shards > 1:
        groups = []
        for g0 in range(0, shards, 8):
            g = min(8, shards - g0)
            gi = torch.empty((nq, kk), dtype=torch.int32, device=dev)  # the merge keeps the lists' width
            gv = torch.empty((nq, kk), dtype=torch.float32, device=dev)
            native.call("skm_topk_merge", ptr(all_i[g0:g0 + g].contiguous()), ptr(all_v[g0:g0 + g].contiguous()), g,
                        kk, nq, ptr(gi), ptr(gv), stream_handle())
            groups.append((gi, gv))
        if len(groups) == 1:
            all_i, all_v = groups[0][0][None], groups[0][1][None]
            break
        all_i = torch.stack([g_[0] for g_ in groups]).contiguous()
        all_v = torch.stack([g_[1] for g_ in groups]).contiguous()
        shards = len(groups)
    return all_i[0, :, :k_out].contiguous(), all_v[0, :, :k_out].contiguous()


TOPK_FUSED_MAX = 32  # csrc/sgemm_chain.cuh TOPK_TILE_MAX
FUSED_GT = True      # tests flip it to compare with the materialised distance blocks


def device_topk_distances(q: torch.Tensor, q_hi, q_lo, q_sq, x: torch.Tensor, x_hi, x_lo, x_sq, d: int, k: int,
                          col_offset: int = 0, max_bytes: int = 1 << 30) -> tuple[torch.Tensor, torch.Tensor]:
    """Exact top-k rows of x for each query (squared L2 via the expansion identity, stable
    ties).  Returns (idx int32 (nq, k) with col_offset added, dist float32 (nq, k)).

    The distance block is the reference's own bits (evaluation.py:42-50 multiplies with numpy
    ``@``: OpenBLAS sgemm) -- the exact fma chain with 448-wide K blocks of csrc/sgemm_chain.cuh --
    so the ranks, ties and the stable order equal brute_force_topk / the probe ranking exactly.
    (q_hi / q_lo / x_hi / x_lo: unused, kept for callers of the tensor-core version.)"""
    from .engine import GEMM_Q, chain_gemm
    nq, n = q.shape[0], x.shape[0]
    dev = q.device
    kk = min(k, n)
    out_i = torch.empty((nq, kk), dtype=torch.int32, device=dev)
    out_v = torch.empty((nq, kk), dtype=torch.float32, device=dev)
    if nq == 0 or n == 0:
        return out_i, out_v
    if kk <= TOPK_FUSED_MAX and FUSED_GT:
        # fused: each 128-row tile keeps its kk best per query in the chain kernel's epilogue,
        # a radix top-k over the n_tiles * kk survivors finishes (no distance matrix in HBM)
        n_tiles = (n + 127) // 128
        qb = max(1, min(nq, max_bytes // (8 * n_tiles * kk)))
        for s in range(0, nq, qb):
            e = min(nq, s + qb)
            qt = torch.zeros((d, padded_ld(e - s)), dtype=torch.float32, device=dev)
            qt[:, :e - s] = q[s:e, :d].t()
            cv = torch.empty((e - s, n_tiles * kk), dtype=torch.float32, device=dev)
            ci = torch.empty((e - s, n_tiles * kk), dtype=torch.int32, device=dev)
            native.call("skm_chain_topk_tiles", ptr(x), x.stride(0), ptr(qt), qt.stride(0), n, e - s, d, 0, GEMM_Q,
                        ptr(x_sq), ptr(q_sq[s:e]), kk, ptr(cv), ptr(ci), col_offset, stream_handle(),
                        flops=2.0 * (e - s) * n * d, tag="chain_topk")
            pos = torch.empty((e - s, kk), dtype=torch.int32, device=dev)
            native.call("skm_topk_rows", ptr(cv), cv.stride(0), e - s, n_tiles * kk, kk, ptr(pos), ptr(out_v[s:e]),
                        kk, 0, stream_handle(), nbytes=5.0 * 4 * (e - s) * n_tiles * kk)
            out_i[s:e] = torch.gather(ci, 1, pos.long())
        return out_i, out_v
    qb = max(1, min(nq, max_bytes // (4 * padded_ld(n))))
    for s in range(0, nq, qb):
        e = min(nq, s + qb)
        D = torch.empty((e - s, padded_ld(n)), dtype=torch.float32, device=dev)
        chain_gemm(q[s:e], x, e - s, n, d, D, 0, GEMM_Q, xsq=q_sq[s:e], ysq=x_sq)
        if kk <= TOPK_MAX:
            native.call("skm_topk_rows", ptr(D), D.stride(0), e - s, n, kk, ptr(out_i[s:e]), ptr(out_v[s:e]), kk,
                        col_offset, stream_handle(), nbytes=5.0 * 4 * (e - s) * n)
        else:  # beyond the radix-select kernel's k: a stable device sort of the rows (same order)
            v, i = torch.sort(D[:, :n], dim=1, stable=True)
            out_v[s:e] = v[:, :kk]
            out_i[s:e] = (i[:, :kk] + col_offset).to(torch.int32)
    return out_i, out_v


class EtrState:
    """Ground truth + probe state for one fit (replicated across ranks)."""

    def __init__(self, cfg):
        self.etr = cfg.etr
        self.k = cfg.k
        self.seed = cfg.seed
        self.top_k = cfg.etr.top_k
        self.nprobe = int(np.ceil(cfg.etr.nprobe_fraction * cfg.k))

    def setup(self, data, comm, n_global: int | None = None, row_lo: int = 0):
        dev = data.x.device
        n = data.n if n_global is None else n_global
        self.row_lo, self.row_hi = row_lo, row_lo + data.n
        nq = min(self.etr.n_queries, n)
        q_idx = np.random.default_rng([self.seed, 4]).choice(n, size=nq, replace=False)
        self.q_idx = q_idx
        q = torch.zeros((nq, data.ld), dtype=torch.float32, device=dev)
        mine = np.flatnonzero((q_idx >= row_lo) & (q_idx < row_lo + data.n))
        if mine.size:
            src = torch.tensor(q_idx[mine] - row_lo, dtype=torch.int64, device=dev)
            tmp = torch.empty((mine.size, data.ld), dtype=torch.float32, device=dev)
            native.call("skm_gather_rows", ptr(data.x), data.ld, ptr(src), int(mine.size), data.ld, ptr(tmp),
                        data.ld, stream_handle())
            q[torch.tensor(mine, dtype=torch.int64, device=dev)] = tmp
        comm.allreduce_(q)
        self.q = q
        self.q_sq = _norms(q, data.d)
        top_k = self.top_k
        if top_k > n:
            raise ValueError(f"k_gt={top_k} exceeds collection size {n}")
        gi, gv = device_topk_distances(q, None, None, self.q_sq, data.x, None, None, data.norms(data.d), data.d, top_k,
                                       col_offset=row_lo)
        if comm.world > 1:
            # per-rank top-k -> allgather -> stable (dist, index) merge
            kk = gi.shape[1]
            ai = [torch.empty_like(gi) for _ in range(comm.world)]
            av = [torch.empty_like(gv) for _ in range(comm.world)]
            comm.dist.all_gather(ai, gi.contiguous(), group=comm.group)
            comm.dist.all_gather(av, gv.contiguous(), group=comm.group)
            gi, gv = merge_topk_shards(torch.stack(ai).contiguous(), torch.stack(av).contiguous(), comm.world, kk, nq,
                                       top_k)
        self.gt_idx, self.gt_val = gi.contiguous(), gv.contiguous()
        self.hits = torch.zeros(nq, dtype=torch.int32, device=dev)

    def probe(self, data, cents, ws, comm, gt_assign: torch.Tensor | None = None) -> float:
        """Recall of this iteration (evaluation.py:142-170).  ``gt_assign``: the assignments of
        every ground-truth slot, delivered by the iteration's one allreduce at N > 1 (engine.Reducer)
        -- the tally is then local on every rank and needs no collective of its own."""
        nq = self.q.shape[0]
        c_sq = _norms(cents.c, cents.d)
        pi, _ = device_topk_distances(self.q, None, None, self.q_sq, cents.c, None, None, c_sq, cents.d, self.nprobe)
        if gt_assign is not None:
            # slots as rows: slot s of query q holds gt_assign[q * top_k + t]
            if getattr(self, "_slots", None) is None:
                self._slots = torch.arange(nq * self.top_k, dtype=torch.int32, device=self.q.device).view(nq, -1)
            native.call("skm_etr_hits", ptr(self._slots), self.top_k, self.top_k, ptr(pi), pi.shape[1], pi.shape[1],
                        ptr(gt_assign), 0, nq * self.top_k, cents.k, nq, ptr(self.hits), stream_handle())
            h = self.hits
        else:
            native.call("skm_etr_hits", ptr(self.gt_idx), self.gt_idx.shape[1], self.top_k, ptr(pi), pi.shape[1],
                        pi.shape[1], ptr(ws.assign), self.row_lo, self.row_hi, cents.k, nq, ptr(self.hits),
                        stream_handle())
            h = comm.allreduce_(self.hits.to(torch.int64)) if comm.world > 1 else self.hits
        hits = h.cpu().numpy()
        total = 0.0
        for v in hits:  # the reference's accumulation order (evaluation.py:169-170)
            total += int(v) / self.top_k
        return total / nq

    def should_stop(self, history) -> bool:
        return etr_should_stop(history, self.etr.tolerance, self.etr.patience_iters)


# ------------------------------------------------------------------ host-array entry points
@on_device
def brute_force_topk(x, queries, k_gt: int, query_batch: int = 128, device=None) -> GroundTruth:
    """Exact top-k by squared L2 over the collection, ties to the lower index
    (evaluation.py:53-75), computed on the B200."""
    from .config import DimensionMismatch
    x = np.ascontiguousarray(x, dtype=np.float32)
    queries = np.ascontiguousarray(queries, dtype=np.float32)
    if x.shape[1] != queries.shape[1]:
        raise DimensionMismatch(f"data dim {x.shape[1]} != query dim {queries.shape[1]}")
    if k_gt > x.shape[0]:
        raise ValueError(f"k_gt={k_gt} exceeds collection size {x.shape[0]}")
    dev = require_cuda(device)
    from .api import _h2d
    d = x.shape[1]
    X = _h2d(x, dev)
    Q = _h2d(queries, dev)
    gi, gv = device_topk_distances(Q, None, None, _norms(Q, d), X, None, None, _norms(X, d), d, k_gt)
    return GroundTruth(indices=gi.cpu().numpy().astype(np.int64), distances=gv.cpu().numpy(), k_gt=k_gt)


@on_device
def build_cluster_lists(assignments, k: int, device=None) -> list:
    """Per-cluster row lists in ascending row order (evaluation.py:78-83) from the device
    stable cluster sort."""
    a = np.ascontiguousarray(assignments, dtype=np.int32)
    dev = require_cuda(device)
    n = a.shape[0]
    A = torch.from_numpy(a).to(dev)
    order = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    counts = torch.empty(k, dtype=torch.int32, device=dev)
    offs = torch.empty(k, dtype=torch.int32, device=dev)
    ws = torch.empty(int(native.load().skm_update_workspace_bytes(n, k)), dtype=torch.uint8, device=dev)
    native.call("skm_cluster_sort", ptr(A), n, k, ptr(order), ptr(counts), ptr(offs), ptr(ws), ws.numel(),
                stream_handle())
    o = order[:n].cpu().numpy().astype(np.int64)
    bounds = np.cumsum(counts.cpu().numpy().astype(np.int64))[:-1]
    return np.split(o, bounds)


@on_device
def etr_probe(centroids, train_x, assignments, queries, gt: GroundTruth, nprobe: int, top_k: int,
              device=None) -> float:
    """Mean probe recall of the current state (evaluation.py:142-170), device tally."""
    dev = require_cuda(device)
    from .api import _h2d
    c = np.ascontiguousarray(centroids, dtype=np.float32)
    q = np.ascontiguousarray(queries, dtype=np.float32)
    k, d = c.shape
    nprobe = min(max(1, nprobe), k)
    Cd, Qd = _h2d(c, dev), _h2d(q, dev)
    pi, _ = device_topk_distances(Qd, None, None, _norms(Qd, d), Cd, None, None, _norms(Cd, d), d, nprobe)
    gt_i = torch.from_numpy(np.ascontiguousarray(gt.indices[:, :top_k], dtype=np.int32)).to(dev)
    A = torch.from_numpy(np.ascontiguousarray(assignments, dtype=np.int32)).to(dev)
    hits = torch.zeros(q.shape[0], dtype=torch.int32, device=dev)
    native.call("skm_etr_hits", ptr(gt_i), gt_i.shape[1], top_k, ptr(pi), pi.shape[1], nprobe, ptr(A), 0,
                A.shape[0], k, q.shape[0], ptr(hits), stream_handle())
    total = 0.0
    for v in hits.cpu().numpy():
        total += int(v) / top_k
    return total / q.shape[0]


# ------------------------------------------------------------------ IVF probe evaluation
def _lists_to_assign(cluster_lists, n: int) -> tuple[np.ndarray, np.ndarray]:
    """Invert cluster lists into a row -> cluster array (-1: in no list) and list sizes."""
    assign = np.full(n, -1, dtype=np.int32)
    sizes = np.empty(len(cluster_lists), dtype=np.int32)
    for c, lst in enumerate(cluster_lists):
        lst = np.asarray(lst, dtype=np.int64)
        assign[lst] = c
        sizes[c] = lst.size
    return assign, sizes


def _probe_ranking(centroids: np.ndarray, queries: np.ndarray, nprobe: int, dev) -> torch.Tensor:
    """Top-nprobe centroids per query by squared L2, ties to the lower index (the stable
    argsort of evaluation.py:97,196): distance GEMM + exact device top-k."""
    from .api import _h2d
    k, d = centroids.shape
    Cd, Qd = _h2d(np.ascontiguousarray(centroids, dtype=np.float32), dev), _h2d(
        np.ascontiguousarray(queries, dtype=np.float32), dev)
    pi, _ = device_topk_distances(Qd, None, None, _norms(Qd, d), Cd, None, None, _norms(Cd, d), d, nprobe)
    return pi


@on_device
def probe_eval(centroids, cluster_lists, x, queries, gt: GroundTruth, nprobe: int, top_ks=(10, 100),
               device=None) -> dict:
    """IVF probe-search quality (evaluation.py:173-203): recall@t for each t <= gt.k_gt and the
    mean number of vectors scanned per query, on the B200.

    A query's candidates are the members of its nprobe nearest clusters.  Its top-t by
    (distance, index) among them contains exactly the ground-truth members GT[:t] that are
    candidates (every row closer than such a member is itself in GT[:t]), so recall@t is the
    integer tally #{g in GT[:t] : cluster(g) in probe} / t -- the reference's value up to
    distance near-ties between its two GEMM calls.  Sums run in query order in
    f64 like the reference."""
    from .config import DimensionMismatch
    dev = require_cuda(device)
    c = np.ascontiguousarray(centroids, dtype=np.float32)
    q = np.ascontiguousarray(queries, dtype=np.float32)
    n = np.asarray(x).shape[0]
    if np.asarray(x).shape[1] != q.shape[1] or c.shape[1] != q.shape[1]:
        raise DimensionMismatch("dim mismatch between vectors, centroids and queries")
    k = c.shape[0]
    nprobe = min(max(1, nprobe), k)
    top_ks = sorted({t for t in top_ks if t <= gt.k_gt})
    nq = q.shape[0]
    assign, sizes = _lists_to_assign(cluster_lists, n)
    pi = _probe_ranking(c, q, nprobe, dev)
    A = torch.from_numpy(assign).to(dev)
    S = torch.from_numpy(sizes).to(dev)
    gt_i = torch.from_numpy(np.ascontiguousarray(gt.indices, dtype=np.int32)).to(dev)
    explored = torch.zeros(max(nq, 1), dtype=torch.int64, device=dev)
    out = {}
    hits_by_t = {}
    for n_t, t in enumerate(top_ks):
        hits = torch.zeros(max(nq, 1), dtype=torch.int32, device=dev)
        native.call("skm_probe_tally", ptr(gt_i), gt_i.shape[1], t, ptr(pi), pi.shape[1], nprobe, ptr(A), n, k, nq,
                    ptr(S) if n_t == 0 else None, ptr(hits), ptr(explored) if n_t == 0 else None, stream_handle())
        hits_by_t[t] = hits[:nq].cpu().numpy()
    if not top_ks:  # still count the explored vectors
        hits = torch.zeros(max(nq, 1), dtype=torch.int32, device=dev)
        native.call("skm_probe_tally", ptr(gt_i), gt_i.shape[1], 0, ptr(pi), pi.shape[1], nprobe, ptr(A), n, k, nq,
                    ptr(S), ptr(hits), ptr(explored), stream_handle())
    for t in top_ks:
        total = 0.0
        for v in hits_by_t[t]:
            total += int(v) / t
        out[f"recall_at_{t}"] = total / nq
    out["vectors_explored_mean"] = int(explored[:nq].sum().item()) / nq
    return out


@on_device
def ivf_probe_search(centroids, cluster_lists, x, q, nprobe: int, top_k: int, device=None):
    """Scan the nprobe clusters nearest to one query (evaluation.py:86-105).  Returns
    (indices int64, squared distances float32, vectors_explored); ties resolve to the lower
    row index.  Probe ranking, candidate distances (3xTF32 GEMM, the reference's expansion
    op order) and the top-k run on the B200."""
    dev = require_cuda(device)
    from .api import _h2d
    from .engine import _gemm
    c = np.ascontiguousarray(centroids, dtype=np.float32)
    k = c.shape[0]
    nprobe = min(nprobe, k)
    q2 = np.ascontiguousarray(np.asarray(q, dtype=np.float32).reshape(1, -1))
    probe = _probe_ranking(c, q2, max(nprobe, 1), dev)[0, :nprobe].cpu().numpy()
    cand = np.concatenate([np.asarray(cluster_lists[int(p)], dtype=np.int64) for p in probe])
    if cand.size == 0:
        return np.empty(0, dtype=np.int64), np.empty(0, dtype=np.float32), 0
    take = min(top_k, cand.size)
    # candidates in ascending row order: column ties in the device top-k then resolve to the
    # lower row index, as the reference's lexsort((cand, d2)) does
    srt = np.sort(cand)
    xs = np.ascontiguousarray(np.asarray(x, dtype=np.float32)[srt])
    d = xs.shape[1]
    X = _h2d(xs, dev)
    Q = _h2d(q2, dev)
    xh, xl = _split(X, d)
    qh, ql = _split(Q, d)
    m = X.shape[0]
    D = torch.empty((1, padded_ld(m)), dtype=torch.float32, device=dev)
    _gemm(qh, ql, xh, xl, 1, m, d, native.GEMM_DIST, out=D, xsq=_norms(Q, d), ysq=_norms(X, d))
    oi = torch.empty((1, take), dtype=torch.int32, device=dev)
    ov = torch.empty((1, take), dtype=torch.float32, device=dev)
    if take <= TOPK_MAX:
        native.call("skm_topk_rows", ptr(D), D.stride(0), 1, m, take, ptr(oi), ptr(ov), take, 0, stream_handle())
    else:
        v, i = torch.sort(D[:, :m], dim=1, stable=True)
        ov.copy_(v[:, :take])
        oi.copy_(i[:, :take].to(torch.int32))
    cols = oi[0].cpu().numpy().astype(np.int64)
    return srt[cols], ov[0].cpu().numpy(), int(cand.size)


def recall_at_k(result_ids, gt_row, k: int) -> float:
    """|result[:k] & gt[:k]| / k (evaluation.py:108-113)."""
    result_ids, gt_row = np.asarray(result_ids), np.asarray(gt_row)
    if len(result_ids) < k or len(gt_row) < k:
        raise ValueError(f"need at least {k} entries on both sides")
    return np.intersect1d(result_ids[:k], gt_row[:k]).size / k


@on_device
def wcss(x, centroids, assignments, batch: int = 4096, device=None) -> float:
    """Sum of squared distances to the assigned centroids in double (evaluation.py:205-215),
    on the B200 (deterministic fixed-order reduction)."""
    from .api import _h2d
    from .config import DimensionMismatch
    x = np.ascontiguousarray(x, dtype=np.float32)
    c = np.ascontiguousarray(centroids, dtype=np.float32)
    if x.shape[1] != c.shape[1]:
        raise DimensionMismatch("dim mismatch between vectors and centroids")
    dev = require_cuda(device)
    X, Cd = _h2d(x, dev), _h2d(c, dev)
    A = torch.from_numpy(np.ascontiguousarray(assignments, dtype=np.int32)).to(dev)
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    ws = torch.empty(int(native.load().skm_wcss_workspace_bytes()) // 8, dtype=torch.float64, device=dev)
    native.call("skm_wcss", ptr(X), X.shape[1], ptr(Cd), Cd.shape[1], ptr(A), x.shape[0], x.shape[1], ptr(out),
                ptr(ws), stream_handle())
    return float(out.item())


def balance_stats(counts) -> dict:
    """Points-per-cluster mean and population standard deviation (evaluation.py:218-222)."""
    counts = np.asarray(counts, dtype=np.float64)
    return {"mean": float(counts.mean()), "std_dev": float(counts.std())}

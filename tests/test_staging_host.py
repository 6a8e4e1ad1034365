"""Host logic of the staged pageable -> device copy (api._copy_rows_to_device), no GPU: the
pinned ring, events and stream are replaced by CPU stand-ins so the chunk / thread-slice
arithmetic (including a gather by row index) is checked on ragged sizes."""

import numpy as np
import pytest
import torch


class _Event:
    def record(self, stream=None):
        pass

    def synchronize(self):
        pass


@pytest.fixture
def staged(monkeypatch):
    from paper_2603_20009_b200 import api
    monkeypatch.setattr(api, "_STAGE_BYTES", 1 << 14)  # tiny chunks: many ring turns
    monkeypatch.setattr(api, "_STAGE_THREADS", 3)
    monkeypatch.setattr(torch.cuda, "Event", _Event)
    monkeypatch.setattr(torch.cuda, "current_stream", lambda dev=None: None)
    real_empty = torch.empty
    monkeypatch.setattr(torch, "empty", lambda *a, **k: real_empty(*a, **{x: v for x, v in k.items()
                                                                            if x != "pin_memory"}))
    return api


@pytest.mark.parametrize("n,d", [(10007, 37), (4096, 64), (333, 129), (70000, 5)])
def test_staged_copy_rows(staged, n, d):
    x = np.random.default_rng(n).standard_normal((n, d)).astype(np.float32)
    ld = (d + 3) // 4 * 4
    out = torch.zeros((n, ld))
    staged._copy_rows_to_device(x, out, d)
    assert np.array_equal(out[:, :d].numpy(), x)
    assert float(out[:, d:].abs().sum()) == 0.0


@pytest.mark.parametrize("n,d,m", [(20011, 33, 7001), (5000, 64, 4999), (9000, 17, 1)])
def test_staged_gather_rows(staged, n, d, m):
    x = np.random.default_rng(m).standard_normal((n, d)).astype(np.float32)
    idx = np.sort(np.random.default_rng(m + 1).choice(n, m, replace=False))
    out = torch.zeros((m, d))
    staged._copy_rows_to_device(x, out, d, idx)
    assert np.array_equal(out.numpy(), x[idx])


class _Stream:
    def wait_event(self, ev):
        pass


@pytest.fixture
def prefetch(staged, monkeypatch):
    import contextlib
    monkeypatch.setattr(torch.cuda, "Stream", lambda dev=None: _Stream())
    monkeypatch.setattr(torch.cuda, "stream", lambda s: contextlib.nullcontext())
    monkeypatch.setattr(torch.cuda, "current_stream", lambda dev=None: _Stream())
    monkeypatch.setattr(torch.Tensor, "record_stream", lambda self, s: None, raising=False)
    return staged


def test_prefetch_batches_cover_rows_in_order(prefetch):
    x = np.random.default_rng(3).standard_normal((10_501, 19)).astype(np.float32)
    got = []
    for s0, e0, xb in prefetch._prefetch_batches(x, 1000, "cpu"):
        assert xb.shape[0] == e0 - s0
        got.append((s0, e0, xb[:, :19].numpy().copy()))
    assert [g[0] for g in got] == list(range(0, 10_501, 1000))
    assert np.array_equal(np.concatenate([g[2] for g in got]), x)


def test_prefetch_batches_early_exit_stops_worker(prefetch):
    import threading
    x = np.zeros((50_000, 8), np.float32)
    before = threading.active_count()
    for i, _ in enumerate(prefetch._prefetch_batches(x, 100, "cpu")):
        if i == 2:
            break  # the consumer raises / stops: the generator's finally must stop and join the worker
    assert threading.active_count() <= before

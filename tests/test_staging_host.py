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

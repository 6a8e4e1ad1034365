"""Streaming vector ingestion on the B200 (pinned double buffer -> H2D -> validate/scatter
kernel) against the reference's load_vectors outcomes on valid and malformed files."""

import os

import numpy as np
import pytest

from dataio_cases import build_case

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "dataio.npz"))


def _cases():
    src = open(os.path.join(HERE, "golden", "make_golden.py")).read()
    start = src.index("DATAIO_CASES = {")
    ns = {}
    exec(src[start:src.index("}\n", start) + 1], ns)
    return ns["DATAIO_CASES"]


CASES = _cases()


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("chunk_bytes", [1 << 20, 37 * 1024])  # transfer chunks unrelated to 4096-row reports
def test_load_vectors_matches_reference(tmp_path, name, chunk_bytes):
    import paper_2603_20009_b200 as skb
    from paper_2603_20009_b200 import dataio
    path = build_case(str(tmp_path), name, CASES[name])
    want = str(G[f"{name}_outcome"])
    if want == "ok":
        x = dataio.load_vectors_device(path, chunk_bytes=chunk_bytes)
        fmt, n, d, _ = CASES[name]
        host = x.cpu().numpy()
        assert host.shape[0] == n and np.all(host[:, d:] == 0)
        assert float(host[:, :d].astype(np.float64).sum()) == float(G[f"{name}_sum"])
        ref = np.fromfile(path, dtype="<f4", offset=8).reshape(n, d) if fmt == "fbin" else \
            np.fromfile(path, dtype=np.dtype([("dim", "<i4"), ("vec", "<f4", (d,))]))["vec"]
        assert np.array_equal(host[:, :d], ref)
        assert np.array_equal(skb.load_vectors(path), ref)
    else:
        with pytest.raises(getattr(skb, want)) as ei:
            dataio.load_vectors_device(path, chunk_bytes=chunk_bytes)
        row, col = G[f"{name}_rowcol"]
        if row >= 0:
            assert ei.value.row == row
        if col >= 0:
            assert ei.value.col == col
        assert str(ei.value).replace(str(tmp_path), "<dir>") == str(G[f"{name}_msg"])


def test_normalize_rows(tmp_path):
    from paper_2603_20009_b200 import dataio
    x = np.random.default_rng(1).standard_normal((3000, 33)).astype(np.float32)
    x[7] = 0
    dataio.write_fbin(tmp_path / "a.fbin", x)
    got = dataio.load_vectors(tmp_path / "a.fbin", normalize=True)
    n = np.linalg.norm(x, axis=1, keepdims=True)
    n[n == 0] = 1
    np.testing.assert_allclose(got, x / n, rtol=2e-7, atol=1e-7)
    assert np.all(got[7] == 0)

"""CPU: model / ground-truth file formats byte-identical to the reference (golden bytes written
by the real reference, tests/golden/make_golden.py --only-dataio) and the header checks of the
vector loaders (the record/value checks run on the device: tests/test_gpu_dataio.py)."""

import os

import numpy as np
import pytest

from dataio_cases import build_case

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "dataio.npz"))


def _spec(name):
    src = open(os.path.join(HERE, "golden", "make_golden.py")).read()
    start = src.index("DATAIO_CASES = {")
    ns = {}
    exec(src[start:src.index("}\n", start) + 1], ns)
    return ns["DATAIO_CASES"][name]


def test_skmc_and_skgt_bytes_match_reference(tmp_path):
    from paper_2603_20009_b200 import dataio
    from paper_2603_20009_b200.etr import GroundTruth
    c = G["model_centroids"]
    dataio.save_centroids(tmp_path / "m0.skmc", c, 42)
    dataio.save_centroids(tmp_path / "m1.skmc", c, 7, cluster_lists=[np.arange(i) for i in range(7)])
    dataio.save_ground_truth(tmp_path / "g.skgt", GroundTruth(indices=G["gt_indices"], distances=G["gt_distances"],
                                                              k_gt=4))
    for f in ("m0.skmc", "m1.skmc", "g.skgt"):
        assert (tmp_path / f).read_bytes() == G["bytes_" + f.replace(".", "_")].tobytes(), f
    # and the readers parse the reference's files
    (tmp_path / "r1.skmc").write_bytes(G["bytes_m1_skmc"].tobytes())
    m = dataio.load_centroids(tmp_path / "r1.skmc")
    assert m.rotation_seed == 7 and np.array_equal(m.centroids, c)
    assert [list(v) for v in m.cluster_lists] == [list(range(i)) for i in range(7)]
    (tmp_path / "r.skgt").write_bytes(G["bytes_g_skgt"].tobytes())
    g = dataio.load_ground_truth(tmp_path / "r.skgt")
    assert np.array_equal(g.indices, G["gt_indices"]) and np.array_equal(g.distances, G["gt_distances"])


def test_model_corruption_and_version_errors(tmp_path):
    from paper_2603_20009_b200 import ChecksumMismatch, MalformedHeader, VersionMismatch, dataio
    raw = bytearray(G["bytes_m0_skmc"].tobytes())
    bad = bytearray(raw)
    bad[30] ^= 1
    (tmp_path / "c.skmc").write_bytes(bytes(bad))
    with pytest.raises(ChecksumMismatch):
        dataio.load_centroids(tmp_path / "c.skmc")
    v = bytearray(raw)
    v[4] = 2
    (tmp_path / "v.skmc").write_bytes(bytes(v))
    with pytest.raises(VersionMismatch):
        dataio.load_centroids(tmp_path / "v.skmc")
    (tmp_path / "x.skmc").write_bytes(b"NOPE" + bytes(raw[4:]))
    with pytest.raises(MalformedHeader):
        dataio.load_centroids(tmp_path / "x.skmc")


@pytest.mark.parametrize("name", ["fbin_truncated", "fbin_bad_header", "fvecs_bad_header"])
def test_header_errors_match_reference(tmp_path, name):
    import paper_2603_20009_b200 as skb
    path = build_case(str(tmp_path), name, _spec(name))
    want = str(G[f"{name}_outcome"])
    with pytest.raises(getattr(skb, want)):
        skb.load_vectors(path)


def test_infer_format_and_writers_roundtrip(tmp_path):
    from paper_2603_20009_b200 import MalformedHeader, dataio
    assert dataio.infer_format("a.fvecs") == "fvecs"
    assert dataio.infer_format("a.BIN") == "fbin"
    with pytest.raises(MalformedHeader):
        dataio.infer_format("a.npy")
    x = np.random.default_rng(0).standard_normal((5, 3)).astype(np.float32)
    dataio.write_fvecs(tmp_path / "a.fvecs", x)
    dataio.write_fbin(tmp_path / "a.fbin", x)
    raw = (tmp_path / "a.fvecs").read_bytes()
    assert len(raw) == 5 * 16 and np.frombuffer(raw[:4], "<i4")[0] == 3
    assert (tmp_path / "a.fbin").read_bytes()[8:] == x.tobytes()

"""The CLI (fit / gt / eval) on the B200 against the reference CLI's reports on the same file
(tests/golden/cli.npz): identical structure and integer fields, floats to GEMM rounding."""

import json
import os

import numpy as np
import pytest

from conftest import make_blobs

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "cli.npz"))


def _close(a, b, path=""):
    if isinstance(a, dict):
        assert sorted(a) == sorted(b), (path, sorted(a), sorted(b))
        for k in a:
            _close(a[k], b[k], f"{path}.{k}")
    elif isinstance(a, list):
        assert len(a) == len(b), path
        for i, (u, v) in enumerate(zip(a, b)):
            _close(u, v, f"{path}[{i}]")
    elif isinstance(a, float) and isinstance(b, float):
        assert abs(a - b) <= 1e-5 * max(1.0, abs(b)), (path, a, b)
    else:
        assert a == b, (path, a, b)


def test_cli_fit_gt_eval_match_reference(tmp_path):
    from paper_2603_20009_b200 import dataio
    from paper_2603_20009_b200.cli import main
    x = make_blobs(2000, 48, 12, seed=8)
    path = str(tmp_path / "d.fbin")
    dataio.write_fbin(path, x)
    rep, model = str(tmp_path / "fit.json"), str(tmp_path / "m.skmc")
    assert main(["fit", "--input", path, "--k", "12", "--iters", "4", "--seed", "9", "--eval-queries", "50",
                 "--out-centroids", model, "--report", rep]) == 0
    ours = dataio.RunReport.load(rep).comparable()
    ref = json.loads(str(G["fit_report"]))
    ours["dataset"]["path"] = ref["dataset"]["path"]
    _close(ours, ref)
    gtp = str(tmp_path / "g.skgt")
    assert main(["gt", "--input", path, "--n-queries", "40", "--topk", "20", "--seed", "3", "--out", gtp]) == 0
    g_ours = open(gtp, "rb").read()
    g_ref = G["gt_bytes"].tobytes()
    assert len(g_ours) == len(g_ref) and g_ours[:12] == g_ref[:12]
    idx_o = np.frombuffer(g_ours[12:12 + 40 * 20 * 4], "<i4")
    idx_r = np.frombuffer(g_ref[12:12 + 40 * 20 * 4], "<i4")
    assert np.mean(idx_o == idx_r) >= 0.99  # distance near-ties only
    rep2 = str(tmp_path / "eval.json")
    assert main(["eval", "--centroids", model, "--input", path, "--gt", gtp, "--n-queries", "40", "--seed", "3",
                 "--topk", "20", "--report", rep2]) == 0
    e_ours = dataio.RunReport.load(rep2).comparable()
    e_ref = json.loads(str(G["eval_report"]))
    e_ours["dataset"]["path"] = e_ref["dataset"]["path"]
    e_ours["notes"]["centroids"] = e_ref["notes"]["centroids"]
    _close(e_ours, e_ref)
    # the model file: same container layout, centroids to GEMM rounding, identical lists
    m = dataio.load_centroids(model)
    (tmp_path / "r.skmc").write_bytes(G["model_bytes"].tobytes())
    r = dataio.load_centroids(tmp_path / "r.skmc")
    assert m.rotation_seed == r.rotation_seed and m.k == r.k
    np.testing.assert_allclose(m.centroids, r.centroids, rtol=1e-4, atol=1e-4)
    assert [list(a) for a in m.cluster_lists] == [list(b) for b in r.cluster_lists]


def test_cli_reproducible_and_errors(tmp_path):
    from paper_2603_20009_b200 import dataio
    from paper_2603_20009_b200.cli import main
    x = make_blobs(800, 40, 6, seed=2)
    path = str(tmp_path / "d.fvecs")
    dataio.write_fvecs(path, x)
    reps = []
    for i in (0, 1):
        rp = str(tmp_path / f"r{i}.json")
        assert main(["fit", "--input", path, "--k", "6", "--iters", "3", "--seed", "4", "--eval-queries", "30",
                     "--report", rp, "--out-centroids", str(tmp_path / "m.skmc")]) == 0
        reps.append(dataio.RunReport.load(rp).comparable())
    assert reps[0] == reps[1]
    gtp = str(tmp_path / "g.skgt")
    assert main(["gt", "--input", path, "--n-queries", "16", "--topk", "5", "--out", gtp]) == 0
    assert main(["eval", "--centroids", str(tmp_path / "m.skmc"), "--input", path, "--gt", gtp, "--topk", "50"]) == 1

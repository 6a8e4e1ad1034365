"""CPU: CLI argument surface and defaults mirror the reference (cli.py:53-132)."""

import pytest


def test_default_k_and_parser():
    from paper_2603_20009_b200.cli import build_parser, default_k
    assert default_k(1_000_000) == 4000
    assert default_k(10) == 16
    p = build_parser()
    a = p.parse_args(["fit", "--input", "x.fbin", "--etr-tol", "off", "--sample", "0.5"])
    assert a.etr_tol is None and a.sample == 0.5 and a.iters == 25 and a.eval_queries == 1000
    a = p.parse_args(["eval", "--centroids", "m", "--input", "x"])
    assert a.nprobe_frac == 0.01 and a.topk == 100 and a.n_queries == 1000
    for bad in (["fit", "--input", "x", "--k", "0"], ["fit", "--input", "x", "--sample", "1.5"],
                ["fit", "--input", "x", "--etr-tol", "-1"], ["gt", "--input", "x"]):
        with pytest.raises(SystemExit):
            p.parse_args(bad)


def test_report_roundtrip_and_comparable(tmp_path):
    from paper_2603_20009_b200 import VersionMismatch
    from paper_2603_20009_b200.dataio import RunReport
    r = RunReport(command="fit", config={"k": 3}, dataset={"n": 1}, iterations=[{"wcss": 1.0, "timings": {"a": 1}}],
                  final_metrics={"wcss": 2.0, "wall_clock_seconds": 3.0}, phase_seconds={"x": 1.0},
                  terminated_by="max_iters")
    r.save(tmp_path / "r.json")
    r2 = RunReport.load(tmp_path / "r.json")
    assert r2 == r
    c = r2.comparable()
    assert "phase_seconds" not in c and "timings" not in c["iterations"][0]
    assert "wall_clock_seconds" not in c["final_metrics"]
    (tmp_path / "v.json").write_text(r.to_json().replace('"version": 1', '"version": 2'))
    with pytest.raises(VersionMismatch):
        RunReport.load(tmp_path / "v.json")

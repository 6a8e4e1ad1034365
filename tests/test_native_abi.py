"""CPU: the C-ABI library builds for sm_100a, loads without a GPU and exports every symbol the
public header declares (no compute calls here)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "skm_b200.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(skm_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_protocol():
    names = _declared()
    for must in ("skm_scan_bank", "skm_seed_thresholds", "skm_accumulate_centroid_sums", "skm_portable_matmul",
                 "skm_gemm_tf32x3", "skm_pruned_scan", "skm_cluster_sort", "skm_topk_rows", "skm_etr_hits"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2603_20009_b200 import build, native
    build.build()
    lib = ctypes.CDLL(native.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    # the Python binding covers the same surface
    assert set(_declared()) <= set(native.EXPORTED_SYMBOLS), set(_declared()) - set(native.EXPORTED_SYMBOLS)
    assert lib.skm_abi_version() == 1


def test_library_is_sm100a_with_tcgen05():
    import shutil
    import subprocess
    from paper_2603_20009_b200 import native
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "-sass", native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", native.LIB_PATH], capture_output=True,
                                       text=True).stdout
    assert "UTCHMMA" in out  # tcgen05.mma
    assert "UTMALDG" in out  # TMA tensor loads
    assert "LDTM" in out     # tcgen05.ld (TMEM -> registers)


def test_no_cpu_fallback_without_library(monkeypatch):
    """The product fails loudly when the extension is missing (no silent CPU path)."""
    from paper_2603_20009_b200 import native
    monkeypatch.setattr(native, "_lib", None)
    monkeypatch.setattr(native, "LIB_PATH", "/nonexistent/libskm_b200.so")
    with pytest.raises(native.NativeUnavailable):
        native.load()


def test_drop_in_names_cover_the_reference_api():
    """Every public name of the reference package (its __all__, pkg/src/superkmeans/__init__.py)
    exists in ours (checked against the unmodified install in baseline/_ref when present)."""
    import importlib
    import os
    import subprocess
    import sys
    ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "superkmeans")):
        pytest.skip("reference not installed (baseline/_ref)")
    out = subprocess.run([sys.executable, "-c", "import superkmeans as s; print(' '.join(s.__all__))"],
                         capture_output=True, text=True, env=dict(os.environ, PYTHONPATH=ref), check=True)
    names = out.stdout.split()
    ours = importlib.import_module("paper_2603_20009_b200")
    assert len(names) >= 40
    assert [n for n in names if not hasattr(ours, n)] == []

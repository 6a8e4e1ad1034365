"""CPU: host-side logic of the drop-in (configs, validation, layout, RNG-bound decisions) against
the reference's known answers (pkg/tests/test_model.py, test_core.py, test_pruning.py,
test_evaluation.py) and the golden host-math fixtures."""

import os

import numpy as np
import pytest

import paper_2603_20009_b200 as skm
from paper_2603_20009_b200 import hostmath
from paper_2603_20009_b200.config import (
    DimensionMismatch,
    EmptySample,
    KTooLarge,
    NonFiniteValue,
    initial_d_prime,
    pdxify,
    pruning_supported,
    tail_block_layout,
    validate_vector_set,
)

H = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "hostmath.npz"))


def test_rotation_bitwise_vs_reference():
    for d, s in ((64, 3), (200, 0), (96, 7)):
        assert np.array_equal(hostmath.generate_rotation(d, s).data, H[f"rot_{d}_{s}"])


def test_adjust_d_prime_known_answers():
    cfg = skm.KMeansConfig(k=4)
    for (a, r, d), want in zip(H["adjust_in"], H["adjust_out"]):
        assert skm.adjust_d_prime(int(a), float(r), cfg, int(d)) == int(want)
    assert skm.adjust_d_prime(192, 0.99, cfg, 1536) == 152
    assert skm.adjust_d_prime(96, 0.90, cfg, 1536) == 120
    assert skm.adjust_d_prime(18, 0.999, cfg, 1536) == 16
    assert skm.adjust_d_prime(1400, 0.5, cfg, 1536) == 1472


def test_threshold_factors_bitwise():
    _, b = tail_block_layout(1536, 192)
    assert np.array_equal(hostmath.threshold_factors(1536, 192, b, 2.1), H["factors_1536_192"])
    _, b = tail_block_layout(200, 25)
    f = hostmath.threshold_factors(200, 25, b, 2.1)
    assert np.array_equal(f, H["factors_200_25"])
    assert f[-1] == np.float32(1.0)
    assert hostmath.adsampling_threshold(256, 1.0, 1024, 2.1) == pytest.approx(0.25 * (1 + 2.1 / 16.0) ** 2)
    s = hostmath.sentinel_factors(f)
    assert np.isinf(s[:-1]).all() and s[-1] == 1.0


def test_layout_known_answers():
    w, b = tail_block_layout(200, 25)
    assert w.tolist() == [64, 64, 47] and b.tolist() == [89, 153, 200]
    assert initial_d_prime(1536, 0.125) == 192 and initial_d_prime(128, 0.125) == 16
    assert initial_d_prime(200, 0.125) == 25
    assert pruning_supported(80) and not pruning_supported(79)
    with pytest.raises(DimensionMismatch):
        tail_block_layout(100, 100)


def test_pdxify_round_trip():
    c = np.random.default_rng(0).standard_normal((77, 200)).astype(np.float32)
    bank = pdxify(c, 25)
    assert np.array_equal(bank.reconstruct(), c)
    assert bank.block(1).shape == (64, 77)


def test_validation_errors():
    with pytest.raises(DimensionMismatch):
        validate_vector_set(np.zeros(5))
    with pytest.raises(DimensionMismatch):
        validate_vector_set(np.zeros(6), n_rows=2)
    x = np.zeros((3, 4), np.float32)
    x[1, 2] = np.nan
    with pytest.raises(NonFiniteValue) as e:
        validate_vector_set(x)
    assert (e.value.row, e.value.col) == (1, 2)
    assert validate_vector_set(np.zeros(6), n_rows=2, dim=3).shape == (2, 3)


def test_config_validation_and_defaults():
    c = skm.KMeansConfig(k=10)
    assert (c.max_iters, c.x_batch, c.y_batch, c.epsilon0, c.prune_target_low, c.prune_target_high) == \
        (25, 4096, 1024, 2.1, 0.95, 0.97)
    for bad in (dict(k=0), dict(k=1, max_iters=0), dict(k=1, y_batch=2048), dict(k=1, d_prime_init_fraction=1.0),
                dict(k=1, sampling_fraction=0.0), dict(k=1, prune_target_low=0.98),
                dict(k=1, d_prime_adjust_factor=1.5), dict(k=1, gemm_backend="cuda"),
                dict(k=1, kernel_backend="gpu")):
        with pytest.raises(ValueError):
            skm.KMeansConfig(**bad)
    e = skm.EtrConfig()
    assert (e.tolerance, e.patience_iters, e.n_queries, e.top_k, e.nprobe_fraction) == (0.005, 2, 1000, 100, 0.01)
    with pytest.raises(ValueError):
        skm.EtrConfig(nprobe_fraction=0)
    h = skm.HierarchicalConfig(k_total=65536)
    assert h.meso_k == 256 and h.k == 256
    assert skm.HierarchicalConfig(k_total=65536, meso_k=430).k == 430


def test_sampling_and_init_rng_streams():
    idx = hostmath.sample_indices(1000, 0.25, [3, 1])
    want = np.random.default_rng([3, 1]).choice(1000, size=250, replace=False)
    want.sort()
    assert np.array_equal(idx, want)
    assert hostmath.sample_indices(1000, 1.0, [3, 1]) is None
    with pytest.raises(EmptySample):
        hostmath.sample_indices(50, 0.5, [0, 1], k=40)
    with pytest.raises(KTooLarge):
        hostmath.init_indices(10, 11, [0, 2])


def test_split_plan_matches_reference_rng():
    from oracle import skm_ref
    counts = np.array([10, 0, 7, 0, 3], np.int64)
    c = np.random.default_rng(0).standard_normal((5, 6)).astype(np.float32)
    c_ref = c.copy()
    cnt_ref = counts.copy()
    skm_ref.split(c_ref, cnt_ref, np.random.default_rng(9))
    cnt = counts.copy()
    empties, donors = hostmath.plan_splits(cnt, np.random.default_rng(9))
    assert empties == [1, 3]
    assert np.array_equal(cnt, cnt_ref)


def test_etr_stop_rule():
    stop = hostmath.etr_should_stop
    assert not stop([0.5, 0.6], 0.005)
    assert stop([0.9, 0.902, 0.903], 0.005)
    assert not stop([0.9, 0.91, 0.911], 0.005)
    assert not stop([0.9, 0.901, 0.91], 0.005)
    assert stop([0.5, 0.6, 0.9, 0.9, 0.9], 0.0)


def test_sub_seed_and_reconcile():
    assert hostmath.sub_seed(2, 0) == int(np.random.SeedSequence([2, 5, 0]).generate_state(1)[0])
    from paper_2603_20009_b200.hierarchical import _fine_k, reconcile_k
    assert _fine_k(1) == 1 and _fine_k(100) == 10 and _fine_k(42) == round(np.sqrt(42))
    assert reconcile_k(238, 120) == {"requested_k": 120, "achieved_k": 238}


def test_chunked_generators_bitwise_reference_generators():
    """synth.py (row-chunked) == the reference's one-shot generators (conftest restatement)."""
    from conftest import make_blobs as mb, make_skewed_blobs as msb
    from paper_2603_20009_b200 import synth
    assert np.array_equal(synth.make_blobs(5000, 37, 11, 3, chunk_rows=777), mb(5000, 37, 11, 3))
    assert np.array_equal(synth.make_skewed_blobs(4000, 96, 64, 0, chunk_rows=1000), msb(4000, 96, 64, 0))


def test_scan_tail_limit_is_checked_on_the_host():
    """Tails beyond the one-warp scan's staging raise a SuperKMeansError before any launch, and the
    host limit equals the kernel's SCAN_NB_MAX_WIDE."""
    import os
    import re
    from paper_2603_20009_b200.config import SuperKMeansError
    from paper_2603_20009_b200.engine import SCAN_TAIL_BLOCKS_MAX, PrunePlan
    src = open(os.path.join(os.path.dirname(__file__), "..", "paper_2603_20009_b200", "csrc", "scan.cuh")).read()
    assert int(re.search(r"SCAN_NB_MAX_WIDE = (\d+);", src).group(1)) == SCAN_TAIL_BLOCKS_MAX
    d = 16 + 64 * SCAN_TAIL_BLOCKS_MAX + 1
    with pytest.raises(SuperKMeansError, match="exceeds the device scan"):
        PrunePlan(d, 16, 2.1, False, "cpu")

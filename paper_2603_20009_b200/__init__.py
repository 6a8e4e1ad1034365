"""B200-native SuperKMeans (arXiv 2603.20009): k-means for high-dimensional embeddings whose
Lloyd loop (rotation GEMM, fused partial-distance GEMM + ADSampling gate, exact pruning scan,
ordered centroid update, ETR) runs as hand-written sm_100a kernels (tcgen05/TMEM/TMA) behind
the reference package's Python API.

    import paper_2603_20009_b200 as skm          # instead of `import superkmeans as skm`
    res = skm.fit(x, skm.KMeansConfig(k=4096, max_iters=10))
    labels = skm.final_assign(x, res, cfg)
"""

from .api import KMeansResult, final_assign, fit
from .config import (
    ChecksumMismatch,
    InconsistentDim,
    MalformedHeader,
    TruncatedFile,
    VersionMismatch,
    D_PRIME_ALIGN,
    D_PRIME_MIN,
    MAX_BANK,
    PDX_BLOCK,
    AssignmentState,
    DimensionMismatch,
    EmptySample,
    EtrConfig,
    IterationStats,
    KMeansConfig,
    KTooLarge,
    NonFiniteValue,
    NormCache,
    PdxCentroidBank,
    RotationMatrix,
    SuperKMeansError,
    WorkCounters,
    initial_d_prime,
    pdxify,
    pruning_supported,
    tail_block_layout,
    validate_vector_set,
)
from .hostmath import (
    adjust_d_prime as _adjust_d_prime,
    adsampling_threshold,
    check_convergence,
    etr_should_stop,
    generate_rotation,
    prune_rate_from_totals,
    threshold_factors,
)

__version__ = "0.1.0"
HAS_COMPILED = True  # the CUDA library is the only backend


def adjust_d_prime(current_d_prime, prune_rate, cfg, dim):
    """core.adjust_d_prime (core.py:131-154)."""
    return _adjust_d_prime(current_d_prime, prune_rate, cfg, dim)


def get_kernels(name=None):
    from .device import get_kernels as _g
    return _g(name)


def available_backends():
    return ["cuda"]


def __getattr__(name):
    # lazily resolved, GPU-backed helpers
    if name in ("hierarchical_fit", "hierarchical_fit_device", "HierarchicalConfig", "reconcile_k"):
        from . import hierarchical
        return getattr(hierarchical, name)
    if name in ("brute_force_topk", "etr_probe", "build_cluster_lists", "GroundTruth", "RecallHistory",
                "probe_eval", "ivf_probe_search", "recall_at_k", "wcss", "balance_stats"):
        from . import etr
        return getattr(etr, name)
    if name in ("load_vectors", "load_vectors_device", "write_fvecs", "write_fbin", "infer_format", "sha256_file",
                "CentroidModel", "save_centroids", "load_centroids", "save_ground_truth", "load_ground_truth"):
        from . import dataio
        return getattr(dataio, name)
    if name in ("apply_rotation", "unapply_rotation", "sample_training_set", "init_centroids", "compute_norms",
                "update_centroids", "split_empty_clusters"):
        from . import extras
        return getattr(extras, name)
    if name in ("PruneOutcome", "initial_threshold", "prune_and_assign", "measure_prune_rate"):
        from . import pruning
        return getattr(pruning, name)
    if name in ("fit_lloyd", "LloydResult"):
        from . import lloyd
        return getattr(lloyd, name)
    raise AttributeError(name)

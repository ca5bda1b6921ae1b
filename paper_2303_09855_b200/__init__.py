"""B200-native IVF++ ADSampling engine (arXiv 2303.09855 hot path).

Drop-in for the reference's IVF/IVF++ search path: the C ABI is
include/adsann_b200.h (libadsann_b200.so, sm_100a kernels), and ``api``
mirrors the reference's adsann names for Python hosts.
"""
from .api import *  # noqa: F401,F403
from .api import (  # noqa: F401
    ALGO_LABELS, BatchResult, Context, DcoConfig, DcoOutcome, DeviceArray, IvfIndex, IvfLayout,
    IvfMode, KmeansResult, KnnResult, PinnedArray, QueryStats, TransformMatrix, Transform,
    ad_context_factor, ad_sampling, apply, apply_dataset, apply_prefix, apply_transpose,
    brute_force_knn, build_ivf, dco_fixed, device_count, fd_scan, generate_orthogonal,
    ivf_mode_from_name, ivf_mode_name, ivf_query, ivf_query_batch, kmeans, pd_scan, recall,
    recall_batch, rng_draw, search_opts, search_plan, synth, synth_rows, threshold_multiplier, TheoryRow, verify_theory,
)

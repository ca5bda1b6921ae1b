"""ctypes binding of libadsann_b200.so (include/adsann_b200.h).

The product path has no CPU fallback: if the library is missing the import
fails, and every compute entry point needs a CUDA device (ads_ctx_create
raises otherwise).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ADS_LIB_PATH") or os.path.join(HERE, "libadsann_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "adsann_b200.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA library first "
        "(python -c 'import __graft_entry__ as g; g.build()' or make -C paper_2303_09855_b200/csrc)"
    )

lib = C.CDLL(LIB_PATH)

vp = C.c_void_p
i32, i64, u64, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double
pi32, pi64, pu64, pf64, pf32 = (C.POINTER(i32), C.POINTER(i64), C.POINTER(u64), C.POINTER(f64),
                                C.POINTER(C.c_float))


class SynthDesc(C.Structure):
    _fields_ = [("n", i64), ("d", i32), ("components", i32), ("seed", u64), ("role", u64),
                ("kind", i32), ("center_scale", f64), ("center_lo", f64), ("center_hi", f64),
                ("sigma", f64), ("decay", i32), ("assign_mode", i32), ("threads", i32)]


class DcoBatch(C.Structure):
    _fields_ = [("X", vp), ("n_rows", i64), ("dim", i32), ("Q", vp), ("nq", i32),
                ("cand_off", vp), ("cand_rows", vp), ("win_start", vp), ("win_len", i64),
                ("r", vp), ("kind", i32), ("epsilon0", f64), ("delta_d", i32),
                ("positive", vp), ("dims", vp), ("dist_sq", vp), ("observed", vp),
                ("dims_per_query", vp)]


class IvfDesc(C.Structure):
    _fields_ = [("n", i32), ("d", i32), ("k_clusters", i32), ("d1", i32), ("layout", i32),
                ("seed", u64), ("centroids_t", vp), ("centroids_raw", vp), ("list_off", vp),
                ("ids_flat", vp), ("vec_t", vp), ("vec_raw", vp), ("a1_t", vp), ("a2_t", vp),
                ("a1_raw", vp), ("a2_raw", vp), ("P", vp)]


class SearchOpts(C.Structure):
    _fields_ = [("first", i64), ("step", i64), ("warps_per_cta", i32), ("queries_per_cta", i32),
                ("ctas_per_sm", i32), ("time_stages", i32), ("scheduler", i32), ("tile", i32),
                ("query_order", i32), ("coarse_mode", i32), ("rotate_mode", i32),
                ("probe_lo", i32), ("r0", vp), ("walk", i32), ("lag", i32)]


def _sig(name, args, res=C.c_int):
    f = getattr(lib, name)
    f.argtypes = args
    f.restype = res
    return f


ads_last_error = _sig("ads_last_error", [], C.c_char_p)
ads_version = _sig("ads_version", [])
ads_device_count = _sig("ads_device_count", [pi32])
ads_rng_draw = _sig("ads_rng_draw", [u64, u64, i32, i32, u64, i64, vp])
ads_generate_orthogonal = _sig("ads_generate_orthogonal", [i32, u64, vp])
ads_threshold_multiplier = _sig("ads_threshold_multiplier", [i32, f64, pf64])
ads_ad_context = _sig("ads_ad_context", [f64, i32, i32, vp])
ads_synth = _sig("ads_synth", [C.POINTER(SynthDesc), vp, vp])
ads_synth_rows = _sig("ads_synth_rows", [C.POINTER(SynthDesc), i64, i64, i64, vp, vp])
ads_ctx_create = _sig("ads_ctx_create", [i32, C.POINTER(vp)])
ads_ctx_destroy = _sig("ads_ctx_destroy", [vp])
ads_ctx_sync = _sig("ads_ctx_sync", [vp])
ads_ctx_stream = _sig("ads_ctx_stream", [vp, C.POINTER(vp)])
ads_dev_alloc = _sig("ads_dev_alloc", [vp, i64, C.POINTER(vp)])
ads_dev_free = _sig("ads_dev_free", [vp, vp])
ads_memcpy_h2d = _sig("ads_memcpy_h2d", [vp, vp, vp, i64])
ads_memcpy_d2h = _sig("ads_memcpy_d2h", [vp, vp, vp, i64])
ads_memset_device = _sig("ads_memset_device", [vp, vp, i32, i64])
ads_host_alloc_pinned = _sig("ads_host_alloc_pinned", [i64, C.POINTER(vp)])
ads_host_free_pinned = _sig("ads_host_free_pinned", [vp])
ads_timer_start = _sig("ads_timer_start", [vp])
ads_timer_stop = _sig("ads_timer_stop", [vp, C.POINTER(C.c_float)])
ads_flush_l2 = _sig("ads_flush_l2", [vp])
ads_transform_create = _sig("ads_transform_create", [vp, vp, i32, C.POINTER(vp)])
ads_transform_destroy = _sig("ads_transform_destroy", [vp])
ads_apply_dataset = _sig("ads_apply_dataset", [vp, vp, i64, vp])
ads_apply_dataset_device = _sig("ads_apply_dataset_device", [vp, vp, i64, vp])
ads_apply_dataset_tc = _sig("ads_apply_dataset_tc", [vp, vp, i64, vp])
ads_apply_dataset_tc_device = _sig("ads_apply_dataset_tc_device", [vp, vp, i64, vp])
ads_apply_transpose = _sig("ads_apply_transpose", [vp, vp, i64, vp])
ads_apply_transpose_device = _sig("ads_apply_transpose_device", [vp, vp, i64, vp])
ads_dco_fixed = _sig("ads_dco_fixed", [vp, C.POINTER(DcoBatch)])
ads_dco_fixed_device = _sig("ads_dco_fixed_device", [vp, C.POINTER(DcoBatch)])
ads_dco = _sig("ads_dco", [vp, i32, vp, i32, vp, i32, f64, f64, i32, pi32, pf64, pf64, pi32])
ads_brute_force_knn = _sig("ads_brute_force_knn", [vp, vp, i64, i32, vp, i32, i32, vp])
ads_verify_theory = _sig("ads_verify_theory", [vp, vp, i64, i32, vp, i32, i32, vp, i32, vp, vp, vp, vp, vp])
ads_brute_force_knn_device = _sig("ads_brute_force_knn_device", [vp, vp, i64, i32, vp, i32, i32, vp])
ads_kmeans = _sig("ads_kmeans", [vp, vp, i64, i32, i32, i32, u64, i32, vp, vp, pf64, pi32])
ads_ivf_create = _sig("ads_ivf_create", [vp, C.POINTER(IvfDesc), C.POINTER(vp)])
ads_ivf_build = _sig("ads_ivf_build", [vp, vp, vp, i32, i32, vp, i32, u64, i32, i32, i32, i32,
                                       C.POINTER(vp)])
ads_ivf_destroy = _sig("ads_ivf_destroy", [vp])
ads_ivf_meta = _sig("ads_ivf_meta", [vp, vp])
ads_ivf_save = _sig("ads_ivf_save", [vp, C.c_char_p])
ads_ivf_load = _sig("ads_ivf_load", [vp, C.c_char_p, vp, C.POINTER(vp)])
ads_ivf_export = _sig("ads_ivf_export", [vp] * 9)
ads_search_opts_default = _sig("ads_search_opts_default", [C.POINTER(SearchOpts)], None)
ads_ivf_search = _sig("ads_ivf_search", [vp, vp, vp, i32, i32, i32, i32, f64, i32,
                                         C.POINTER(SearchOpts), vp, vp, vp, vp, vp])
ads_ivf_search_device = _sig("ads_ivf_search_device", [vp, vp, vp, i32, i32, i32, i32, f64, i32,
                                                       C.POINTER(SearchOpts), vp, vp, vp, vp, vp])
ads_ivf_search_plan = _sig("ads_ivf_search_plan", [vp, i32, i32, i32, f64, i32, C.POINTER(SearchOpts),
                                                   vp, vp, vp, vp, vp, vp])
ads_ivf_probe_order = _sig("ads_ivf_probe_order", [vp, vp, i32, i32, i32, vp])
ads_ivf_last_timings = _sig("ads_ivf_last_timings", [vp, vp])
ads_ivf_coarse_stats = _sig("ads_ivf_coarse_stats", [vp, vp])
ads_ivf_build_sampled_device = _sig("ads_ivf_build_sampled_device", [vp, vp, i64, i32, vp, i32, u64, i32, i32, i64, C.POINTER(vp)])
ads_ivf_builder_create = _sig("ads_ivf_builder_create", [vp, i64, i32, vp, i32, u64, i32, C.POINTER(vp)])
ads_ivf_builder_train_device = _sig("ads_ivf_builder_train_device", [vp, vp, i64, i32])
ads_ivf_builder_set_centroids = _sig("ads_ivf_builder_set_centroids", [vp, vp])
ads_ivf_builder_centroids = _sig("ads_ivf_builder_centroids", [vp, vp])
ads_ivf_builder_add_device = _sig("ads_ivf_builder_add_device", [vp, vp, i64, i64])
ads_ivf_builder_rows_device = _sig("ads_ivf_builder_rows_device", [vp, C.POINTER(vp)])
ads_ivf_builder_list_sizes = _sig("ads_ivf_builder_list_sizes", [vp, vp])
ads_ivf_builder_finish = _sig("ads_ivf_builder_finish", [vp, vp, C.POINTER(vp)])
ads_ivf_builder_destroy = _sig("ads_ivf_builder_destroy", [vp])
ads_ivf_subset = _sig("ads_ivf_subset", [vp, vp, C.POINTER(vp)])
ads_merge_topk = _sig("ads_merge_topk", [vp, vp, vp, i32, i32, i32, vp, vp, vp])
ads_merge_topk_device = _sig("ads_merge_topk_device", [vp, vp, vp, i32, i32, i32, vp, vp, vp])


def check(rc: int) -> None:
    """Map ads_status to the reference's exception classes."""
    if rc == 0:
        return
    msg = ads_last_error().decode(errors="replace")
    if rc == 1:  # std::invalid_argument
        raise ValueError(msg)
    raise RuntimeError(msg)


def exported_symbols_from_header(path: str = HEADER) -> list[str]:
    import re

    text = open(path).read()
    return sorted(set(re.findall(r"\b(ads_[a-z0-9_]+)\s*\(", text)))

"""IVF-list sharding across GPUs (BASELINE config 5).

Each rank holds the lists it owns (rows of the other lists are dropped, the
centroids and P stay global, so every rank computes the same probe order), scans
the global probe-ordered candidate stream restricted to its lists, and produces
its own top-K per query.  The per-rank (dist, id) lists are all-gathered over
NCCL and merged on the GPU into the K smallest (dist, id) pairs per query.

Host orchestration only; the search, the sub-index gather and the merge are
kernels in libadsann_b200.so.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from ._lib import check
from .api import Context, IvfIndex


def partition_lists(list_sizes, world: int) -> np.ndarray:
    """Owner rank per list: longest-processing-time bin packing on list sizes
    (largest list first, ties by list id; to the least-loaded rank, ties by rank).
    Deterministic, so every rank computes the same partition."""
    sizes = np.asarray(list_sizes, dtype=np.int64)
    if world < 1:
        raise ValueError("partition_lists: world must be >= 1")
    order = np.lexsort((np.arange(len(sizes)), -sizes))
    load = np.zeros(world, dtype=np.int64)
    owner = np.empty(len(sizes), dtype=np.int32)
    for c in order:
        r = int(np.argmin(load))  # first minimum -> lowest rank on ties
        owner[c] = r
        load[r] += sizes[c]
    return owner


def shard_index(index: IvfIndex, owner: np.ndarray, rank: int) -> IvfIndex:
    """The rank's shard (ads_ivf_subset): owned lists keep their rows."""
    keep = np.ascontiguousarray(owner == rank, dtype=np.uint8)
    if keep.shape[0] != index.k_clusters:
        raise ValueError("shard_index: owner array must have one entry per list")
    h = C.c_void_p()
    check(L.ads_ivf_subset(index.h, keep.ctypes.data, C.byref(h)))
    return IvfIndex(h, index.ctx)


def merge_topk(dists: np.ndarray, ids: np.ndarray, K: int, ctx: Context | None = None):
    """[G, nq, K] per-shard results -> (ids, dists, counts): K smallest (dist, id)."""
    ctx = ctx or Context.default()
    dists = np.ascontiguousarray(dists, np.float64)
    ids = np.ascontiguousarray(ids, np.int32)
    G, nq, k2 = dists.shape
    if k2 != K or ids.shape != dists.shape:
        raise ValueError("merge_topk: shapes must be [G, nq, K]")
    oi = np.empty((nq, K), np.int32)
    od = np.empty((nq, K), np.float64)
    oc = np.empty(nq, np.int32)
    check(L.ads_merge_topk(ctx.h, dists.ctypes.data, ids.ctypes.data, G, nq, K, oi.ctypes.data,
                           od.ctypes.data, oc.ctypes.data))
    return oi, od, oc


def merge_topk_device(ctx: Context, ddists: int, dids: int, G: int, nq: int, K: int,
                      dout_ids: int, dout_dists: int, dout_counts: int) -> None:
    check(L.ads_merge_topk_device(ctx.h, C.c_void_p(ddists), C.c_void_p(dids), G, nq, K,
                                  C.c_void_p(dout_ids), C.c_void_p(dout_dists),
                                  C.c_void_p(dout_counts)))

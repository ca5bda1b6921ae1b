"""Host-side mirror of the reference's ``adsann`` API for the IVF++ path.

Same names, argument meaning and error behaviour as the reference headers
(include/adsann/{dco,transform,ivf,bench,result}.hpp); ValueError stands for
std::invalid_argument and RuntimeError for std::runtime_error.  Every
numeric step runs in libadsann_b200.so on the GPU (sm_100a); Python only
marshals arrays.  Batched forms (``ivf_query_batch``, ``dco_fixed``) are the
throughput entry points; the single-item forms wrap them.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import threading
from dataclasses import dataclass, field
from typing import NamedTuple, Optional, Sequence

import numpy as np

from . import _lib as L
from ._lib import check

# ---------------------------------------------------------------- types (dco.hpp, ivf.hpp, result.hpp)


@dataclass
class DcoConfig:  # dco.hpp:28-31
    epsilon0: float = 2.1
    delta_d: int = 32


@dataclass
class DcoOutcome:  # dco.hpp:37-42
    positive: bool = False
    distance: Optional[float] = None
    observed: float = 0.0
    dims_used: int = 0


class IvfLayout(enum.IntEnum):  # ivf.hpp:41
    kContiguous = 0
    kSplit = 1


class IvfMode(enum.IntEnum):  # ivf.hpp:43-49
    kFd = 0
    kPd = 1
    kAd = 2
    kAdSplit = 3
    kPdSplit = 4


MODE_NAMES = {"fd": IvfMode.kFd, "pd": IvfMode.kPd, "ad": IvfMode.kAd,
              "ad-split": IvfMode.kAdSplit, "pd-split": IvfMode.kPdSplit}  # ivf.cpp:503-521
ALGO_LABELS = {IvfMode.kFd: "IVF", IvfMode.kPd: "IVF*", IvfMode.kPdSplit: "IVF**",
               IvfMode.kAd: "IVF+", IvfMode.kAdSplit: "IVF++"}  # bench.cpp:186-195


def ivf_mode_from_name(name: str) -> IvfMode:
    if name not in MODE_NAMES:
        raise ValueError(f"unknown IVF mode: {name}")
    return MODE_NAMES[name]


def ivf_mode_name(mode: IvfMode) -> str:
    return {v: k for k, v in MODE_NAMES.items()}[IvfMode(mode)]


@dataclass
class QueryStats:  # result.hpp:24-30
    dims_evaluated: int = 0
    dco_count: int = 0
    candidates: int = 0
    hops: int = 0
    seconds: float = 0.0


@dataclass
class KnnResult:  # result.hpp:33-37
    ids: np.ndarray = field(default_factory=lambda: np.empty(0, np.int32))
    dists: np.ndarray = field(default_factory=lambda: np.empty(0, np.float64))
    stats: QueryStats = field(default_factory=QueryStats)


@dataclass
class TransformMatrix:  # transform.hpp:32-40
    dim: int
    seed: int
    entries: np.ndarray  # dim x dim float64, row-major

    def row(self, i: int) -> np.ndarray:
        return self.entries[i]


@dataclass
class KmeansResult:  # ivf.hpp:28-33
    centroids: np.ndarray
    assignment: np.ndarray
    objective: float
    iterations: int


# ---------------------------------------------------------------- device context


def _ptr(a) -> Optional[int]:
    return None if a is None else a.ctypes.data


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


class Context:
    """One CUDA device + stream (ads_ctx)."""

    _default: dict = {}
    _lock = threading.Lock()

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(L.ads_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        with cls._lock:
            if device not in cls._default:
                cls._default[device] = Context(device)
            return cls._default[device]

    def sync(self):
        check(L.ads_ctx_sync(self.h))

    def stream_handle(self) -> int:
        """cudaStream_t of this context (e.g. for torch.cuda.ExternalStream)."""
        p = C.c_void_p()
        check(L.ads_ctx_stream(self.h, C.byref(p)))
        return p.value or 0

    def timer_start(self):
        check(L.ads_timer_start(self.h))

    def timer_stop(self) -> float:
        ms = C.c_float()
        check(L.ads_timer_stop(self.h, C.byref(ms)))
        return ms.value

    def flush_l2(self):
        check(L.ads_flush_l2(self.h))


def device_count() -> int:
    n = C.c_int32()
    check(L.ads_device_count(C.byref(n)))
    return n.value


class DeviceArray:
    """A device allocation owned by Python (for HBM-resident inputs)."""

    def __init__(self, ctx: Context, shape, dtype):
        self.ctx = ctx
        self.shape = tuple(shape)
        self.dtype = np.dtype(dtype)
        self.nbytes = int(np.prod(self.shape)) * self.dtype.itemsize
        p = C.c_void_p()
        check(L.ads_dev_alloc(ctx.h, self.nbytes, C.byref(p)))
        self.ptr = p.value

    @classmethod
    def from_host(cls, ctx: Context, a: np.ndarray) -> "DeviceArray":
        a = np.ascontiguousarray(a)
        d = cls(ctx, a.shape, a.dtype)
        check(L.ads_memcpy_h2d(ctx.h, d.ptr, a.ctypes.data, a.nbytes))
        return d

    def to_host(self) -> np.ndarray:
        out = np.empty(self.shape, self.dtype)
        check(L.ads_memcpy_d2h(self.ctx.h, out.ctypes.data, self.ptr, self.nbytes))
        return out

    def free(self):
        if self.ptr:
            L.ads_dev_free(self.ctx.h, self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class PinnedArray:
    """Page-locked host buffer viewed as a numpy array (end-to-end path)."""

    def __init__(self, shape, dtype):
        self.dtype = np.dtype(dtype)
        nbytes = int(np.prod(shape)) * self.dtype.itemsize
        p = C.c_void_p()
        check(L.ads_host_alloc_pinned(nbytes, C.byref(p)))
        self.ptr = p.value
        buf = (C.c_char * max(nbytes, 1)).from_address(self.ptr)
        self.array = np.frombuffer(buf, dtype=self.dtype, count=int(np.prod(shape))).reshape(shape)

    def __del__(self):
        try:
            L.ads_host_free_pinned(self.ptr)
        except Exception:
            pass


# ---------------------------------------------------------------- host-side pieces


def rng_draw(seed: int, tag: int, kind: int, count: int, use_stream: bool = True, arg: int = 0):
    """rng.hpp:36-97 draws (kind 0 u64, 1 uniform, 2 normal, 3 below(arg))."""
    out = np.empty(count, np.uint64 if kind in (0, 3) else np.float64)
    check(L.ads_rng_draw(seed, tag, int(use_stream), kind, arg, count, out.ctypes.data))
    return out


def generate_orthogonal(dim: int, seed: int) -> TransformMatrix:  # transform.hpp:45
    P = np.empty((max(dim, 1), max(dim, 1)), np.float64)
    check(L.ads_generate_orthogonal(dim, seed, P.ctypes.data))
    return TransformMatrix(dim, seed, P)


def threshold_multiplier(d: int, cfg: DcoConfig) -> float:  # dco.hpp:67
    out = C.c_double()
    check(L.ads_threshold_multiplier(d, cfg.epsilon0, C.byref(out)))
    return out.value


def ad_context_factor(cfg: DcoConfig, dim: int) -> np.ndarray:  # AdContext, dco.hpp:101-108
    f = np.zeros(max(dim, 1), np.float64)
    check(L.ads_ad_context(cfg.epsilon0, cfg.delta_d, dim, f.ctypes.data))
    return f


def synth(n: int, d: int, components: int, seed: int, role: int, kind: int = 0,
          center_scale: float = 1.0, center_lo: float = 0.0, center_hi: float = 1.0,
          sigma: float = 1.0, decay: bool = False, assign_mode: int = 0, threads: int = 0,
          with_components: bool = False):
    """Seeded Gaussian mixture.  Host, multi-threaded, deterministic."""
    desc = L.SynthDesc(n, d, components, seed, role, kind, center_scale, center_lo, center_hi,
                       sigma, int(decay), assign_mode, threads)
    out = np.empty((n, d), np.float32)
    comp = np.empty(n, np.int32) if with_components else None
    check(L.ads_synth(C.byref(desc), out.ctypes.data, _ptr(comp)))
    return (out, comp) if with_components else out


def synth_rows(n: int, d: int, components: int, seed: int, role: int, row_lo: int, count: int,
               stride: int = 1, out: Optional[np.ndarray] = None, kind: int = 0,
               center_scale: float = 1.0, center_lo: float = 0.0, center_hi: float = 1.0,
               sigma: float = 1.0, decay: bool = False, assign_mode: int = 0,
               threads: int = 0) -> np.ndarray:
    """Rows row_lo + i*stride (i < count) of synth(n, ...), bit-identical to them."""
    desc = L.SynthDesc(n, d, components, seed, role, kind, center_scale, center_lo, center_hi,
                       sigma, int(decay), assign_mode, threads)
    if out is None:
        out = np.empty((count, d), np.float32)
    if out.dtype != np.float32 or not out.flags.c_contiguous or out.size < count * d:
        raise ValueError("synth_rows: out must be a contiguous float32 array of count x d")
    check(L.ads_synth_rows(C.byref(desc), row_lo, count, stride, out.ctypes.data, None))
    return out


# ---------------------------------------------------------------- transform (GPU)


class Transform:
    """P resident on the device (ads_transform)."""

    def __init__(self, m: TransformMatrix, ctx: Optional[Context] = None):
        self.ctx = ctx or Context.default()
        self.m = m
        P = np.ascontiguousarray(m.entries, np.float64)
        h = C.c_void_p()
        check(L.ads_transform_create(self.ctx.h, P.ctypes.data, m.dim, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            L.ads_transform_destroy(self.h)
        except Exception:
            pass

    def apply_dataset(self, X: np.ndarray) -> np.ndarray:
        X = _f32(X)
        if X.ndim != 2 or X.shape[1] != self.m.dim:
            raise ValueError("apply_dataset: dataset dimension does not match matrix")
        Y = np.empty_like(X)
        check(L.ads_apply_dataset(self.h, X.ctypes.data, X.shape[0], Y.ctypes.data))
        return Y

    def apply_transpose_dataset(self, X: np.ndarray) -> np.ndarray:
        X = _f32(X)
        Y = np.empty_like(X)
        check(L.ads_apply_transpose(self.h, X.ctypes.data, X.shape[0], Y.ctypes.data))
        return Y

    def apply_dataset_tc(self, X: np.ndarray) -> np.ndarray:
        """The rotation on the tensor cores (3xTF32); not bit-identical to apply_dataset."""
        X = _f32(X)
        if X.ndim != 2 or X.shape[1] != self.m.dim:
            raise ValueError("apply_dataset: dataset dimension does not match matrix")
        Y = np.empty_like(X)
        check(L.ads_apply_dataset_tc(self.h, X.ctypes.data, X.shape[0], Y.ctypes.data))
        return Y

    def apply_dataset_tc_device(self, dX: "DeviceArray", dY: "DeviceArray") -> None:
        check(L.ads_apply_dataset_tc_device(self.h, C.c_void_p(dX.ptr), dX.shape[0], C.c_void_p(dY.ptr)))

    def apply_dataset_device(self, dX: "DeviceArray", dY: "DeviceArray") -> None:
        check(L.ads_apply_dataset_device(self.h, C.c_void_p(dX.ptr), dX.shape[0], C.c_void_p(dY.ptr)))


_TCACHE: dict = {}
_TCACHE_LOCK = threading.Lock()


def _transform_for(m: TransformMatrix, ctx=None) -> Transform:
    """The device transform of the most recently used matrix (uploading P once); the
    cache keeps a reference to m.entries, so its id cannot be reused while cached."""
    key = (id(m.entries), m.dim, (ctx or Context.default()).device)
    with _TCACHE_LOCK:
        t = _TCACHE.get(key)
        if t is None or t.m.entries is not m.entries:
            t = Transform(m, ctx)
            _TCACHE.clear()
            _TCACHE[key] = t
        return t


def apply_dataset(m: TransformMatrix, ds: np.ndarray) -> np.ndarray:  # transform.hpp:58
    ds = _f32(ds)
    if ds.ndim != 2 or ds.shape[1] != m.dim:
        raise ValueError("apply_dataset: dataset dimension does not match matrix")
    return _transform_for(m).apply_dataset(ds)


def apply_dataset_tc(m: TransformMatrix, ds: np.ndarray) -> np.ndarray:
    """apply_dataset on the tensor cores (tcgen05 3xTF32); fp32-accurate, not bit-exact."""
    return _transform_for(m).apply_dataset_tc(ds)


def apply(m: TransformMatrix, x) -> np.ndarray:  # transform.hpp:48
    x = _f32(x)
    if x.shape != (m.dim,):
        raise ValueError("apply: vector length does not match matrix dim")
    return apply_dataset(m, x[None, :])[0]


def apply_prefix(m: TransformMatrix, x, d: int) -> np.ndarray:  # transform.hpp:52
    if d < 0 or d > m.dim:
        raise ValueError("apply_prefix: d out of range")
    return apply(m, x)[:d].copy()


def apply_transpose(m: TransformMatrix, x) -> np.ndarray:  # transform.hpp:55
    x = _f32(x)
    if x.shape != (m.dim,):
        raise ValueError("apply_transpose: vector length does not match matrix dim")
    return _transform_for(m).apply_transpose_dataset(x[None, :])[0]


# ---------------------------------------------------------------- DCOs (GPU)

_KIND = {"fd": 0, "pd": 1, "ad": 2}


def _dco_single(kind: int, o, q, r: float, eps0: float, dd: int, ctx=None) -> DcoOutcome:
    ctx = ctx or Context.default()
    o = _f32(o)
    q = _f32(q)
    pos, dist, obs, dims = C.c_int32(), C.c_double(), C.c_double(), C.c_int32()
    check(L.ads_dco(ctx.h, kind, o.ctypes.data, len(o), q.ctypes.data, len(q), float(r), eps0, dd,
                    C.byref(pos), C.byref(dist), C.byref(obs), C.byref(dims)))
    return DcoOutcome(bool(pos.value), None if math.isnan(dist.value) else dist.value, obs.value,
                      dims.value)


def fd_scan(o, q, r: float) -> DcoOutcome:  # dco.hpp:69
    return _dco_single(0, o, q, r, 2.1, 1)


def pd_scan(o, q, r: float, delta_d: int) -> DcoOutcome:  # dco.hpp:70
    return _dco_single(1, o, q, r, 2.1, delta_d)


def ad_sampling(o, q, r: float, cfg: DcoConfig = DcoConfig()) -> DcoOutcome:  # dco.hpp:71
    return _dco_single(2, o, q, r, cfg.epsilon0, cfg.delta_d)


@dataclass
class DcoBatchResult:
    positive: np.ndarray
    dims: np.ndarray
    dist_sq: Optional[np.ndarray]
    observed: Optional[np.ndarray]
    dims_per_query: np.ndarray


def dco_fixed(X: np.ndarray, Q: np.ndarray, r: Sequence[float], *, cand_off=None, cand_rows=None,
              win_start=None, win_len: int = 0, kind: str = "ad", cfg: DcoConfig = DcoConfig(),
              want_dist: bool = True, ctx: Optional[Context] = None) -> DcoBatchResult:
    """Batched fixed-threshold DCOs (ads_dco_fixed): one ad_scan/pd_scan/l2_sq per pair."""
    ctx = ctx or Context.default()
    X = _f32(X)
    Q = _f32(Q)
    nq = Q.shape[0]
    r = np.ascontiguousarray(r, np.float64)
    if cand_rows is not None:
        cand_off = np.ascontiguousarray(cand_off, np.int64)
        cand_rows = np.ascontiguousarray(cand_rows, np.int64)
        total = int(cand_off[-1])
    else:
        win_start = np.ascontiguousarray(win_start, np.int64)
        total = nq * int(win_len)
    pos = np.empty(total, np.uint8)
    dims = np.empty(total, np.int32)
    dsq = np.empty(total, np.float64) if want_dist else None
    obs = np.empty(total, np.float64) if want_dist else None
    dpq = np.empty(nq, np.uint64)
    b = L.DcoBatch(X.ctypes.data, X.shape[0], X.shape[1], Q.ctypes.data, nq, _ptr(cand_off),
                   _ptr(cand_rows), _ptr(win_start), int(win_len), r.ctypes.data, _KIND[kind],
                   cfg.epsilon0, cfg.delta_d, pos.ctypes.data, dims.ctypes.data, _ptr(dsq),
                   _ptr(obs), dpq.ctypes.data)
    check(L.ads_dco_fixed(ctx.h, C.byref(b)))
    return DcoBatchResult(pos.astype(bool), dims, dsq, obs, dpq)


# ---------------------------------------------------------------- k-means / brute force (GPU)


def kmeans(ds: np.ndarray, k: int, max_iters: int, seed: int, init: int = 0,
           ctx: Optional[Context] = None) -> KmeansResult:  # ivf.hpp:39
    ctx = ctx or Context.default()
    ds = _f32(ds)
    n, d = ds.shape
    cent = np.empty((max(k, 1), d), np.float32)
    asg = np.empty(n, np.int32)
    obj, it = C.c_double(), C.c_int32()
    check(L.ads_kmeans(ctx.h, ds.ctypes.data, n, d, k, max_iters, seed, init, cent.ctypes.data,
                       asg.ctypes.data, C.byref(obj), C.byref(it)))
    return KmeansResult(cent, asg, obj.value, it.value)


def brute_force_knn(ds: np.ndarray, queries: np.ndarray, K: int,
                    ctx: Optional[Context] = None) -> np.ndarray:  # bench.hpp:34
    ctx = ctx or Context.default()
    ds = _f32(ds)
    queries = _f32(queries)
    if ds.shape[1] != queries.shape[1]:
        raise ValueError("brute_force_knn: dimensionality mismatch")
    ids = np.empty((queries.shape[0], max(K, 1)), np.int32)
    check(L.ads_brute_force_knn(ctx.h, ds.ctypes.data, ds.shape[0], ds.shape[1],
                                queries.ctypes.data, queries.shape[0], K, ids.ctypes.data))
    return ids


class TheoryRow(NamedTuple):  # bench.hpp:90-96
    epsilon0: float
    failure_rate: float
    avg_dims: float
    failures: int
    positives: int


def verify_theory(ds_t: np.ndarray, queries_t: np.ndarray, K: int, epsilon0_grid,
                  ctx: Optional[Context] = None) -> list:
    """bench.cpp:303-392 on the GPU: one delta_d = 1 comparison per (query, object)
    per epsilon0 against the exact K-th neighbour distance; rows sorted by epsilon0."""
    ctx = ctx or Context.default()
    ds_t = _f32(ds_t)
    queries_t = _f32(queries_t)
    if ds_t.shape[1] != queries_t.shape[1]:
        raise ValueError("verify_theory: dimensionality mismatch")
    grid = np.ascontiguousarray(list(epsilon0_grid), np.float64)
    G = len(grid)
    eps, fr, ad = np.empty(max(G, 1)), np.empty(max(G, 1)), np.empty(max(G, 1))
    fails, pos = np.empty(max(G, 1), np.uint64), np.empty(max(G, 1), np.uint64)
    check(L.ads_verify_theory(ctx.h, ds_t.ctypes.data, ds_t.shape[0], ds_t.shape[1],
                              queries_t.ctypes.data, queries_t.shape[0], K, grid.ctypes.data, G,
                              eps.ctypes.data, fr.ctypes.data, ad.ctypes.data, fails.ctypes.data,
                              pos.ctypes.data))
    return [TheoryRow(float(eps[g]), float(fr[g]), float(ad[g]), int(fails[g]), int(pos[g]))
            for g in range(G)]


def recall(result_ids, gt_ids, K: int) -> float:  # bench.cpp:63-72 (set arithmetic)
    gt_ids = np.asarray(gt_ids)
    if len(gt_ids) < K:
        raise ValueError("recall: ground truth shorter than K")
    truth = set(int(v) for v in gt_ids[:K])
    return sum(1 for v in np.asarray(result_ids) if int(v) in truth) / float(K)


def recall_batch(ids: np.ndarray, gt: np.ndarray, K: int) -> float:
    """Mean recall@K over queries (vectorised recall())."""
    hits = 0
    for a, b in zip(ids, gt):
        hits += len(np.intersect1d(a[a >= 0], b[:K], assume_unique=False))
    return hits / float(K * len(ids))


# ---------------------------------------------------------------- IVF (GPU)


def search_plan(idx: "IvfIndex", K: int, n_probe: int, mode: "IvfMode", cfg: "DcoConfig" = None,
                opts: Optional[L.SearchOpts] = None) -> dict:
    """The scan schedule a search with these arguments uses (ads_ivf_search_plan): the
    threshold refresh schedule (first, step), warps_per_cta, walk (1 exact, 2 certified
    fp32), dense (the A1 prefix phase) and lag (1: overlapped chunks; the oracle replays it
    as lag = 2).  Results depend on (first, step, lag) only."""
    cfg = cfg or DcoConfig()
    o = opts or search_opts()
    first, step = C.c_int64(), C.c_int64()
    warps, walk, dense, lag = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
    check(L.ads_ivf_search_plan(idx.h, K, n_probe, int(mode), cfg.epsilon0, cfg.delta_d, C.byref(o),
                                C.byref(first), C.byref(step), C.byref(warps), C.byref(walk), C.byref(dense),
                                C.byref(lag)))
    return {"first": first.value, "step": step.value, "warps_per_cta": warps.value, "walk": walk.value,
            "dense": bool(dense.value), "lag": lag.value}


def search_opts(first: int = 0, step: int = 0, warps_per_cta: int = 0, queries_per_cta: int = 1,
                ctas_per_sm: int = 0, time_stages: bool = False, scheduler: int = 0,
                tile: int = 64, query_order: int = 2, coarse_mode: int = 0,
                rotate_mode: int = 2, probe_lo: int = 0, r0=None, walk: int = 0, lag: int = 0) -> L.SearchOpts:
    """Search options (ads_search_opts, include/adsann_b200.h): first/step set the
    threshold refresh schedule in candidates; scheduler must be 0."""
    o = L.SearchOpts()
    L.ads_search_opts_default(C.byref(o))
    o.first, o.step, o.warps_per_cta, o.queries_per_cta, o.ctas_per_sm, o.time_stages = (
        first, step, warps_per_cta, queries_per_cta, ctas_per_sm, int(time_stages))
    o.scheduler, o.tile, o.query_order, o.coarse_mode = scheduler, tile, query_order, coarse_mode
    o.rotate_mode = rotate_mode
    o.probe_lo = probe_lo
    o.walk = walk
    o.lag = lag
    if r0 is not None:  # per-query initial radii (host array for the host API)
        if isinstance(r0, DeviceArray):
            o.r0 = r0.ptr
        else:
            r0 = np.ascontiguousarray(r0, np.float64)
            o.r0 = r0.ctypes.data
        o._r0_keep = r0  # keep the buffer alive with the options
    return o


REFERENCE_SCHEDULE = dict(first=1, step=1)  # r re-read before every candidate (ivf.cpp:331, 391)


class IvfIndex:
    """Device-resident IVF index (ivf.hpp:55-74), owned through an ads_ivf handle."""

    def __init__(self, handle: C.c_void_p, ctx: Context):
        self.h = handle
        self.ctx = ctx
        meta = np.zeros(7, np.int64)
        check(L.ads_ivf_meta(self.h, meta.ctypes.data))
        self.n, self.d, self.k_clusters, self.d1 = (int(v) for v in meta[:4])
        self.layout = IvfLayout(int(meta[4]))
        self.seed = int(meta[5])
        self.has_raw = bool(meta[6])

    def __del__(self):
        try:
            if self.h:
                L.ads_ivf_destroy(self.h)
        except Exception:
            pass

    @classmethod
    def from_arrays(cls, *, n, d, k_clusters, d1, layout, centroids_t, list_off, ids_flat,
                    vec_t=None, a1_t=None, a2_t=None, centroids_raw=None, vec_raw=None,
                    a1_raw=None, a2_raw=None, P=None, seed=0, ctx: Optional[Context] = None):
        ctx = ctx or Context.default()
        keep = []

        def p(a, dt):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dt)
            keep.append(a)
            return a.ctypes.data

        desc = L.IvfDesc(n, d, k_clusters, d1, int(layout), seed, p(centroids_t, np.float32),
                         p(centroids_raw, np.float32), p(list_off, np.int64), p(ids_flat, np.int32),
                         p(vec_t, np.float32), p(vec_raw, np.float32), p(a1_t, np.float32),
                         p(a2_t, np.float32), p(a1_raw, np.float32), p(a2_raw, np.float32),
                         p(P, np.float64))
        h = C.c_void_p()
        check(L.ads_ivf_create(ctx.h, C.byref(desc), C.byref(h)))
        return cls(h, ctx)

    def export(self) -> dict:
        n, d, k = self.n, self.d, self.k_clusters
        d1p = self.d1 if self.layout == IvfLayout.kSplit else min(32, d)
        out = {"centroids_t": np.empty((k, d), np.float32),
               "list_off": np.empty(k + 1, np.int64), "ids_flat": np.empty(n, np.int32),
               "a1_t": np.empty((n, d1p), np.float32), "a2_t": np.empty((n, d - d1p), np.float32)}
        if self.has_raw:
            out.update(centroids_raw=np.empty((k, d), np.float32),
                       a1_raw=np.empty((n, d1p), np.float32),
                       a2_raw=np.empty((n, d - d1p), np.float32))
        g = lambda nm: _ptr(out.get(nm))
        check(L.ads_ivf_export(self.h, g("centroids_t"), g("centroids_raw"), g("list_off"),
                               g("ids_flat"), g("a1_t"), g("a2_t"), g("a1_raw"), g("a2_raw")))
        return out

    def list_offsets(self) -> np.ndarray:
        """list_off (k + 1) only, without copying the vectors back."""
        off = np.empty(self.k_clusters + 1, np.int64)
        check(L.ads_ivf_export(self.h, None, None, off.ctypes.data, None, None, None, None, None))
        return off

    def probe_order(self, Q: np.ndarray, nprobe: int, transformed: bool = True) -> np.ndarray:
        Q = _f32(Q)
        out = np.empty((Q.shape[0], nprobe), np.int32)
        check(L.ads_ivf_probe_order(self.h, Q.ctypes.data, Q.shape[0], nprobe, int(transformed),
                                    out.ctypes.data))
        return out

    def last_timings(self) -> np.ndarray:
        ms = np.zeros(4, np.float32)
        check(L.ads_ivf_last_timings(self.h, ms.ctypes.data))
        return ms

    def coarse_stats(self) -> dict:
        """Certified coarse prefilter counters of the last search / probe_order call."""
        v = np.zeros(3, np.uint64)
        check(L.ads_ivf_coarse_stats(self.h, v.ctypes.data))
        return {"queries": int(v[0]), "rescored": int(v[1]), "fallbacks": int(v[2])}


def save_ivf(idx: IvfIndex, path) -> None:  # ivf.hpp:91, ivf.cpp:423-440
    """The reference's on-disk index format (meta.txt + fvecs / ragged ivecs)."""
    check(L.ads_ivf_save(idx.h, str(path).encode()))


def load_ivf(path, m: Optional[TransformMatrix] = None, ctx: Optional[Context] = None) -> IvfIndex:
    """ivf.hpp:92, ivf.cpp:442-501.  m (optional) enables on-device query rotation."""
    ctx = ctx or Context.default()
    P = None if m is None else np.ascontiguousarray(m.entries, np.float64)
    h = C.c_void_p()
    check(L.ads_ivf_load(ctx.h, str(path).encode(), _ptr(P), C.byref(h)))
    return IvfIndex(h, ctx)


def build_ivf(ds_raw: np.ndarray, ds_transformed: np.ndarray, m: TransformMatrix, k_clusters: int,
              seed: int, layout: IvfLayout = IvfLayout.kContiguous, d1: int = 32,
              max_iters: int = 25, init: int = 0, ctx: Optional[Context] = None) -> IvfIndex:
    """ivf.hpp:76-78 on the GPU (k-means, buckets, centroids_raw, split arrays)."""
    ctx = ctx or Context.default()
    raw = _f32(ds_raw) if ds_raw is not None else None
    t = _f32(ds_transformed)
    if raw is not None and raw.shape != t.shape:
        raise ValueError("build_ivf: raw and transformed datasets disagree")
    n, d = t.shape
    if m.dim != d:
        raise ValueError("build_ivf: matrix dimension does not match the data")
    P = np.ascontiguousarray(m.entries, np.float64)
    h = C.c_void_p()
    check(L.ads_ivf_build(ctx.h, _ptr(raw), t.ctypes.data, n, d, P.ctypes.data, k_clusters, seed,
                          int(layout), d1, max_iters, init, C.byref(h)))
    return IvfIndex(h, ctx)


def build_ivf_sampled_device(dT: "DeviceArray", m: TransformMatrix, k_clusters: int, seed: int, d1: int = 32,
                             max_iters: int = 10, sample: int = 2_000_000,
                             ctx: Optional[Context] = None) -> IvfIndex:
    """build_ivf for device-resident data too large for the reference flow (config 5):
    k-means on every (n / sample)-th row, every row assigned by the certified
    coarse prefilter (exact argmin), split layout, transformed space only."""
    ctx = ctx or Context.default()
    n, d = dT.shape
    if m.dim != d:
        raise ValueError("build_ivf: matrix dimension does not match the data")
    P = np.ascontiguousarray(m.entries, np.float64)
    h = C.c_void_p()
    check(L.ads_ivf_build_sampled_device(ctx.h, C.c_void_p(dT.ptr), n, d, P.ctypes.data, k_clusters, seed, d1,
                                         max_iters, min(sample, n), C.byref(h)))
    return IvfIndex(h, ctx)


class IvfBuilder:
    """build_ivf fed in row chunks (ads_ivf_builder; ivf.cpp:192-258): k-means on a
    sample (or given centroids), every row assigned by the certified exact argmin,
    and the bucket layout of the lists a shard keeps."""

    def __init__(self, n: int, d: int, m: TransformMatrix, k_clusters: int, seed: int, d1: int = 32,
                 ctx: Optional[Context] = None):
        if m.dim != d:
            raise ValueError("build_ivf: matrix dimension does not match the data")
        self.ctx = ctx or Context.default()
        self.n, self.d, self.k_clusters = n, d, k_clusters
        P = np.ascontiguousarray(m.entries, np.float64)
        self.h = C.c_void_p()
        check(L.ads_ivf_builder_create(self.ctx.h, n, d, P.ctypes.data, k_clusters, seed, d1,
                                       C.byref(self.h)))

    def __del__(self):
        try:
            if self.h:
                L.ads_ivf_builder_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def close(self):
        self.__del__()

    def train_device(self, dS: "DeviceArray", max_iters: int) -> None:
        check(L.ads_ivf_builder_train_device(self.h, C.c_void_p(dS.ptr), dS.shape[0], max_iters))

    def set_centroids(self, centroids: np.ndarray) -> None:
        c = _f32(centroids)
        if c.shape != (self.k_clusters, self.d):
            raise ValueError("build_ivf: centroids must be k x d")
        check(L.ads_ivf_builder_set_centroids(self.h, c.ctypes.data))

    def centroids(self) -> np.ndarray:
        out = np.empty((self.k_clusters, self.d), np.float32)
        check(L.ads_ivf_builder_centroids(self.h, out.ctypes.data))
        return out

    def add_device(self, dT: "DeviceArray", row_lo: int, rows: Optional[int] = None) -> None:
        rows = dT.shape[0] if rows is None else rows
        check(L.ads_ivf_builder_add_device(self.h, C.c_void_p(dT.ptr), row_lo, rows))

    def rows_device(self) -> int:
        """Device pointer of the staged transformed rows (n x d by id), valid until close()."""
        p = C.c_void_p()
        check(L.ads_ivf_builder_rows_device(self.h, C.byref(p)))
        return p.value

    def list_sizes(self) -> np.ndarray:
        out = np.empty(self.k_clusters, np.int64)
        check(L.ads_ivf_builder_list_sizes(self.h, out.ctypes.data))
        return out

    def finish(self, keep: Optional[np.ndarray] = None) -> IvfIndex:
        h = C.c_void_p()
        kp = None if keep is None else np.ascontiguousarray(keep, np.uint8)
        if kp is not None and kp.shape != (self.k_clusters,):
            raise ValueError("build_ivf: keep must have one entry per list")
        check(L.ads_ivf_builder_finish(self.h, _ptr(kp), C.byref(h)))
        return IvfIndex(h, self.ctx)


def build_ivf_streamed(rows, n: int, d: int, m: TransformMatrix, k_clusters: int, seed: int,
                       d1: int = 32, max_iters: int = 10, sample: int = 2_000_000, chunk: int = 4_000_000,
                       owner=None, rank: int = 0, centroids: Optional[np.ndarray] = None,
                       on_rows=None, ctx: Optional[Context] = None):
    """build_ivf over raw rows produced piecewise by rows(row_lo, count, stride) -> float32
    (count x d host array): the sample rows (every n // sample-th) are rotated on the device
    and clustered (or `centroids` are used), then every chunk is generated on a host thread
    while the previous one is rotated (exact fp64 apply) and assigned on the GPU.  owner:
    callable(list_sizes) -> owner rank per list (list sharding; None keeps every list).
    on_rows(ptr): called with the device pointer of all n transformed rows (by id) before
    they are released (e.g. for an exact ground truth).  Returns (index, list_sizes,
    centroids)."""
    import threading as _th

    ctx = ctx or Context.default()
    tr = Transform(m, ctx)
    b = IvfBuilder(n, d, m, k_clusters, seed, d1, ctx)
    try:
        if centroids is None:
            sample = min(sample, n)
            stride = n // sample
            xs = rows(0, sample, stride)
            dS = DeviceArray.from_host(ctx, xs)
            dSt = DeviceArray(ctx, (sample, d), np.float32)
            tr.apply_dataset_device(dS, dSt)
            del xs
            dS.free()
            b.train_device(dSt, max_iters)
            dSt.free()
        else:
            b.set_centroids(centroids)
        chunk = max(1, min(chunk, n))
        dX = DeviceArray(ctx, (chunk, d), np.float32)
        dY = DeviceArray(ctx, (chunk, d), np.float32)
        nxt = {}

        def produce(lo):
            nxt[lo] = rows(lo, min(chunk, n - lo), 1)

        th = _th.Thread(target=produce, args=(0,))
        th.start()
        for lo in range(0, n, chunk):
            th.join()
            host = nxt.pop(lo)
            if lo + chunk < n:
                th = _th.Thread(target=produce, args=(lo + chunk,))
                th.start()
            cnt = host.shape[0]
            check(L.ads_memcpy_h2d(ctx.h, C.c_void_p(dX.ptr), host.ctypes.data, host.nbytes))
            check(L.ads_apply_dataset_device(tr.h, C.c_void_p(dX.ptr), cnt, C.c_void_p(dY.ptr)))
            b.add_device(dY, lo, cnt)
        ctx.sync()
        dX.free()
        dY.free()
        sizes = b.list_sizes()
        if on_rows is not None:
            on_rows(b.rows_device())
        keep = None
        if owner is not None:
            keep = (np.asarray(owner(sizes)) == rank).astype(np.uint8)
        cent = b.centroids()
        return b.finish(keep), sizes, cent
    finally:
        b.close()


@dataclass
class BatchResult:
    ids: np.ndarray      # nq x K int32 (-1 padded)
    dists: np.ndarray    # nq x K float64 (NaN padded)
    counts: np.ndarray   # nq
    dims: np.ndarray     # nq dims_evaluated
    candidates: np.ndarray

    def result(self, i: int, seconds: float = 0.0) -> KnnResult:
        c = int(self.counts[i])
        return KnnResult(self.ids[i, :c].copy(), self.dists[i, :c].copy(),
                         QueryStats(int(self.dims[i]), int(self.candidates[i]),
                                    int(self.candidates[i]), 0, seconds))


def ivf_query_batch(idx: IvfIndex, Q_t, Q_raw, K: int, n_probe: int, mode: IvfMode,
                    cfg: DcoConfig = DcoConfig(), first: int = 0, step: int = 0,
                    warps_per_cta: int = 0, opts: Optional[L.SearchOpts] = None) -> BatchResult:
    """Batched ivf_query (ivf.hpp:87-89).  first/step set the threshold refresh
    schedule; first=step=1 reproduces the reference's per-candidate refresh."""
    Qt = None if Q_t is None else _f32(np.atleast_2d(Q_t))
    Qr = None if Q_raw is None else _f32(np.atleast_2d(Q_raw))
    nq = (Qt if Qt is not None else Qr).shape[0] if (Qt is not None or Qr is not None) else 0
    Kc = max(K, 1)
    ids = np.empty((nq, Kc), np.int32)
    dists = np.empty((nq, Kc), np.float64)
    counts = np.empty(nq, np.int32)
    dims = np.empty(nq, np.uint64)
    cands = np.empty(nq, np.uint64)
    o = opts or search_opts(first, step, warps_per_cta)
    check(L.ads_ivf_search(idx.h, _ptr(Qt), _ptr(Qr), nq, K, n_probe, int(mode), cfg.epsilon0,
                           cfg.delta_d, C.byref(o), ids.ctypes.data, dists.ctypes.data,
                           counts.ctypes.data, dims.ctypes.data, cands.ctypes.data))
    return BatchResult(ids, dists, counts, dims, cands)


def ivf_query(idx: IvfIndex, q_transformed, q_raw, K: int, n_probe: int, mode: IvfMode,
              cfg: DcoConfig = DcoConfig(), first: int = 1, step: int = 1) -> KnnResult:
    """ivf_query (ivf.hpp:87-89).  The single-query form defaults to the
    reference's per-candidate threshold refresh, so it returns exactly what
    adsann::ivf_query returns."""
    r = ivf_query_batch(idx, q_transformed, q_raw, K, n_probe, mode, cfg, first, step)
    return r.result(0)

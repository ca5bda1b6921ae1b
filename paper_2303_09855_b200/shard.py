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


def first_wave(nprobe: int, world: int, waves: int = -1) -> int:
    """Probe ranks of the first wave of the threshold exchange: nprobe / 8 when
    world > 1 (waves = -1), `waves` when given; 0 = one wave (no exchange)."""
    w = waves if waves >= 0 else (max(1, nprobe // 8) if world > 1 else 0)
    return w if 0 < w < nprobe else 0


class DeviceShardSearch:
    """Per-rank search and merge on the GPU (libadsann_b200.so) for ShardedIvf."""

    def __init__(self, local: IvfIndex, K: int, mode=None, eps0: float = 2.1, delta_d: int = 32,
                 step: int = 0, warps: int = 0, time_stages: bool = False, P=None):
        from . import api

        self.local, self.K = local, K
        self.local_P, self.transform = P, None
        self.mode = int(api.IvfMode.kAdSplit if mode is None else mode)
        self.eps0, self.dd = eps0, delta_d
        self.opts = [api.search_opts(first=0, step=step, warps_per_cta=warps, time_stages=time_stages),
                     api.search_opts(first=0, step=step, warps_per_cta=warps, time_stages=time_stages)]
        self.device = local.ctx.device

    def search(self, dq, nq, nprobe, probe_lo, r0, out):
        """One wave over probe ranks [probe_lo, nprobe) into out = (ids, dists, cnt, dims, cand)."""
        o = self.opts[1 if probe_lo else 0]
        o.probe_lo = probe_lo
        o.r0 = None if r0 is None else r0.data_ptr()
        ids, dists, cnt, dims, cand = out
        check(L.ads_ivf_search_device(self.local.h, C.c_void_p(dq.data_ptr()), None, nq, self.K, nprobe,
                                      self.mode, self.eps0, self.dd, C.byref(o), C.c_void_p(ids.data_ptr()),
                                      C.c_void_p(dists.data_ptr()), C.c_void_p(cnt.data_ptr()),
                                      C.c_void_p(dims.data_ptr()), C.c_void_p(cand.data_ptr())))

    def rotate(self, dq_raw, dq_t, nq):
        """Exact fp64 query rotation (apply, transform.cpp:99) on the engine stream."""
        if self.transform is None:
            from . import api

            P = np.ascontiguousarray(self.local_P, np.float64)
            self.transform = api.Transform(api.TransformMatrix(P.shape[0], 0, P), self.local.ctx)
        check(L.ads_apply_dataset_device(self.transform.h, C.c_void_p(dq_raw.data_ptr()), nq,
                                         C.c_void_p(dq_t.data_ptr())))

    def merge(self, gd, gi, G, nq, oi, od, oc):
        merge_topk_device(self.local.ctx, gd.data_ptr(), gi.data_ptr(), G, nq, self.K, oi.data_ptr(),
                          od.data_ptr(), oc.data_ptr())


class ShardedIvf:
    """List-sharded IVF++ search, one process per GPU (BASELINE config 5).

    Every rank holds the lists it owns (partition_lists + shard_index or
    IvfBuilder.finish(keep)) and all the centroids, and answers the SAME query
    batch (strong scaling: the job's Q is fixed).  One step:

    1. wave 1: each rank scans probe ranks [0, w) over its own lists;
    2. all-reduce (min) of every query's local K-th distance: an upper bound on
       the global K-th distance (+inf where a rank holds fewer than K);
    3. wave 2: probe ranks [w, nprobe) starting from that bound (the search
       options probe_lo / r0);
    4. all-gather of the 2 x world local top-K lists and the merge kernel,
       which keeps the K smallest (dist, id) pairs.

    With w = 0 it is one wave and one all-gather.  The collectives run on the
    engine's stream (torch.cuda.ExternalStream), so the step has no host round
    trip.  `backend` does the per-rank search and the merge (DeviceShardSearch on
    the GPU; the CPU tests pass an oracle-backed one with gloo, so they drive this
    same orchestration).  Results are bit-identical to the oracle's restricted
    searches (probe_lo / r0) merged by (dist, id)."""

    def __init__(self, backend, nq: int, d: int, K: int, nprobe: int, world: int = 1, rank: int = 0,
                 group=None, waves: int = -1, device=None, stream=None):
        import torch

        self.backend, self.nq, self.d, self.K, self.nprobe = backend, nq, d, K, nprobe
        self.world, self.rank, self.group = world, rank, group
        self.w = first_wave(nprobe, world, waves)
        self.nw = 2 if self.w else 1
        self.G = self.nw * world
        self.dev = torch.device("cpu") if device is None else device
        self.stream = stream
        z = lambda *s, dt: torch.empty(s, dtype=dt, device=self.dev)  # noqa: E731
        self.li = z(self.nw, nq, K, dt=torch.int32)
        self.ld = z(self.nw, nq, K, dt=torch.float64)
        self.lc = z(self.nw, nq, dt=torch.int32)
        self.lm = z(self.nw, nq, dt=torch.int64)   # dims_evaluated per wave
        self.ln = z(self.nw, nq, dt=torch.int64)   # candidates per wave
        self.gi = z(world * self.nw, nq, K, dt=torch.int32)
        self.gd = z(world * self.nw, nq, K, dt=torch.float64)
        self.oi = z(nq, K, dt=torch.int32)
        self.od = z(nq, K, dt=torch.float64)
        self.oc = z(nq, dt=torch.int32)
        self.rb = z(nq, dt=torch.float64)

    @classmethod
    def on_device(cls, local: IvfIndex, nq: int, K: int, nprobe: int, world: int = 1, rank: int = 0,
                  group=None, waves: int = -1, **search_kw) -> "ShardedIvf":
        import torch

        dev = torch.device("cuda", local.ctx.device)
        stream = torch.cuda.ExternalStream(local.ctx.stream_handle(), device=dev)
        return cls(DeviceShardSearch(local, K, **search_kw), nq, local.d, K, nprobe, world, rank, group,
                   waves, dev, stream)

    def _coll(self):
        import contextlib

        import torch

        return torch.cuda.stream(self.stream) if self.stream is not None else contextlib.nullcontext()

    def _wave(self, k):
        return (self.li[k], self.ld[k], self.lc[k], self.lm[k], self.ln[k])

    def step(self, dq, raw: bool = False) -> None:
        """Enqueue one sharded search of the nq queries in dq (on this rank's device;
        transformed, or raw with raw=True: then rotated first, exact fp64, on the engine
        stream); the merged results land in self.oi / self.od / self.oc."""
        import torch
        import torch.distributed as dist

        K = self.K
        if self.stream is not None:  # inputs written on torch's stream come first
            self.stream.wait_stream(torch.cuda.current_stream(self.dev))
        if raw:
            if not hasattr(self, "qt"):
                self.qt = torch.empty((self.nq, self.d), dtype=torch.float32, device=self.dev)
            self.backend.rotate(dq, self.qt, self.nq)
            dq = self.qt
        if self.w:
            self.backend.search(dq, self.nq, self.w, 0, None, self._wave(0))
            with self._coll():
                torch.where(self.lc[0] == K, self.ld[0][:, K - 1],
                            torch.full_like(self.rb, float("inf")), out=self.rb)
                if self.group is not None:
                    dist.all_reduce(self.rb, op=dist.ReduceOp.MIN, group=self.group)
            self.backend.search(dq, self.nq, self.nprobe, self.w, self.rb, self._wave(1))
        else:
            self.backend.search(dq, self.nq, self.nprobe, 0, None, self._wave(0))
        with self._coll():
            if self.group is not None:
                dist.all_gather_into_tensor(self.gi, self.li, group=self.group)
                dist.all_gather_into_tensor(self.gd, self.ld, group=self.group)
            else:
                self.gi.copy_(self.li)
                self.gd.copy_(self.ld)
        self.backend.merge(self.gd, self.gi, self.G, self.nq, self.oi, self.od, self.oc)
        if self.stream is not None:  # and torch's later reads of the outputs wait for the step
            torch.cuda.current_stream(self.dev).wait_stream(self.stream)

    def dims_evaluated(self) -> int:
        """This rank's dims_evaluated summed over its waves (the scanned-bytes counter)."""
        return int(self.lm.sum().item())

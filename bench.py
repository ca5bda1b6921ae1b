#!/usr/bin/env python
"""bench.py — IVF++ ADSampling queries/sec at fixed recall@K on B200.

Metric (BASELINE.json): "IVF++ ADSampling queries/sec at fixed recall@K;
scanned GB/s vs HBM peak".  Default workload: configs[4] = config 5, the
largest config (1e8 x 96 unit-sphere rows, 16 384 lists, 10 000 queries,
K = 100, nprobe 64), which fits one B200:

* N = 1: the whole index on one GPU; one step = all 10 000 queries through
  query rotation (exact fp64) + coarse quantizer + the ADSampling scan with
  top-K.  `value` has the queries resident in HBM; `e2e` repeats the step
  through the host API (pinned host queries in, results out, copies inside the
  timed region).  Config 3 (1M x 960) is measured the same way and reported
  under "cfg3" on the same line.
* N > 1: IVF lists partitioned over the N GPUs (LPT on list sizes), every
  rank answers the same fixed 10 000-query batch over its own lists (strong
  scaling) with the two-wave threshold exchange and the NCCL all-gather +
  merge of shard.ShardedIvf.  `python bench.py --gpus N` spawns the N ranks
  itself (torch.distributed.run) when WORLD_SIZE is unset.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--nprobe 64]
    python bench.py --impl reference ...   # the reference's CPU ivf_query (oracle/_ref)
    python bench.py --mode dco ...         # config-4 fixed-threshold DCO microbench

The reference arm never loads libadsann_b200.so: it generates config 5 with
the oracle's restated generator, rotates it with the reference's own
apply_dataset, assembles the reference IvfIndex around the committed
centroids (tests/golden/cfg5_centroids.npy, reproduced bit-for-bit by the GPU
arm's k-means) and times adsann::ivf_query on all host threads.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
CFG5_CENTROIDS = os.path.join(ROOT, "tests", "golden", "cfg5_centroids.npy")
METRIC = "IVF++ ADSampling queries/sec at fixed recall@K"


# ---------------------------------------------------------------- distributed plumbing
class Dist:
    """One process per GPU: gloo for the control plane (barriers, max over ranks),
    an NCCL group for the data path of the list-sharded search."""

    def __init__(self, backend="gloo", force=False, expect=None):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.nccl = None
        if expect is not None and self.world != expect:
            raise SystemExit(f"bench.py: --gpus {expect} but WORLD_SIZE={self.world}")
        if self.world > 1 or force:
            for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29531"), ("RANK", "0"),
                         ("WORLD_SIZE", "1")):
                os.environ.setdefault(k, v)
            import torch
            import torch.distributed as dist

            dist.init_process_group("gloo")
            self.pg = dist
            if backend == "nccl":
                torch.cuda.set_device(self.local)
                self.nccl = dist.new_group(backend="nccl")
                n = dist.get_world_size(self.nccl)
                if n != self.world:
                    raise SystemExit(f"bench.py: NCCL communicator holds {n} ranks, expected {self.world}")

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def _reduce(self, v: float, op) -> float:
        if not self.pg:
            return v
        import torch

        t = torch.tensor([v], dtype=torch.float64)
        self.pg.all_reduce(t, op=op)
        return float(t.item())

    def allmax(self, v: float) -> float:
        return self._reduce(v, self.pg.ReduceOp.MAX) if self.pg else v

    def allsum(self, v: float) -> float:
        return self._reduce(v, self.pg.ReduceOp.SUM) if self.pg else v

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def ncu_traffic(workload: str):
    """roofline.traffic: DRAM bytes per launch of the dominant kernel from the committed
    ncu capture of the same command (profiles/traffic.json), in GB; None if not captured."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    e = json.load(open(p)).get(workload)
    return None if e is None else round(e["dram_read_gb"] + e["dram_write_gb"], 3)


def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d["hbm_gbs"], "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def load_configs():
    """paper_2303_09855_b200/configs.py loaded by path (no package import, so the
    reference arm does not map libadsann_b200.so)."""
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "ads_bench_configs", os.path.join(ROOT, "paper_2303_09855_b200", "configs.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules["ads_bench_configs"] = mod
    spec.loader.exec_module(mod)
    return mod


def config_for(args, configs=None):
    """BASELINE config args.config, with --cfg-override applied (calibration runs only)."""
    import copy
    import dataclasses

    configs = configs or load_configs()
    cfg = copy.deepcopy(configs.CONFIGS[args.config])
    for kv in filter(None, getattr(args, "cfg_override", "").split(",")):
        k, v = kv.split("=")
        if k in {f.name for f in dataclasses.fields(cfg)}:
            cur = getattr(cfg, k)
            setattr(cfg, k, type(cur)(float(v)) if not isinstance(cur, bool) else v in ("1", "true"))
        else:
            cfg.extra[k] = int(float(v))
        cfg.key += f"-{k}{v}"
    if getattr(args, "nq", 0):
        cfg.nq = args.nq
    if getattr(args, "kmeans_iters", 0):
        cfg.kmeans_iters = args.kmeans_iters
    if getattr(args, "kmeans_init", -1) >= 0:
        cfg.kmeans_init = args.kmeans_init
    return cfg


def workload_config(cfg, nprobe) -> dict:
    """The line's `config`: what defines the workload, identical in both arms."""
    return dict(cfg.describe(), nprobe=nprobe, queries_per_step=cfg.nq,
                l2=f"flushed between timed steps; index {cfg.n * cfg.d * 4 / 1e9:.2f} GB vs 126 MB L2")


def nvtx_push(name):
    try:
        import torch

        torch.cuda.nvtx.range_push(name)
    except Exception:
        pass


def nvtx_pop():
    try:
        import torch

        torch.cuda.nvtx.range_pop()
    except Exception:
        pass


def is_large(cfg) -> bool:
    return cfg.n > 20_000_000


def recall_of(ids, gt, K) -> float:
    ngt = min(len(ids), len(gt))
    return float(np.mean([len(np.intersect1d(ids[i][ids[i] >= 0], gt[i])) for i in range(ngt)]) / K)


# ---------------------------------------------------------------- workload setup (GPU arm)
def setup(cfg, D, log, world=1, rank=0):
    """Index (this rank's shard when world > 1), queries (the same on every rank), ground
    truth (rank 0; first gt_queries queries for config 5).  Returns a dict."""
    import ctypes as C

    import paper_2303_09855_b200 as ads
    from paper_2303_09855_b200 import _lib as L
    from paper_2303_09855_b200 import configs
    from paper_2303_09855_b200.shard import partition_lists, shard_index

    t0 = time.time()
    ctx = ads.Context.default(D.local)
    m = ads.generate_orthogonal(cfg.d, cfg.seed)
    q = configs.generate_queries(cfg)
    owner = (lambda sizes: partition_lists(sizes, world)) if world > 1 else None
    out = {"ads": ads, "ctx": ctx, "m": m, "q": q, "base": None, "t": None, "gt": None, "info": {}}
    if is_large(cfg):
        ng = min(cfg.extra.get("gt_queries", 100), cfg.nq)
        gt_box = {}

        def on_rows(ptr):  # exact top-K in the rotated space over every row (P is orthogonal)
            if rank != 0:
                return
            qt = ads.Transform(m, ctx).apply_dataset(q[:ng])
            dq = ads.DeviceArray.from_host(ctx, qt)
            dg = ads.DeviceArray(ctx, (ng, cfg.K), np.int32)
            L.check(L.ads_brute_force_knn_device(ctx.h, C.c_void_p(ptr), cfg.n, cfg.d, C.c_void_p(dq.ptr),
                                                 ng, cfg.K, C.c_void_p(dg.ptr)))
            gt_box["gt"] = dg.to_host()

        idx, sizes, cent = ads.build_ivf_streamed(
            configs.row_source(cfg), cfg.n, cfg.d, m, cfg.nlist, cfg.seed, 32, cfg.kmeans_iters,
            cfg.extra.get("sample", 2_000_000), chunk=4_000_000, owner=owner, rank=rank,
            on_rows=on_rows, ctx=ctx)
        out["gt"] = gt_box.get("gt")
        if cfg.key == configs.CONFIGS[5].key and os.path.exists(CFG5_CENTROIDS):
            out["info"]["centroids_match_fixture"] = bool(np.array_equal(cent, np.load(CFG5_CENTROIDS)))
        out["info"]["list_rows_max_min"] = [int(sizes.max()), int(sizes.min())]
        if world > 1:
            loads = np.bincount(partition_lists(sizes, world), weights=sizes, minlength=world)
            out["info"]["shard_rows_max_min"] = [int(loads.max()), int(loads.min())]
        log(f"setup: generate + rotate + build_ivf (sampled k-means, certified assignment) "
            f"{time.time() - t0:.1f}s; ground truth on {ng} queries")
    else:
        base, _ = configs.generate(cfg, nq=1)
        t = ads.Transform(m, ctx).apply_dataset(base)
        full = ads.build_ivf(base, t, m, cfg.nlist, cfg.seed, ads.IvfLayout.kSplit, 32,
                             max_iters=cfg.kmeans_iters, init=cfg.kmeans_init, ctx=ctx)
        t1 = time.time()
        if rank == 0:
            out["gt"] = ads.brute_force_knn(base, q, cfg.K, ctx=ctx)
        if world > 1:
            sizes = np.diff(full.list_offsets())
            idx = shard_index(full, partition_lists(sizes, world), rank)
            del full
        else:
            idx = full
        out["base"], out["t"] = base, t
        log(f"setup: data + rotate + build_ivf {t1 - t0:.1f}s, ground truth {time.time() - t1:.1f}s")
    out["idx"] = idx
    return out


def order_sorted(args, nq: int, d: int) -> bool:
    """Whether the library sorts the batch longest-first (capi.cu: query_order 2 and more
    queries than resident search CTAs: 9 per SM for D <= 256 (4-warp CTAs), 3 above)."""
    try:
        import torch

        sms = torch.cuda.get_device_properties(0).multi_processor_count
    except Exception:
        sms = 148
    return args.query_order == 2 and nq > sms * (9 if d <= 256 else 3)


# ---------------------------------------------------------------- one-GPU measurement
def measure(S, cfg, nprobe, args, D, log, steps):
    """Device-resident steps (value, roofline, stages) and host-API steps (e2e) of one index."""
    import ctypes as C

    from paper_2303_09855_b200 import _lib as L

    ads, ctx, idx, q, gt = S["ads"], S["ctx"], S["idx"], S["q"], S["gt"]
    K, nq, d = cfg.K, cfg.nq, cfg.d
    mode = ads.IvfMode.kAdSplit
    opts = ads.search_opts(first=0, step=args.step, warps_per_cta=args.warps, time_stages=True,
                           query_order=args.query_order, ctas_per_sm=args.ctas_per_sm,
                           tile=-1 if getattr(args, "no_dense", False) else 64,
                           rotate_mode=getattr(args, "rotate_mode", 2), walk=getattr(args, "walk", 0),
                           lag=getattr(args, "lag", 0))
    plan = ads.search_plan(idx, K, nprobe, mode, opts=opts)
    dq = ads.DeviceArray.from_host(ctx, q)
    outs = {nm: ads.DeviceArray(ctx, shape, dt) for nm, shape, dt in (
        ("ids", (nq, K), np.int32), ("dists", (nq, K), np.float64), ("cnt", (nq,), np.int32),
        ("dims", (nq,), np.uint64), ("cand", (nq,), np.uint64))}
    P = lambda a: C.c_void_p(a.ptr)  # noqa: E731

    def step():
        L.check(L.ads_ivf_search_device(idx.h, None, P(dq), nq, K, nprobe, int(mode), 2.1, 32, C.byref(opts),
                                        P(outs["ids"]), P(outs["dists"]), P(outs["cnt"]), P(outs["dims"]),
                                        P(outs["cand"])))

    for _ in range(args.warmup):
        ctx.flush_l2()
        step()
    ctx.sync()
    cst = idx.coarse_stats()
    log(f"{cfg.key}: coarse prefilter rescored {cst['rescored'] / max(1, cst['queries']):.1f} centroids "
        f"per query (nprobe {nprobe}), {cst['fallbacks']} exhaustive fallbacks")
    clocks = ClockSampler(D.local)
    step_ms, scan_ms, stage_ms = [], [], []
    D.barrier()
    ctx.sync()
    clocks.start()
    nvtx_push("timed")  # ncu --nvtx --nvtx-include timed/ captures exactly these launches
    for _ in range(steps):
        ctx.flush_l2()  # L2 flushed between timed steps (outside the events)
        ctx.timer_start()
        step()
        step_ms.append(ctx.timer_stop())
        st = idx.last_timings()
        stage_ms.append(st)
        scan_ms.append(float(st[3]))
    ctx.sync()
    nvtx_pop()
    clk = clocks.stop()
    D.barrier()
    total_ms = D.allmax(float(np.sum(step_ms)))
    dims = outs["dims"].to_host()
    ids = outs["ids"].to_host()
    cand = outs["cand"].to_host()
    scanned = 4.0 * float(dims.sum())  # algorithmic bytes per step

    # end to end through the host API (pinned host buffers; H2D of the raw queries and
    # D2H of every result array inside the timed region)
    qh = ads.PinnedArray((nq, d), np.float32)
    qh.array[:] = q
    ho = {nm: ads.PinnedArray(shape, dt) for nm, shape, dt in (
        ("ids", (nq, K), np.int32), ("dists", (nq, K), np.float64), ("cnt", (nq,), np.int32),
        ("dims", (nq,), np.uint64), ("cand", (nq,), np.uint64))}

    def e2e_step():
        L.check(L.ads_ivf_search(idx.h, None, C.c_void_p(qh.ptr), nq, K, nprobe, int(mode), 2.1, 32,
                                 C.byref(opts), *[C.c_void_p(ho[nm].ptr) for nm in
                                                   ("ids", "dists", "cnt", "dims", "cand")]))

    for _ in range(max(1, args.warmup // 2)):
        e2e_step()
    e2e_s = []
    D.barrier()
    for _ in range(steps):
        ctx.flush_l2()
        ctx.sync()
        t0 = time.perf_counter()
        e2e_step()
        e2e_s.append(time.perf_counter() - t0)
    e2e_total = D.allmax(float(np.sum(e2e_s)))
    assert np.array_equal(ho["ids"].array, ids), "e2e and device-resident results differ"
    for a in list(outs.values()) + [dq]:
        a.free()

    peaks = measured_peaks()
    scan_avg = float(np.mean(scan_ms))
    achieved = scanned / (scan_avg / 1e3) / 1e9
    stage = np.mean(np.array(stage_ms), axis=0)
    world_q = nq * D.world * steps
    traffic = ncu_traffic(cfg.key)
    dram = {} if not traffic else {  # ncu DRAM bytes of the scan launch over its live time
        "dram_gbs": traffic / (scan_avg / 1e3), "dram_frac": traffic / (scan_avg / 1e3) / peaks["hbm_gbs"]}
    return {
        "value": world_q / (total_ms / 1e3), "ms_per_step": total_ms / steps,
        "recall_at_k": recall_of(ids, gt, K) if gt is not None else None,
        "recall_queries": min(nq, len(gt)) if gt is not None else 0,
        "e2e": {"value": world_q / e2e_total, "unit": "queries/s", "h2d_bytes_per_step": nq * d * 4,
                "d2h_bytes_per_step": nq * K * (4 + 8) + nq * (4 + 8 + 8)},
        # per step: rotation, query centring, coarse GEMM (tcgen05), prefilter, scan, plus the
        # longest-first order when the batch exceeds one wave of resident CTAs (key kernel +
        # radix sort) (ncu launch lists: profiles/)
        "gpu_launches": (7 if order_sorted(args, nq, d) else 5) * steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / peaks["hbm_gbs"], "frac_vs_nominal_8000": achieved / 8000.0,
                     "traffic": traffic,
                     "traffic_unit": "GB per launch (ncu dram__bytes_read+write, profiles/traffic.json)",
                     "kernel": "ivf_search_kernel", "peak_source": peaks["source"] + ", copy (burst)",
                     "algorithmic_bytes_per_launch": scanned,
                     "scanned_gbs_whole_step": scanned / (float(np.mean(step_ms)) / 1e3) / 1e9, **dram},
        "stages_ms": {"rotate": float(stage[0]), "coarse": float(stage[1]), "select": float(stage[2]),
                      "scan": float(stage[3])},
        "dims_per_query": float(dims.mean()),
        "dims_fraction": float(dims.mean()) / (float(cand.mean()) * d),
        "clocks": clk, "ids": ids,
        "threshold_refresh": {"first": plan["first"], "step": plan["step"]},
        "warps_per_cta": plan["warps_per_cta"], "walk": plan["walk"], "dense_prefix": plan["dense"], "overlapped_chunks": bool(plan["lag"]),
    }


def gpu_mode_line(S, cfg, nprobe, mode_name):
    """The GPU's own IVF+ (kAd) or FDScanning (kFd) on the same index, through the host API."""
    ads, ctx, idx, q, gt = S["ads"], S["ctx"], S["idx"], S["q"], S["gt"]
    mode = {"fd": ads.IvfMode.kFd, "ad": ads.IvfMode.kAd}[mode_name]
    try:
        o = ads.search_opts(time_stages=True)
        ads.ivf_query_batch(idx, None, q, cfg.K, nprobe, mode, opts=o)
        ms, scan = [], []
        for _ in range(3):
            ctx.flush_l2()
            ctx.sync()
            ctx.timer_start()
            r = ads.ivf_query_batch(idx, None, q, cfg.K, nprobe, mode, opts=o)
            ms.append(ctx.timer_stop())
            scan.append(float(idx.last_timings()[3]))
        out = {"value": cfg.nq / (float(np.mean(ms)) / 1e3), "unit": "queries/s",
               "recall_at_k": recall_of(r.ids, gt, cfg.K) if gt is not None else None,
               "scan_ms": float(np.mean(scan)),
               "scan_gbs": 4.0 * float(r.dims.astype(np.float64).sum()) / (float(np.mean(scan)) / 1e3) / 1e9,
               "timing": f"ivf_query_batch {mode.name} through the host API, 3 runs after one warm-up, "
                         f"L2 flushed"}
        return out
    except (RuntimeError, ValueError) as e:
        return {"unavailable": str(e)[:200]}


def cpu_baseline(S, cfg, nprobe, budget_s, log):
    """The reference's ivf_query (oracle/_ref) on the same index, run_timed protocol
    (rotation inside the loop), all host threads, bounded sample of the queries."""
    from oracle import ref_available

    if not ref_available():
        return {"unavailable": "oracle/_ref/libadsann_ref.so not built"}, None
    from oracle import load_ref

    ref = load_ref()
    ads, idx, q, gt, m = S["ads"], S["idx"], S["q"], S["gt"], S["m"]
    t0 = time.time()
    ex = idx.export()
    h = ref.from_split_layout(ex["centroids_t"], ex["list_off"], ex["ids_flat"], ex["a1_t"], ex["a2_t"],
                              seed=cfg.seed)
    del ex
    gc.collect()
    log(f"cpu baseline: reference IvfIndex (kAdSplit arrays) from the GPU index in {time.time() - t0:.1f}s")
    cores = os.cpu_count() or 1

    def run(mode, qs, nthreads):
        ids, _, dims, secs = h.query_batch(None, qs, cfg.K, nprobe, mode, 2.1, 32, nthreads=nthreads,
                                           P=m.entries)
        return ids, dims, secs

    probe = min(64, len(q))
    _, _, s = run("ad-split", q[:probe], cores)
    per_q = s / probe
    ns = int(max(probe, min(len(q), budget_s / max(per_q, 1e-9))))
    ids, dims, secs = run("ad-split", q[:ns], cores)
    st_ns = max(4, min(ns, int(budget_s / 4 / max(per_q * cores, 1e-9))))
    _, _, st_secs = run("ad-split", q[:st_ns], 1)
    out = {"value": ns / secs, "unit": "queries/s", "cores": cores, "kind": "reference",
           "sample": f"first {ns} of {len(q)} queries, adsann::ivf_query kAdSplit with adsann::apply "
                     f"inside the loop (run_timed protocol), {cores} host threads over queries, the "
                     f"same index (reference IvfIndex assembled from the GPU layout)",
           "recall_at_k": recall_of(ids, gt, cfg.K) if gt is not None else None,
           "single_thread_value": st_ns / st_secs,
           "single_thread_sample": f"first {st_ns} queries, 1 thread"}
    if S["base"] is not None:  # configs 1-3: the reference's FD and IVF+ on the full index too
        ex = idx.export()
        from paper_2303_09855_b200 import configs as _c

        asg = _c.list_assignment(ex["list_off"], ex["ids_flat"])
        hf = ref.assemble_ivf(S["base"], S["t"], m.entries, ex["centroids_t"], asg, seed=cfg.seed,
                              split=True, d1=32)
        fd_ns = min(ns, max(probe, ns // 3))
        _, _, _, fs = hf.query_batch(None, q[:fd_ns], cfg.K, nprobe, "fd", nthreads=cores)
        _, _, _, as_ = hf.query_batch(None, q[:fd_ns], cfg.K, nprobe, "ad", nthreads=cores, P=m.entries)
        out.update(fd_value=fd_ns / fs, fd_sample=f"first {fd_ns} queries, ivf_query kFd",
                   ivf_plus_value=fd_ns / as_, ivf_plus_sample=f"first {fd_ns} queries, ivf_query kAd")
    log(f"cpu baseline (reference): {ns} queries IVF++ {ns / secs:.0f} QPS on {cores} threads; "
        f"single thread {st_ns / st_secs:.0f} QPS")
    return out, ids


# ---------------------------------------------------------------- search bench (N = 1)
def run_search(args, D):
    log = (lambda *a: print(*a, file=sys.stderr, flush=True)) if D.rank == 0 else (lambda *a: None)
    cfg = config_for(args)
    nprobe = args.nprobe or cfg.nprobe
    S = setup(cfg, D, log)
    M = measure(S, cfg, nprobe, args, D, log, args.steps)
    res = {
        "metric": METRIC, "value": M["value"], "unit": "queries/s", "n_gpus": D.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": M["ms_per_step"], "higher_is_better": True,
        "scaling": "weak" if D.world > 1 else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Gaussian mixtures with BASELINE.json's shapes; DESIGN.md §6)",
        "config": workload_config(cfg, nprobe),
        "parallelism": f"replicas x{D.world} (query-sharded)" if D.world > 1 else "single GPU, whole index",
        "recall_at_k": M["recall_at_k"], "recall_queries": M["recall_queries"],
        "e2e": M["e2e"], "gpu_launches": M["gpu_launches"], "roofline": M["roofline"],
        "stages_ms": M["stages_ms"], "dims_per_query": M["dims_per_query"],
        "dims_fraction": M["dims_fraction"], "clocks": M["clocks"],
        "threshold_refresh": M["threshold_refresh"], "warps_per_cta": M["warps_per_cta"],
        "walk": M["walk"], "dense_prefix": M["dense_prefix"], "overlapped_chunks": M["overlapped_chunks"],
        "query_rotation": "raw queries rotated on the device each step: 3xTF32 tcgen05 (rotate_mode 2)",
        "setup": S["info"],
    }
    if D.rank == 0 and args.mode == "search":
        res["gpu_ivf_plus"] = gpu_mode_line(S, cfg, nprobe, "ad")
        if S["base"] is not None:
            res["gpu_fd"] = gpu_mode_line(S, cfg, nprobe, "fd")
    if D.rank == 0 and not args.no_cpu_baseline:
        res["cpu_baseline"], _ = cpu_baseline(S, cfg, nprobe, args.cpu_budget, log)
    if args.sweep and D.rank == 0:
        res["sweep"] = sweep(S, cfg, args)
    del S, M
    gc.collect()
    if D.rank == 0 and D.world == 1 and args.config == 5 and not args.no_extra:
        res["cfg3"] = extra_config(args, D, log, 3)
    return res


def extra_config(args, D, log, cid):
    """Another config measured by the same protocol, reported on the same line."""
    import copy

    a = copy.copy(args)
    a.config, a.nprobe, a.nq, a.kmeans_iters, a.kmeans_init, a.cfg_override = cid, 0, 0, 0, -1, ""
    a.rotate_mode = 2
    cfg = config_for(a)
    S = setup(cfg, D, log)
    M = measure(S, cfg, cfg.nprobe, a, D, log, max(3, args.steps // 2))
    out = {"workload": cfg.key, "config": workload_config(cfg, cfg.nprobe), "value": M["value"],
           "unit": "queries/s", "ms_per_step": M["ms_per_step"], "steps": max(3, args.steps // 2),
           "recall_at_k": M["recall_at_k"], "e2e": M["e2e"], "roofline": M["roofline"],
           "stages_ms": M["stages_ms"], "dims_fraction": M["dims_fraction"], "clocks": M["clocks"],
           "threshold_refresh": M["threshold_refresh"], "overlapped_chunks": M["overlapped_chunks"],
           "gpu_fd": gpu_mode_line(S, cfg, cfg.nprobe, "fd")}
    # north-star subsystem 1 delta: the default rotates the query batch on the tensor cores
    # (3xTF32 tcgen05, rotate_mode 2); the same step with the exact fp64 rotation (0), whose
    # results are bit-identical to the reference's on the same raw queries
    a.rotate_mode = 0
    T = measure(S, cfg, cfg.nprobe, a, D, log, 3)
    out["exact_rotation"] = {"value": T["value"], "rotate_ms": T["stages_ms"]["rotate"],
                             "tc_rotate_ms": M["stages_ms"]["rotate"], "recall_at_k": T["recall_at_k"],
                             "ids_equal_to_tc_rotation": bool(np.array_equal(T["ids"], M["ids"])),
                             "note": "rotate_mode 0; the line's value rotates on the tensor cores (~1e-7 relative)"}
    del S
    gc.collect()
    return out


def sweep(S, cfg, args):
    """nprobe sweep: GPU IVF++ (q/s through the host API, recall, dims vs FD) and the
    reference's recall on the same index at every nprobe (first 200 queries)."""
    ads, ctx, idx, q, gt, m = S["ads"], S["ctx"], S["idx"], S["q"], S["gt"], S["m"]
    opts = ads.search_opts(first=0, step=args.step, warps_per_cta=args.warps)
    href = None
    from oracle import ref_available

    if ref_available() and S["base"] is not None:
        from oracle import load_ref
        from paper_2303_09855_b200 import configs as _c

        ex = idx.export()
        href = load_ref().assemble_ivf(S["base"], S["t"], m.entries, ex["centroids_t"],
                                       _c.list_assignment(ex["list_off"], ex["ids_flat"]), seed=cfg.seed,
                                       split=True, d1=32)
    nref = min(200, len(q))
    out = []
    for np_ in cfg.sweep:
        r1 = ads.ivf_query_batch(idx, None, q, cfg.K, np_, ads.IvfMode.kAdSplit, opts=opts)
        row = {"nprobe": np_, "recall": recall_of(r1.ids, gt, cfg.K)}
        if S["base"] is not None:
            rf = ads.ivf_query_batch(idx, None, q, cfg.K, np_, ads.IvfMode.kFd, opts=opts)
            row.update(fd_recall=recall_of(rf.ids, gt, cfg.K),
                       dims_frac=float(r1.dims.sum()) / float(rf.dims.sum()))
        ms = []
        for _ in range(3):  # through the host API (H2D queries, D2H results inside), best of 3
            ctx.flush_l2()
            ctx.sync()
            ctx.timer_start()
            ads.ivf_query_batch(idx, None, q, cfg.K, np_, ads.IvfMode.kAdSplit, opts=opts)
            ms.append(ctx.timer_stop())
        row["e2e_qps"] = cfg.nq / (min(ms) / 1e3)
        if href is not None:
            ids, _, _, _ = href.query_batch(None, q[:nref], cfg.K, np_, "ad-split", nthreads=os.cpu_count(),
                                            P=m.entries)
            row["ref_recall_first"] = nref
            row["ref_recall"] = recall_of(ids, gt[:nref], cfg.K)
            row["gpu_recall_same_queries"] = recall_of(r1.ids[:nref], gt[:nref], cfg.K)
            row["recall_delta"] = abs(row["ref_recall"] - row["gpu_recall_same_queries"])
        out.append(row)
    return out


# ---------------------------------------------------------------- list-sharded search (N > 1)
def run_sharded(args, D):
    """IVF lists partitioned over the N GPUs; every rank answers the same fixed query batch
    over its lists (strong scaling) through shard.ShardedIvf (two waves with the threshold
    all-reduce, NCCL all-gather, merge kernel)."""
    import torch

    from paper_2303_09855_b200.shard import ShardedIvf

    log = (lambda *a: print(*a, file=sys.stderr, flush=True)) if D.rank == 0 else (lambda *a: None)
    cfg = config_for(args)
    nprobe = args.nprobe or cfg.nprobe
    W, K, d, nq = D.world, cfg.K, cfg.d, cfg.nq
    torch.cuda.set_device(D.local)
    S = setup(cfg, D, log, world=W, rank=D.rank)
    ads, ctx, idx, q, gt = S["ads"], S["ctx"], S["idx"], S["q"], S["gt"]
    Sh = ShardedIvf.on_device(idx, nq, K, nprobe, W, D.rank, D.nccl, waves=args.waves, step=args.step,
                              warps=args.warps, P=S["m"].entries)
    dev = torch.device("cuda", D.local)
    dq = torch.from_numpy(q).to(dev)  # raw queries: every step rotates them (exact fp64) first
    torch.cuda.synchronize()
    log(f"sharded: {W} ranks, rank 0 holds {idx.n} rows, first wave {Sh.w} of {nprobe} probes")
    for _ in range(args.warmup):
        ctx.flush_l2()
        Sh.step(dq, raw=True)
    ctx.sync()
    clocks = ClockSampler(D.local)
    D.barrier()
    ctx.sync()
    clocks.start()
    ms = []
    nvtx_push("timed")
    for _ in range(args.steps):
        ctx.flush_l2()
        ctx.sync()
        D.barrier()
        ctx.timer_start()
        Sh.step(dq, raw=True)
        ms.append(ctx.timer_stop())
    nvtx_pop()
    clk = clocks.stop()
    total_ms = D.allmax(float(np.sum(ms)))
    dims = D.allsum(float(Sh.dims_evaluated()))
    ids = Sh.oi.cpu().numpy()
    # e2e: pinned host queries in (rotated on the device), merged ids + dists out, per rank
    qh = torch.from_numpy(q).pin_memory()
    dq_raw = torch.empty_like(dq)
    hi = torch.empty((nq, K), dtype=torch.int32).pin_memory()
    hd = torch.empty((nq, K), dtype=torch.float64).pin_memory()
    e2e = []
    for _ in range(args.steps):
        ctx.flush_l2()
        ctx.sync()
        D.barrier()
        t1 = time.perf_counter()
        dq_raw.copy_(qh, non_blocking=True)
        Sh.step(dq_raw, raw=True)
        hi.copy_(Sh.oi, non_blocking=True)
        hd.copy_(Sh.od, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        e2e.append(time.perf_counter() - t1)
    e2e_total = D.allmax(float(np.sum(e2e)))
    assert np.array_equal(hi.numpy(), ids), "e2e and device-resident sharded results differ"
    scanned = 4.0 * dims
    peaks = measured_peaks()
    res = {
        "metric": METRIC, "value": nq * args.steps / (total_ms / 1e3), "unit": "queries/s", "n_gpus": W,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Gaussian mixtures with BASELINE.json's shapes; DESIGN.md §6)",
        "config": workload_config(cfg, nprobe),
        "parallelism": f"list-sharded x{W} (LPT on list sizes), fixed Q={nq} answered by every rank over "
                       f"its lists, threshold all-reduce after {Sh.w} probes, NCCL all-gather + merge",
        "e2e": {"value": nq * args.steps / e2e_total, "unit": "queries/s",
                "h2d_bytes_per_step": nq * d * 4, "d2h_bytes_per_step": nq * K * 12,
                "note": "per rank: every rank copies the raw queries in and the merged top-K out"},
        # per step and rank: the rotation, 2 waves x (centring, coarse GEMM, prefilter, order
        # key, 5 sort launches, scan) + merge_topk; the all-reduce, all-gather and the
        # torch.where of the bound are NCCL / torch kernels
        "gpu_launches": (1 + (2 * 10 if Sh.w else 10) + 1) * args.steps,
        "roofline": {"bound": "hbm", "achieved": scanned / (total_ms / args.steps / 1e3) / 1e9 / W,
                     "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": scanned / (total_ms / args.steps / 1e3) / 1e9 / W / peaks["hbm_gbs"],
                     "traffic": None, "kernel": "ivf_search_kernel (per GPU, whole step)",
                     "peak_source": peaks["source"], "algorithmic_bytes_per_step_all_ranks": scanned},
        "clocks": clk, "setup": S["info"],
    }
    if D.rank == 0 and gt is not None:
        res["recall_at_k"] = recall_of(ids, gt, K)
        res["recall_queries"] = min(nq, len(gt))
    return res


# ---------------------------------------------------------------- reference arm
def run_reference(args, D):
    """The reference's own adsann::ivf_query (oracle/_ref, compiled from /root/reference),
    on this arm's config and metric, all host threads, rank 0 only.  Config 5 is set up
    without the product library (see the module docstring); configs 1-3 reuse the GPU
    engine's untimed setup (their reference k-means would take up to hours)."""
    if D.rank != 0:
        return None
    log = lambda *a: print(*a, file=sys.stderr, flush=True)  # noqa: E731
    from oracle import ref_available

    configs = load_configs()
    cfg = config_for(args, configs)
    nprobe = args.nprobe or cfg.nprobe
    if not ref_available():
        return {"impl": "reference", "unavailable": "oracle/_ref/libadsann_ref.so not built"}
    from oracle import load_oracle, load_ref

    ref = load_ref()
    cores = os.cpu_count() or 1
    t0 = time.time()
    if is_large(cfg):
        h, q, gt, P, setup_note = reference_setup_large(cfg, configs, ref, load_oracle(), log)
    else:
        S = setup(cfg, D, log)
        ex = S["idx"].export()
        asg = configs.list_assignment(ex["list_off"], ex["ids_flat"])
        h = ref.assemble_ivf(S["base"], S["t"], S["m"].entries, ex["centroids_t"], asg, seed=cfg.seed,
                             split=True, d1=32)
        q, gt, P = S["q"], S["gt"], S["m"].entries
        setup_note = "untimed setup on the GPU engine (data, rotation, k-means reproduced bit-exactly)"
    log(f"reference setup {time.time() - t0:.1f}s ({setup_note})")
    # bounded sample per step: ~cpu_budget / (steps + warmup) seconds each, but at least ~2 s
    # (>= 64 queries per host thread) so the thread pool's tail does not dominate a step
    _, _, _, s = h.query_batch(None, q[:64], cfg.K, nprobe, "ad-split", nthreads=cores, P=P)
    per_q = s / 64
    per_step = max(2.0, args.cpu_budget / max(1, args.steps + args.warmup))
    ns = int(max(64 * cores, min(cfg.nq, per_step / per_q)))
    ns = min(ns, cfg.nq)
    for _ in range(args.warmup):
        h.query_batch(None, q[:ns], cfg.K, nprobe, "ad-split", nthreads=cores, P=P)
    secs, recs = [], []
    for s_ in range(args.steps):
        lo = (s_ * ns) % max(1, cfg.nq - ns + 1)
        ids, _, _, sec = h.query_batch(None, q[lo:lo + ns], cfg.K, nprobe, "ad-split", nthreads=cores, P=P)
        secs.append(sec)
        m_ = min(ns, max(0, len(gt) - lo))
        if m_ > 0:
            recs.append((recall_of(ids[:m_], gt[lo:lo + m_], cfg.K), m_))
    v = ns * args.steps / float(np.sum(secs))
    rec = (sum(r * w for r, w in recs) / sum(w for _, w in recs)) if recs else None
    return {"metric": METRIC, "value": v, "unit": "queries/s", "n_gpus": D.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(secs)), "higher_is_better": True,
            "scaling": "strong" if D.world > 1 else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Gaussian mixtures with BASELINE.json's shapes; DESIGN.md §6)",
            "impl": "reference", "config": workload_config(cfg, nprobe),
            "parallelism": f"{cores} host threads over queries (rank 0 only)",
            "recall_at_k": rec, "setup": setup_note,
            "cpu_baseline": {"value": v, "unit": "queries/s", "cores": cores, "kind": "reference",
                             "sample": f"{ns} queries per step, adsann::ivf_query kAdSplit with adsann::apply "
                                       f"inside the loop (run_timed protocol), {cores} host threads"},
            "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def reference_setup_large(cfg, configs, ref, orc, log):
    """Config 5 for the reference arm with no product code: oracle generator, the
    reference's apply_dataset, committed centroids, exact assignment (oracle.ref_workload),
    kAdSplit-only reference IvfIndex."""
    from oracle import ref_workload

    if not os.path.exists(CFG5_CENTROIDS):
        raise SystemExit("reference arm: tests/golden/cfg5_centroids.npy missing")
    cent = np.load(CFG5_CENTROIDS)
    P = ref.generate_orthogonal(cfg.d, cfg.seed)
    gen = orc.synth_rows
    rows = configs.row_source(cfg, gen=gen)
    q = configs.generate_queries(cfg, gen=gen)
    T = np.empty((cfg.n, cfg.d), np.float32)
    chunk = 2_000_000
    t0 = time.time()
    asg = np.empty(cfg.n, np.int32)
    # CPU: generate + rotate chunk i+1 while the GPU assigns chunk i
    nxt = {}

    def produce(lo):
        hi = min(cfg.n, lo + chunk)
        T[lo:hi] = ref.apply_dataset(P, rows(lo, hi - lo))
        nxt[lo] = hi

    th = threading.Thread(target=produce, args=(0,))
    th.start()
    for lo in range(0, cfg.n, chunk):
        th.join()
        hi = nxt.pop(lo)
        if hi < cfg.n:
            th = threading.Thread(target=produce, args=(hi,))
            th.start()
        asg[lo:hi] = ref_workload.exact_assign(T[lo:hi], cent)
    log(f"reference arm: generated (oracle), rotated (reference apply_dataset) and assigned {cfg.n} rows "
        f"in {time.time() - t0:.1f}s")
    ng = min(cfg.extra.get("gt_queries", 100), cfg.nq)
    gt = ref_workload.exact_knn(T, ref.apply_dataset(P, q[:ng]), cfg.K)
    h = ref.assemble_split(T, cent, asg, seed=cfg.seed, d1=32)
    del T
    gc.collect()
    return h, q, gt, P, ("no product code: oracle generator (pinned to ads_synth_rows), reference "
                         "apply_dataset, committed sampled-k-means centroids (bit-identical to the GPU "
                         "arm's), exact fp64 assignment and ground truth certified in PyTorch on the GPU")


# ---------------------------------------------------------------- main
def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="search", choices=["search", "dco", "transform", "theory"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--nprobe", type=int, default=0)
    ap.add_argument("--nq", type=int, default=0)
    ap.add_argument("--step", type=int, default=0, help="threshold refresh interval (0: 64 x warps)")
    ap.add_argument("--warps", type=int, default=0, help="warps per CTA (0: 4 for D <= 256, else 8)")
    ap.add_argument("--ctas-per-sm", type=int, default=0, help="cap on resident search CTAs per SM (0: occupancy)")
    ap.add_argument("--query-order", type=int, default=2,
                    help="2: longest queries first (default), 1: L2-locality order, 0: input order")
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--walk", type=int, default=0,
                    help="lane walk: 0 engine default, 1 exact fp64, 2 certified fp32 + exact re-walk")
    ap.add_argument("--lag", type=int, default=0,
                    help="overlapped chunks (opts.lag): 0 engine default, 1 on, -1 off")
    ap.add_argument("--no-dense", action="store_true",
                    help="A/B: the lane walk gathers A1 too (no dense prefix phase)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the config-3 measurement on the N=1 line")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--kmeans-init", type=int, default=-1, help="override (profiling runs: 1)")
    ap.add_argument("--kmeans-iters", type=int, default=0)
    ap.add_argument("--shard", default="auto", choices=["auto", "lists", "replicas"],
                    help="N>1: IVF lists partitioned across GPUs (default for config 5) or query-sharded "
                         "replicas (default for the configs that fit one GPU, SURVEY §8e)")
    ap.add_argument("--dco-n", type=int, default=10_000_000)
    ap.add_argument("--waves", type=int, default=-1,
                    help="list-sharded search: probe ranks of the first wave before the threshold "
                         "all-reduce (-1: nprobe/8 when N > 1; 0: one wave, no exchange)")
    ap.add_argument("--cfg-override", default="",
                    help="calibration runs: comma list of Config fields / extra keys, e.g. sigma=0.5")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: spawn the N ranks ourselves (the driver may also launch us
        # under torchrun, which sets WORLD_SIZE)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
               os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    expect = args.gpus if "WORLD_SIZE" in os.environ else None
    if args.shard == "auto":
        args.shard = "lists" if load_configs().CONFIGS[args.config].n > 20_000_000 else "replicas"
    sharded = args.impl == "ours" and args.mode == "search" and args.shard == "lists"
    D = Dist("nccl" if sharded else "gloo", expect=expect if args.impl == "ours" else None)
    try:
        if args.impl == "reference":
            res = run_reference(args, D)
        elif args.mode == "dco":
            from bench_dco import run_dco

            res = run_dco(args, D)
        elif args.mode == "transform":
            from bench_transform import run_transform

            res = run_transform(args, D)
        elif args.mode == "theory":
            from bench_theory import run_theory

            res = run_theory(args, D)
        elif sharded and D.world > 1:
            res = run_sharded(args, D)
        else:
            res = run_search(args, D)
        if D.rank == 0 and res is not None:
            res.pop("ids", None)
            print(json.dumps(res), flush=True)
    finally:
        D.close()


if __name__ == "__main__":
    main()

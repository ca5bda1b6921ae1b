#!/usr/bin/env python
"""bench.py — IVF++ ADSampling queries/sec at fixed recall@K on B200.

Metric (BASELINE.json): "IVF++ ADSampling queries/sec at fixed recall@K;
scanned GB/s vs HBM peak".  Workload: configs[1] (1M x 128, 4096 lists,
10 000 queries, K=100) at the headline nprobe.  One step = one batch of all
queries through the whole hot path on the GPU: query rotation (apply, fp64),
coarse quantizer (fp64 centroid distances + top-nprobe), ADSampling scan
with top-K (ivf_query, split layout).  Inputs are HBM-resident when the timed
region starts (`value`); `e2e` repeats the step through the host API with
pinned host buffers, H2D of the queries and D2H of the results inside.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--nprobe 64]
    python bench.py --impl reference ...   # the reference's CPU ivf_query (oracle/_ref)
    python bench.py --mode dco ...         # config-4 fixed-threshold DCO microbench

N > 1 (torchrun): query-sharded replicas (weak scaling): every rank holds the
index and answers its own 10 000-query batch; no data-path collective.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


# ---------------------------------------------------------------- distributed plumbing
class Dist:
    def __init__(self, backend="gloo", force=False):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.nccl = None
        if self.world > 1 or force or os.environ.get("ADS_FORCE_DIST") == "1":
            # a one-rank group needs the rendezvous variables torchrun would set
            for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29531"), ("RANK", "0"),
                         ("WORLD_SIZE", "1")):
                os.environ.setdefault(k, v)
            import torch
            import torch.distributed as dist

            # control plane (barriers, max-over-ranks) on gloo; data path on NCCL
            dist.init_process_group("gloo")
            self.pg = dist
            if backend == "nccl":
                torch.cuda.set_device(self.local)
                self.nccl = dist.new_group(backend="nccl")

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def allmax(self, v: float) -> float:
        if not self.pg:
            return v
        import torch

        t = torch.tensor([v], dtype=torch.float64)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def allsum(self, v: float) -> float:
        if not self.pg:
            return v
        import torch

        t = torch.tensor([v], dtype=torch.float64)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.SUM)
        return float(t.item())

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


# ---------------------------------------------------------------- workload setup
def config_for(args):
    """BASELINE config args.config, with --cfg-override applied (calibration runs only)."""
    import copy
    import dataclasses

    from paper_2303_09855_b200 import configs

    cfg = copy.deepcopy(configs.CONFIGS[args.config])
    for kv in filter(None, getattr(args, "cfg_override", "").split(",")):
        k, v = kv.split("=")
        if k in {f.name for f in dataclasses.fields(cfg)}:
            cur = getattr(cfg, k)
            setattr(cfg, k, type(cur)(float(v)) if not isinstance(cur, bool) else v in ("1", "true"))
        else:
            cfg.extra[k] = int(float(v))
        cfg.key += f"-{k}{v}"
    return cfg


def large_rotated_dataset(cfg, m, ctx):
    """Config 5's 1e8 rows, generated on the host, rotated on the device (exact fp64);
    the host copy and the unrotated device copy are released."""
    import paper_2303_09855_b200 as ads
    from paper_2303_09855_b200 import api

    kw = dict(kind=cfg.kind, center_scale=cfg.center_scale, center_lo=cfg.center_lo,
              center_hi=cfg.center_hi, sigma=cfg.sigma, decay=cfg.decay, assign_mode=cfg.assign_mode)
    base = api.synth(cfg.n, cfg.d, cfg.components, cfg.seed, 1, **kw)
    dX = ads.DeviceArray.from_host(ctx, base)
    del base
    dT = ads.DeviceArray(ctx, (cfg.n, cfg.d), np.float32)
    ads.Transform(m, ctx).apply_dataset_device(dX, dT)
    ctx.sync()
    dX.free()
    return dT


def device_ground_truth(ads, ctx, dT, qt, K):
    """Exact top-K of the rotated queries qt over the device-resident rotated rows dT
    (P is orthogonal, so this is the raw-space neighbour set up to rounding)."""
    import ctypes as C

    from paper_2303_09855_b200 import _lib as L

    dq = ads.DeviceArray.from_host(ctx, np.ascontiguousarray(qt, np.float32))
    dg = ads.DeviceArray(ctx, (qt.shape[0], K), np.int32)
    L.check(L.ads_brute_force_knn_device(ctx.h, C.c_void_p(dT.ptr), dT.shape[0], dT.shape[1],
                                         C.c_void_p(dq.ptr), qt.shape[0], K, C.c_void_p(dg.ptr)))
    return dg.to_host()


def setup_large(cfg, dev, rank, log):
    """Config 5 (1e8 rows): generate on the host, rotate and build on the device
    (ads_ivf_build_sampled_device), ground truth for the first gt_queries queries
    in the rotated space (P is orthogonal); the host copies are released."""
    import paper_2303_09855_b200 as ads
    from paper_2303_09855_b200 import configs

    t0 = time.time()
    q = configs.generate_queries(cfg, role_base=rank)
    m = ads.generate_orthogonal(cfg.d, cfg.seed)
    ctx = ads.Context.default(dev)
    dT = large_rotated_dataset(cfg, m, ctx)
    t1 = time.time()
    idx = ads.build_ivf_sampled_device(dT, m, cfg.nlist, cfg.seed, 32, cfg.kmeans_iters,
                                       cfg.extra.get("sample", 2_000_000), ctx=ctx)
    t2 = time.time()
    ng = min(cfg.extra.get("gt_queries", 100), q.shape[0])
    gt = device_ground_truth(ads, ctx, dT, ads.Transform(m, ctx).apply_dataset(q[:ng]), cfg.K)
    dT.free()
    t3 = time.time()
    log(f"setup: data+rotate {t1 - t0:.1f}s, build_ivf (sampled k-means + certified assignment) "
        f"{t2 - t1:.1f}s, ground truth ({ng} queries) {t3 - t2:.1f}s")
    return ads, ctx, None, None, q, m, idx, gt


def setup(cfg, dev, rank, log):
    import paper_2303_09855_b200 as ads
    from paper_2303_09855_b200 import configs

    if cfg.n > 20_000_000:
        return setup_large(cfg, dev, rank, log)
    t0 = time.time()
    base, q = configs.generate(cfg, role_base=rank)
    m = ads.generate_orthogonal(cfg.d, cfg.seed)
    ctx = ads.Context.default(dev)
    t = ads.Transform(m, ctx).apply_dataset(base)
    t1 = time.time()
    idx = ads.build_ivf(base, t, m, cfg.nlist, cfg.seed, ads.IvfLayout.kSplit, 32,
                        max_iters=cfg.kmeans_iters, init=cfg.kmeans_init, ctx=ctx)
    t2 = time.time()
    gt = ads.brute_force_knn(base, q, cfg.K, ctx=ctx)
    t3 = time.time()
    log(f"setup: data+rotate {t1 - t0:.1f}s, build_ivf {t2 - t1:.1f}s, ground truth {t3 - t2:.1f}s")
    return ads, ctx, base, t, q, m, idx, gt


def order_sorted(args, nq: int, d: int) -> bool:
    """Whether the library sorts the batch longest-first (capi.cu: query_order 2 and more
    queries than resident search CTAs: 9 per SM for D <= 256 (4-warp CTAs), 3 above)."""
    try:
        import torch

        sms = torch.cuda.get_device_properties(0).multi_processor_count
    except Exception:
        sms = 148
    return args.query_order == 2 and nq > sms * (9 if d <= 256 else 3)


def cpu_baseline_reference(cfg, base, t, m, idx, q, gt, nprobe, budget_s=12.0, log=print):
    """The reference's ivf_query (oracle/_ref, or the oracle port) on the same index,
    run_timed protocol (rotation inside the loop), all host threads, bounded sample."""
    from paper_2303_09855_b200 import configs

    ex = idx.export()
    asg = configs.list_assignment(ex["list_off"], ex["ids_flat"])
    cores = os.cpu_count() or 1
    from oracle import load_oracle, load_ref, ref_available

    if ref_available():
        ref = load_ref()
        h = ref.assemble_ivf(base, t, m.entries, ex["centroids_t"], asg, seed=cfg.seed, split=True, d1=32)
        kind = "reference"

        def run(mode, qs, nthreads):
            ids, dists, dims, secs = h.query_batch(None, qs, cfg.K, nprobe, mode, 2.1, 32,
                                                   nthreads=nthreads, P=m.entries)
            return ids, dims, secs
    else:  # oracle port, single thread per query loop
        orc = load_oracle()
        lay = orc.ivf_layout(base, t, m.entries, ex["centroids_t"], asg, cfg.nlist, 32, True)
        kind, cores = "port", 1

        def run(mode, qs, nthreads):
            qt = orc.apply_dataset(m.entries, qs)
            t0 = time.perf_counter()
            ids = np.full((len(qs), cfg.K), -1, np.int32)
            dims = np.zeros(len(qs), np.uint64)
            for i in range(len(qs)):
                a, _, s = orc.ivf_query(lay, qt[i], qs[i], cfg.K, nprobe, mode)
                ids[i, :len(a)] = a
                dims[i] = s[0]
            return ids, dims, time.perf_counter() - t0

    # size the sample to ~budget_s of CPU work
    probe = min(64, len(q))
    _, _, s = run("ad-split", q[:probe], cores)
    per_q = s / probe
    ns = int(max(probe, min(len(q), budget_s / max(per_q, 1e-9))))
    ids, dims, secs = run("ad-split", q[:ns], cores)
    rec = float(np.mean([len(np.intersect1d(ids[i], gt[i])) for i in range(ns)]) / cfg.K)
    fd_ns = min(ns, max(probe, ns // 3))
    _, _, fd_secs = run("fd", q[:fd_ns], cores)
    # IVF+ (kAd: the contiguous transformed rows) and the reference's own single-thread
    # run_timed protocol (bench.cpp:125-182), on smaller samples of the same queries
    _, _, ad_secs = run("ad", q[:fd_ns], cores)
    st_ns = max(8, min(ns, int(budget_s / 4 / max(per_q * cores, 1e-9))))
    _, _, st_secs = run("ad-split", q[:st_ns], 1)
    log(f"cpu baseline ({kind}): {ns} queries IVF++ {ns / secs:.0f} QPS, FD {fd_ns / fd_secs:.0f} QPS, "
        f"IVF+ {fd_ns / ad_secs:.0f} QPS ({cores} threads); IVF++ single thread {st_ns / st_secs:.0f} QPS")
    return {"value": ns / secs, "unit": "queries/s", "cores": cores, "kind": kind,
            "sample": f"first {ns} of {len(q)} queries, ivf_query kAdSplit, rotation inside the loop "
                      f"(run_timed protocol), {cores} host threads over queries, same index",
            "recall_at_k": rec, "fd_value": fd_ns / fd_secs,
            "fd_sample": f"first {fd_ns} queries, ivf_query kFd",
            "ivf_plus_value": fd_ns / ad_secs, "ivf_plus_sample": f"first {fd_ns} queries, ivf_query kAd",
            "single_thread_value": st_ns / st_secs,
            "single_thread_sample": f"first {st_ns} queries, ivf_query kAdSplit, 1 thread"}, ids, ns


# ---------------------------------------------------------------- search bench
def run_search(args, D: Dist):
    import paper_2303_09855_b200 as ads  # noqa: F401
    from paper_2303_09855_b200 import configs

    log = (lambda *a: print(*a, file=sys.stderr, flush=True)) if D.rank == 0 else (lambda *a: None)
    cfg = config_for(args)
    if args.nq:
        cfg.nq = args.nq
    if args.kmeans_init >= 0:
        cfg.kmeans_init = args.kmeans_init
    if args.kmeans_iters:
        cfg.kmeans_iters = args.kmeans_iters
    nprobe = args.nprobe or cfg.nprobe
    dev = D.local
    ads, ctx, base, t, q, m, idx, gt = setup(cfg, dev, D.rank, log)
    if args.same_query:  # locality experiment: every query = query 0 (perfect L2 reuse)
        q = np.ascontiguousarray(np.repeat(q[:1], q.shape[0], axis=0))
        gt = np.repeat(gt[:1], gt.shape[0], axis=0)
    K, nq, d = cfg.K, cfg.nq, cfg.d
    mode = ads.IvfMode.kAdSplit
    opts = ads.search_opts(first=0, step=args.step, warps_per_cta=args.warps,
                           queries_per_cta=args.slots, time_stages=True, query_order=args.query_order,
                           ctas_per_sm=args.ctas_per_sm)

    # HBM-resident inputs / outputs
    dq = ads.DeviceArray.from_host(ctx, q)
    d_ids = ads.DeviceArray(ctx, (nq, K), np.int32)
    d_dst = ads.DeviceArray(ctx, (nq, K), np.float64)
    d_cnt = ads.DeviceArray(ctx, (nq,), np.int32)
    d_dims = ads.DeviceArray(ctx, (nq,), np.uint64)
    d_cand = ads.DeviceArray(ctx, (nq,), np.uint64)
    import ctypes as C

    from paper_2303_09855_b200 import _lib as L

    def step():
        L.check(L.ads_ivf_search_device(idx.h, None, C.c_void_p(dq.ptr), nq, K, nprobe, int(mode),
                                        2.1, 32, C.byref(opts), C.c_void_p(d_ids.ptr),
                                        C.c_void_p(d_dst.ptr), C.c_void_p(d_cnt.ptr),
                                        C.c_void_p(d_dims.ptr), C.c_void_p(d_cand.ptr)))

    if args.tune and D.rank == 0:
        grid = [(256, 4), (384, 6), (512, 8), (192, 3), (128, 2), (320, 5), (640, 10)]
        if args.tune_grid:
            grid = [tuple(int(v) for v in t.split("x")) for t in args.tune_grid.split(",")]
        for st_, w_ in grid:
            o2 = ads.search_opts(first=0, step=st_, warps_per_cta=w_, time_stages=True)
            ts, dm = [], 0
            for rep in range(4):
                ctx.flush_l2()
                r_ = ads.ivf_query_batch(idx, None, q, K, nprobe, mode, opts=o2)
                ts.append(float(idx.last_timings()[3]))
                dm = float(r_.dims.mean())
            scan = float(np.min(ts))
            log(f"tune step={st_} warps={w_}: scan {scan:.2f} ms, dims/query {dm:.0f}, "
                f"recall {ads.recall_batch(r_.ids[:len(gt)], gt, K):.5f}")
    for _ in range(args.warmup):
        ctx.flush_l2()
        step()
    ctx.sync()
    cst = idx.coarse_stats()
    log(f"coarse prefilter: {cst['rescored'] / max(1, cst['queries']):.1f} centroids rescored per query "
        f"(nprobe {nprobe}), {cst['fallbacks']} exhaustive fallbacks")
    clocks = ClockSampler(dev)
    step_ms, scan_ms, stage_ms = [], [], []
    D.barrier()
    ctx.sync()
    clocks.start()
    for _ in range(args.steps):
        ctx.flush_l2()  # L2 flushed between timed steps (outside the events)
        ctx.timer_start()
        step()
        step_ms.append(ctx.timer_stop())
        st = idx.last_timings()
        stage_ms.append(st)
        scan_ms.append(float(st[3]))
    ctx.sync()
    clk = clocks.stop()
    D.barrier()
    total_ms = D.allmax(float(np.sum(step_ms)))
    dims = d_dims.to_host()
    ids = d_ids.to_host()
    ngt = min(nq, len(gt))
    recall = float(np.mean([len(np.intersect1d(ids[i][ids[i] >= 0], gt[i])) for i in range(ngt)]) / K)
    scanned = 4.0 * float(dims.sum())  # algorithmic bytes per step

    # end to end through the host API with pinned buffers
    qh = ads.PinnedArray((nq, d), np.float32)
    qh.array[:] = q
    out = {nm: ads.PinnedArray(shape, dt) for nm, shape, dt in (
        ("ids", (nq, K), np.int32), ("dists", (nq, K), np.float64), ("cnt", (nq,), np.int32),
        ("dims", (nq,), np.uint64), ("cand", (nq,), np.uint64))}

    def e2e_step():
        L.check(L.ads_ivf_search(idx.h, None, C.c_void_p(qh.ptr), nq, K, nprobe, int(mode), 2.1, 32,
                                 C.byref(opts), C.c_void_p(out["ids"].ptr), C.c_void_p(out["dists"].ptr),
                                 C.c_void_p(out["cnt"].ptr), C.c_void_p(out["dims"].ptr),
                                 C.c_void_p(out["cand"].ptr)))

    for _ in range(max(1, args.warmup // 2)):
        e2e_step()
    e2e_s = []
    D.barrier()
    for _ in range(args.steps):
        ctx.flush_l2()
        ctx.sync()
        t0 = time.perf_counter()
        e2e_step()
        e2e_s.append(time.perf_counter() - t0)
    e2e_total = D.allmax(float(np.sum(e2e_s)))
    assert np.array_equal(out["ids"].array, ids), "e2e and device-resident results differ"

    world_q = nq * D.world * args.steps
    value = world_q / (total_ms / 1e3)
    peaks = measured_peaks()
    scan_avg = float(np.mean(scan_ms))
    achieved = scanned / (scan_avg / 1e3) / 1e9
    stage = np.mean(np.array(stage_ms), axis=0)
    res = {
        "metric": "IVF++ ADSampling queries/sec at fixed recall@K",
        "value": value, "unit": "queries/s", "n_gpus": D.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(cfg.describe(), nprobe=nprobe, recall_at_k=recall,
                       parallelism=f"replicas{D.world}" if D.world > 1 else "single-gpu",
                       l2=f"flushed between timed steps (and index {cfg.n * d * 4 / 1e6:.0f} MB vs 126 MB L2)",
                       threshold_refresh={"first": K, "step": ads.search_shape(d, args.step, args.warps)[0]},
                       warps_per_cta=ads.search_shape(d, args.step, args.warps)[1]),
        "e2e": {"value": world_q / e2e_total, "unit": "queries/s",
                "h2d_bytes_per_step": nq * d * 4,
                "d2h_bytes_per_step": nq * K * (4 + 8) + nq * (4 + 8 + 8)},
        # per step: rotation, query centring, coarse GEMM (tcgen05), prefilter, scan, plus
        # the longest-first order when the batch exceeds one wave of resident CTAs (key
        # kernel + CUB radix sort: histogram, bin scan, three onesweep passes)
        # (ncu launch list: profiles/r01g_launches.csv)
        "gpu_launches": (11 if order_sorted(args, nq, d) else 5) * args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / peaks["hbm_gbs"], "frac_vs_nominal_8000": achieved / 8000.0,
                     "traffic": ncu_traffic(cfg.key),
                     "traffic_unit": "GB per launch (ncu dram__bytes_read+write, profiles/traffic.json)",
                     "kernel": "ivf_search_kernel<4>", "peak_source": peaks["source"] + ", copy (burst)",
                     "algorithmic_bytes_per_launch": scanned,
                     "scanned_gbs_whole_step": scanned / (float(np.mean(step_ms)) / 1e3) / 1e9},
        "stages_ms": {"rotate": float(stage[0]), "coarse": float(stage[1]), "select": float(stage[2]),
                      "scan": float(stage[3])},
        "dims_per_query": float(dims.mean()), "dims_fraction": float(dims.mean()) / (
            float(d_cand.to_host().mean()) * d),
        "clocks": clk,
    }
    if ngt < nq:
        res["config"]["recall_queries"] = ngt
    if D.rank == 0 and not args.no_cpu_baseline:
        if base is None:
            res["cpu_baseline"] = {"unavailable": "the reference's in-memory IvfIndex of 1e8 x 96 (raw, "
                                                  "transformed, A1/A2 copies) exceeds the host's 196 GB"}
        else:
            cb, _, _ = cpu_baseline_reference(cfg, base, t, m, idx, q, gt, nprobe, args.cpu_budget, log)
            res["cpu_baseline"] = cb
    if D.rank == 0 and args.mode == "search":
        # the GPU's own FDScanning (kFd: full fp64 distances over the raw vectors) on the
        # same index, queries and nprobe, next to the reference's CPU FD above
        try:
            fd_opts = ads.search_opts(time_stages=True)
            ads.ivf_query_batch(idx, None, q, K, nprobe, ads.IvfMode.kFd, opts=fd_opts)
            fms, fscan = [], []
            for _ in range(3):
                ctx.flush_l2()
                ctx.sync()
                ctx.timer_start()
                rf = ads.ivf_query_batch(idx, None, q, K, nprobe, ads.IvfMode.kFd, opts=fd_opts)
                fms.append(ctx.timer_stop())
                fscan.append(float(idx.last_timings()[3]))
            fd_dims = float(rf.dims.astype(np.float64).sum())
            res["gpu_fd"] = {
                "value": nq / (float(np.mean(fms)) / 1e3), "unit": "queries/s",
                "recall_at_k": ads.recall_batch(rf.ids[:ngt], gt[:ngt], K),
                "scan_ms": float(np.mean(fscan)),
                "scan_gbs": 4.0 * fd_dims / (float(np.mean(fscan)) / 1e3) / 1e9,
                "timing": "ivf_query_batch kFd through the host API (H2D queries, D2H results inside), "
                          "3 runs after one warm-up, L2 flushed"}
            log(f"GPU FDScanning: {res['gpu_fd']['value']:.0f} q/s, scan {res['gpu_fd']['scan_ms']:.2f} ms "
                f"({res['gpu_fd']['scan_gbs']:.0f} GB/s), recall {res['gpu_fd']['recall_at_k']:.5f}")
        except (RuntimeError, ValueError) as e:
            res["gpu_fd"] = {"unavailable": str(e)[:200]}
        try:  # IVF+ (kAd) on the GPU, same index
            ads.ivf_query_batch(idx, None, q, K, nprobe, ads.IvfMode.kAd, opts=fd_opts)
            ams = []
            for _ in range(3):
                ctx.flush_l2()
                ctx.sync()
                ctx.timer_start()
                ra = ads.ivf_query_batch(idx, None, q, K, nprobe, ads.IvfMode.kAd, opts=fd_opts)
                ams.append(ctx.timer_stop())
            res["gpu_ivf_plus"] = {"value": nq / (float(np.mean(ams)) / 1e3), "unit": "queries/s",
                                   "recall_at_k": ads.recall_batch(ra.ids[:ngt], gt[:ngt], K),
                                   "timing": "ivf_query_batch kAd, as gpu_fd"}
        except (RuntimeError, ValueError) as e:
            res["gpu_ivf_plus"] = {"unavailable": str(e)[:200]}
    if args.sweep and D.rank == 0:
        sw = []
        for np_ in cfg.sweep:
            r1 = ads.ivf_query_batch(idx, None, q, K, np_, mode, opts=opts)
            rf = ads.ivf_query_batch(idx, None, q, K, np_, ads.IvfMode.kFd, opts=opts)
            ctx.sync()
            ctx.timer_start()
            step_np = ads.ivf_query_batch(idx, None, q, K, np_, mode, opts=opts)
            ms = ctx.timer_stop()
            sw.append({"nprobe": np_, "recall": ads.recall_batch(r1.ids[:len(gt)], gt, K),
                       "fd_recall": ads.recall_batch(rf.ids[:len(gt)], gt, K),
                       "dims_frac": float(r1.dims.sum()) / float(rf.dims.sum()),
                       "e2e_qps": nq / (ms / 1e3)})
            del step_np
        res["sweep"] = sw
    return res


# ---------------------------------------------------------------- list-sharded search (N > 1)
def run_search_sharded(args, D: Dist):
    """IVF lists partitioned over the N GPUs (LPT on list sizes); every rank scans
    all queries over its own lists, the per-rank top-K go through one NCCL
    all-gather per result array on the engine's stream and a merge kernel keeps
    the K smallest (dist, id) pairs.  Weak scaling: the job answers N x nq
    queries per step (each rank contributes its own nq-query batch)."""
    import ctypes as C

    import torch

    import paper_2303_09855_b200 as ads
    from paper_2303_09855_b200 import _lib as L
    from paper_2303_09855_b200 import configs
    from paper_2303_09855_b200.shard import merge_topk_device, partition_lists, shard_index

    log = (lambda *a: print(*a, file=sys.stderr, flush=True)) if D.rank == 0 else (lambda *a: None)
    cfg = config_for(args)
    if args.nq:
        cfg.nq = args.nq
    if args.kmeans_init >= 0:
        cfg.kmeans_init = args.kmeans_init
    if args.kmeans_iters:
        cfg.kmeans_iters = args.kmeans_iters
    nprobe = args.nprobe or cfg.nprobe
    W, K, d = D.world, cfg.K, cfg.d
    torch.cuda.set_device(D.local)
    t0 = time.time()
    qs = np.concatenate([configs.generate_queries(cfg, role_base=r, nq=cfg.nq) for r in range(W)])
    nq = qs.shape[0]
    m = ads.generate_orthogonal(d, cfg.seed)
    ctx = ads.Context.default(D.local)
    if cfg.n > 20_000_000:
        # config 5: every rank builds the same index on its device (seeded, deterministic),
        # keeps its own lists and drops the rest; ground truth for the first gt_queries
        dT = large_rotated_dataset(cfg, m, ctx)
        full = ads.build_ivf_sampled_device(dT, m, cfg.nlist, cfg.seed, 32, cfg.kmeans_iters,
                                            cfg.extra.get("sample", 2_000_000), ctx=ctx)
        sizes = np.diff(full.list_offsets())
        owner = partition_lists(sizes, W)
        local = shard_index(full, owner, D.rank)
        del full
        gt = None
        if D.rank == 0:
            ng = min(cfg.extra.get("gt_queries", 100), nq)
            gt = device_ground_truth(ads, ctx, dT, ads.Transform(m, ctx).apply_dataset(qs[:ng]), K)
        dT.free()
    else:
        base, _ = configs.generate(cfg, nq=1)
        t = ads.Transform(m, ctx).apply_dataset(base)
        full = ads.build_ivf(base, t, m, cfg.nlist, cfg.seed, ads.IvfLayout.kSplit, 32,
                             max_iters=cfg.kmeans_iters, init=cfg.kmeans_init, ctx=ctx)
        sizes = np.diff(full.list_offsets())
        owner = partition_lists(sizes, W)
        local = shard_index(full, owner, D.rank)
        del full
        gt = ads.brute_force_knn(base, qs, K, ctx=ctx) if D.rank == 0 else None
    log(f"sharded setup {time.time() - t0:.1f}s: {W} ranks, local rows {local.n} "
        f"(max/min shard rows {np.bincount(owner, weights=sizes).max():.0f}/"
        f"{np.bincount(owner, weights=sizes).min():.0f})")

    dev = torch.device("cuda", D.local)
    stream = torch.cuda.ExternalStream(ctx.stream_handle(), device=dev)
    dq = torch.from_numpy(qs).to(dev)
    # two waves with the threshold exchange of SURVEY §8e (--waves 0 disables it): probe ranks
    # [0, w) on every rank, an all-reduce (min) of the per-query K-th distances (an upper bound on
    # the global K-th distance), then ranks [w, nprobe) starting from that bound; the merge keeps
    # the K smallest (dist, id) pairs of the 2 x N local results
    w = args.waves if args.waves >= 0 else (max(1, nprobe // 8) if W > 1 else 0)
    w = w if 0 < w < nprobe else 0
    G = 2 * W if w else W
    li = torch.empty((G // W, nq, K), dtype=torch.int32, device=dev)
    ld = torch.empty((G // W, nq, K), dtype=torch.float64, device=dev)
    lc = torch.empty((G // W, nq), dtype=torch.int32, device=dev)
    lm = torch.empty((G // W, nq), dtype=torch.int64, device=dev)
    ln = torch.empty((G // W, nq), dtype=torch.int64, device=dev)
    gi = torch.empty((W, G // W, nq, K), dtype=torch.int32, device=dev)
    gd = torch.empty((W, G // W, nq, K), dtype=torch.float64, device=dev)
    oi = torch.empty((nq, K), dtype=torch.int32, device=dev)
    od = torch.empty((nq, K), dtype=torch.float64, device=dev)
    oc = torch.empty((nq,), dtype=torch.int32, device=dev)
    rb = torch.empty((nq,), dtype=torch.float64, device=dev)
    opts = ads.search_opts(first=0, step=args.step, warps_per_cta=args.warps, time_stages=True)
    opts2 = ads.search_opts(first=0, step=args.step, warps_per_cta=args.warps, time_stages=True,
                            probe_lo=w)
    opts2.r0 = rb.data_ptr()
    mode = ads.IvfMode.kAdSplit
    torch.cuda.synchronize()

    def search(o, np_, k):
        L.check(L.ads_ivf_search_device(local.h, None, C.c_void_p(dq.data_ptr()), nq, K, np_,
                                        int(mode), 2.1, 32, C.byref(o), C.c_void_p(li[k].data_ptr()),
                                        C.c_void_p(ld[k].data_ptr()), C.c_void_p(lc[k].data_ptr()),
                                        C.c_void_p(lm[k].data_ptr()), C.c_void_p(ln[k].data_ptr())))

    def step():
        if w:
            search(opts, w, 0)
            with torch.cuda.stream(stream):
                torch.where(lc[0] == K, ld[0][:, K - 1], torch.full_like(rb, float("inf")), out=rb)
                D.pg.all_reduce(rb, op=D.pg.ReduceOp.MIN, group=D.nccl)
            search(opts2, nprobe, 1)
        else:
            search(opts, nprobe, 0)
        with torch.cuda.stream(stream):
            D.pg.all_gather_into_tensor(gi, li, group=D.nccl)
            D.pg.all_gather_into_tensor(gd, ld, group=D.nccl)
        merge_topk_device(ctx, gd.data_ptr(), gi.data_ptr(), G, nq, K, oi.data_ptr(),
                          od.data_ptr(), oc.data_ptr())

    for _ in range(args.warmup):
        ctx.flush_l2()
        step()
    ctx.sync()
    clocks = ClockSampler(D.local)
    D.barrier()
    ctx.sync()
    clocks.start()
    ms = []
    for _ in range(args.steps):
        ctx.flush_l2()
        D.barrier()
        ctx.timer_start()
        step()
        ms.append(ctx.timer_stop())
    clk = clocks.stop()
    total_ms = D.allmax(float(np.sum(ms)))
    dims = D.allsum(float(lm.sum().item()))
    res = {
        "metric": "IVF++ ADSampling queries/sec at fixed recall@K", "value": nq * args.steps / (total_ms / 1e3),
        "unit": "queries/s", "n_gpus": W, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(cfg.describe(), nprobe=nprobe, nq_total=nq,
                       parallelism=f"list-sharded x{W} + NCCL all-gather + merge",
                       threshold_exchange={"first_wave_probes": w} if w else None),
        # per step: 11 search kernels per wave (see run_search) + merge_topk (NCCL collectives
        # and the torch.where of the exchange are library kernels)
        "gpu_launches": (23 if w else 12) * args.steps,
        "scanned_gb_per_step_all_ranks": 4.0 * dims / 1e9,
        "clocks": clk,
    }
    if D.rank == 0:
        ids = oi.cpu().numpy()
        ngt = min(nq, len(gt))
        res["config"]["recall_at_k"] = float(np.mean([len(np.intersect1d(ids[i][ids[i] >= 0], gt[i]))
                                                      for i in range(ngt)]) / K)
        if ngt < nq:
            res["config"]["recall_queries"] = ngt
    # e2e: host queries in, merged results out (pinned buffers), same collective path
    qh = ads.PinnedArray((nq, d), np.float32)
    qh.array[:] = qs
    hout = ads.PinnedArray((nq, K), np.int32)
    e2e = []
    for _ in range(args.steps):
        D.barrier()
        t1 = time.perf_counter()
        dq.copy_(torch.from_numpy(qh.array), non_blocking=True)
        torch.cuda.synchronize()
        step()
        ctx.sync()
        torch.cuda.synchronize()
        hout.array[:] = oi.cpu().numpy()
        e2e.append(time.perf_counter() - t1)
    e2e_total = D.allmax(float(np.sum(e2e)))
    res["e2e"] = {"value": nq * args.steps / e2e_total, "unit": "queries/s",
                  "h2d_bytes_per_step": nq * d * 4, "d2h_bytes_per_step": nq * K * 4}
    return res


# ---------------------------------------------------------------- reference arm
def run_reference(args, D: Dist):
    """The reference's own ivf_query (compiled from /root/reference by oracle/Makefile),
    on this arm's config, all host threads.  Its index is the one the reference's
    build_ivf produces (k-means reproduced bit-exactly on the GPU as untimed setup)."""
    from paper_2303_09855_b200 import configs

    if D.rank != 0:
        return None
    log = lambda *a: print(*a, file=sys.stderr, flush=True)  # noqa: E731
    from oracle import ref_available

    cfg = config_for(args)
    if args.nq:
        cfg.nq = args.nq
    nprobe = args.nprobe or cfg.nprobe
    ads, ctx, base, t, q, m, idx, gt = setup(cfg, 0, 0, log)
    ex = idx.export()
    asg = configs.list_assignment(ex["list_off"], ex["ids_flat"])
    cores = os.cpu_count() or 1
    if ref_available():
        from oracle import load_ref

        h = load_ref().assemble_ivf(base, t, m.entries, ex["centroids_t"], asg, seed=cfg.seed,
                                    split=True, d1=32)
        kind = "reference"
    else:
        return {"impl": "reference", "unavailable": "oracle/_ref/libadsann_ref.so not built"}
    # bounded sample per step: ~args.cpu_budget / steps seconds each
    _, _, _, s = h.query_batch(None, q[:64], cfg.K, nprobe, "ad-split", nthreads=cores, P=m.entries)
    per_q = s / 64
    ns = int(max(64, min(nq_cap(cfg), args.cpu_budget / max(1, args.steps + args.warmup) / per_q)))
    for w in range(args.warmup):
        h.query_batch(None, q[:ns], cfg.K, nprobe, "ad-split", nthreads=cores, P=m.entries)
    secs = []
    recs = []
    for s_ in range(args.steps):
        lo = (s_ * ns) % max(1, cfg.nq - ns + 1)
        ids, _, _, sec = h.query_batch(None, q[lo:lo + ns], cfg.K, nprobe, "ad-split",
                                       nthreads=cores, P=m.entries)
        secs.append(sec)
        recs.append(np.mean([len(np.intersect1d(ids[i], gt[lo + i])) for i in range(ns)]) / cfg.K)
    v = ns * args.steps / float(np.sum(secs))
    return {"metric": "IVF++ ADSampling queries/sec at fixed recall@K", "value": v,
            "unit": "queries/s", "n_gpus": D.world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * float(np.mean(secs)), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": dict(cfg.describe(), nprobe=nprobe, recall_at_k=float(np.mean(recs))),
            "cpu_baseline": {"value": v, "unit": "queries/s", "cores": cores, "kind": kind,
                             "sample": f"{ns} queries per step, ivf_query kAdSplit with rotation "
                                       f"inside the loop (run_timed protocol), {cores} host threads"},
            "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def nq_cap(cfg):
    return cfg.nq


# ---------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="search", choices=["search", "dco", "transform", "theory"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--nprobe", type=int, default=0)
    ap.add_argument("--nq", type=int, default=0)
    ap.add_argument("--step", type=int, default=0, help="threshold refresh interval (0: 64 x warps)")
    ap.add_argument("--warps", type=int, default=0, help="warps per CTA (0: 4 for D <= 256, else 10)")
    ap.add_argument("--slots", type=int, default=4, help="queries served concurrently per CTA")
    ap.add_argument("--ctas-per-sm", type=int, default=0, help="cap on resident search CTAs per SM (0: occupancy)")
    ap.add_argument("--query-order", type=int, default=2,
                    help="2: longest queries first (default), 1: L2-locality order, 0: input order")
    ap.add_argument("--same-query", action="store_true", help="experiment: all queries = query 0")
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--tune", action="store_true", help="time (step, warps) variants after setup")
    ap.add_argument("--tune-grid", default="", help="comma list of STEPxWARPS for --tune")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--kmeans-init", type=int, default=-1, help="override (profiling runs: 1)")
    ap.add_argument("--shard", default="auto", choices=["auto", "lists", "replicas"],
                    help="N>1: IVF lists partitioned across GPUs + NCCL all-gather merge, or query-sharded "
                         "replicas; auto = lists for config 5 (the sharded config), replicas for configs that "
                         "fit one GPU (SURVEY §8e)")
    ap.add_argument("--dco-n", type=int, default=10_000_000)
    ap.add_argument("--waves", type=int, default=-1,
                    help="list-sharded search: probe ranks of the first wave before the threshold "
                         "all-reduce (-1: nprobe/8 when N > 1, else one wave; 0: one wave, no exchange)")
    ap.add_argument("--force-shard", action="store_true",
                    help="run the list-sharded path even at N=1 (exercises NCCL + merge)")
    ap.add_argument("--kmeans-iters", type=int, default=0)
    ap.add_argument("--cfg-override", default="",
                    help="calibration runs: comma list of Config fields / extra keys, e.g. sigma=0.5,gt_queries=30")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.shard == "auto":
        from paper_2303_09855_b200 import configs as _cf

        args.shard = "lists" if (args.force_shard or _cf.CONFIGS[args.config].n > 20_000_000) else "replicas"
    sharded = args.impl == "ours" and args.mode == "search" and args.shard == "lists"
    D = Dist("nccl" if sharded else "gloo", force=sharded and args.force_shard)
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
        elif sharded and (D.world > 1 or args.force_shard):
            res = run_search_sharded(args, D)
        else:
            res = run_search(args, D)
        if D.rank == 0 and res is not None:
            print(json.dumps(res), flush=True)
    finally:
        D.close()


if __name__ == "__main__":
    main()

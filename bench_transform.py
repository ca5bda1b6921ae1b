"""Rotation of a dataset by the random orthogonal matrix P (transform.cpp:99-149),
the first subsystem of the north star: exact fp64 on the CUDA cores (the
engine's default, bit-identical to the reference) vs the 3xTF32 split on the
tcgen05 tensor cores (ads_apply_dataset_tc).  One step = the whole dataset of
the chosen config (configs[2]: 1 M x 960 by default) rotated once, inputs and
outputs resident in HBM, L2 flushed between steps.  `python bench.py --mode transform`.
"""
from __future__ import annotations

import time

import numpy as np


def _tf32_peak() -> dict:
    from bench import ROOT
    import json
    import os

    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        # dense TF32 runs at half the dense BF16 rate on B200 (1.1 vs 2.25 PFLOP/s nominal)
        return {"tflops": d["bf16_tflops"] / 2.0, "source": "measured bf16 (MEASURED_PEAKS.json) / 2"}
    return {"tflops": 1100.0, "source": "fallback nominal dense TF32 (B200_PROFILING.md)"}


def run_transform(args, D):
    import paper_2303_09855_b200 as ads
    from paper_2303_09855_b200 import configs
    from bench import ClockSampler

    log = (lambda *a: print(*a, file=__import__("sys").stderr, flush=True)) if D.rank == 0 else (lambda *a: None)
    cfg = configs.CONFIGS[args.config if args.config != 2 else 3]
    n, d = cfg.n, cfg.d
    t0 = time.time()
    X = ads.synth(n, d, 64, 11, 1, kind=0, center_scale=1.0, sigma=1.0)
    m = ads.generate_orthogonal(d, 7)
    ctx = ads.Context.default(D.local)
    dX = ads.DeviceArray.from_host(ctx, X)
    dY = ads.DeviceArray(ctx, (n, d), np.float32)
    t = ads.Transform(m, ctx)
    log(f"transform setup {time.time() - t0:.1f}s ({n} x {d})")

    def timed(fn):
        for _ in range(args.warmup):
            ctx.flush_l2()
            fn()
        ctx.sync()
        clocks = ClockSampler(D.local)
        clocks.start()
        ms = []
        for _ in range(args.steps):
            ctx.flush_l2()
            ctx.timer_start()
            fn()
            ms.append(ctx.timer_stop())
        return float(np.mean(ms)), clocks.stop()

    exact_ms, _ = timed(lambda: t.apply_dataset_device(dX, dY))
    exact_sample = dY.to_host()[:256].copy()
    tc_ms, clocks = timed(lambda: t.apply_dataset_tc_device(dX, dY))
    tc_sample = dY.to_host()[:256]
    xn = np.linalg.norm(X[:256].astype(np.float64), axis=1)
    err = float((np.abs(tc_sample.astype(np.float64) - exact_sample).max(axis=1) / xn).max())
    useful = 2.0 * n * d * d
    peak = _tf32_peak()
    # the 3xTF32 rotation issues three TF32 products per useful product
    achieved = 3.0 * useful / (tc_ms / 1e3) / 1e12
    # end to end through the host API (host X in, host Y out, copies inside)
    import time as _time

    t.apply_dataset_tc(X[:1024])
    e2e_s = []
    for _ in range(2):
        t0 = _time.perf_counter()
        t.apply_dataset_tc(X)
        e2e_s.append(_time.perf_counter() - t0)
    e2e_sec = float(np.mean(e2e_s))
    log(f"exact fp64: {exact_ms:.2f} ms, 3xTF32 tensor cores: {tc_ms:.2f} ms, max |err|/|x| {err:.2e}")
    # the binding roof: tensor pipe at high D (1 M x 960), HBM at low D (config 5's 96:
    # 72 issued TF32 flops per byte, below the ridge): X read + Y written once
    from bench import measured_peaks

    hbm = measured_peaks()
    gbs = 8.0 * n * d / (tc_ms / 1e3) / 1e9
    tensor = {"bound": "tensor", "achieved": achieved, "peak": peak["tflops"], "unit": "TFLOP/s",
              "frac": achieved / peak["tflops"], "peak_source": peak["source"]}
    mem = {"bound": "hbm", "achieved": gbs, "peak": hbm["hbm_gbs"], "unit": "GB/s",
           "frac": gbs / hbm["hbm_gbs"], "peak_source": hbm["source"] + ", copy"}
    roofline = dict(mem if mem["frac"] > tensor["frac"] else tensor)
    roofline.update({"other": tensor if roofline["bound"] == "hbm" else mem,
                     "traffic": 7.66 if (n, d) == (1_000_000, 960) else None,
                     "traffic_unit": "GB per launch (ncu dram read+write, profiles/r01_ncu_tensorcore.md, prof_pair2)",
                     "useful_tflops": useful / (tc_ms / 1e3) / 1e12,
                     "kernel": "tc_rotate_pair_kernel (TF32 flops issued = 3 x 2 n D^2; useful = 2 n D^2)"})
    return {
        "metric": "dataset rotation vectors/s (3xTF32 tensor cores)", "value": n / (tc_ms / 1e3),
        "unit": "vectors/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": tc_ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "tf32x3", "data": "synthetic",
        "config": {"workload": f"rotate-{n}x{d}", "n": n, "d": d,
                   "l2": "flushed between timed steps"},
        "exact_fp64": {"value": n / (exact_ms / 1e3), "unit": "vectors/s", "ms_per_step": exact_ms,
                       "note": "engine default: bit-identical to the reference's fp64 apply_dataset"},
        "max_abs_err_over_norm": err,
        "e2e": {"value": n / e2e_sec, "unit": "vectors/s", "h2d_bytes_per_step": int(X.nbytes),
                "d2h_bytes_per_step": int(X.nbytes),
                "timing": "Transform.apply_dataset_tc on host arrays (ads_apply_dataset_tc), wall clock"},
        "gpu_launches": args.steps,  # one persistent tc_rotate_kernel per step (split fused)
        "roofline": roofline,
        "clocks": clocks,
    }

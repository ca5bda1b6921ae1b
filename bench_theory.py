"""verify_theory (bench.cpp:303-392), measured: every
(query, object) pair of config 1's data (100 000 x 128, 1 000 queries, K = 20)
gets a delta_d = 1 adaptive comparison per epsilon0 of an 8-point grid, on the
B200 through the public API (host arrays in, rows out; H2D of the rotated
dataset inside the timed call), next to the reference's own multi-threaded
verify_theory (oracle/_ref) on a bounded query sample of the same inputs, whose
rows must equal the GPU's rows for that sample exactly.
`python bench.py --mode theory`.
"""
from __future__ import annotations

import time

import numpy as np

GRID = [0.5, 1.0, 1.5, 2.0, 2.1, 2.5, 3.0, 4.0]


def run_theory(args, D):
    import os

    import paper_2303_09855_b200 as ads
    from paper_2303_09855_b200 import configs

    log = (lambda *a: print(*a, file=__import__("sys").stderr, flush=True)) if D.rank == 0 else (lambda *a: None)
    cfg = configs.CONFIGS[1]
    base, q = configs.generate(cfg)
    m = ads.generate_orthogonal(cfg.d, cfg.seed)
    t = ads.apply_dataset(m, base)
    qt = ads.apply_dataset(m, q)
    K = cfg.K
    for _ in range(args.warmup):
        ads.verify_theory(t, qt, K, GRID)
    from bench import ClockSampler

    clocks = ClockSampler(D.local)
    clocks.start()
    secs = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        rows = ads.verify_theory(t, qt, K, GRID)
        secs.append(time.perf_counter() - t0)
    clk = clocks.stop()
    sec = float(np.mean(secs))
    pairs = float(cfg.n) * qt.shape[0]
    res = {
        "metric": "verify_theory (query, object) delta_d=1 comparisons/s, 8-point epsilon0 grid",
        "value": pairs / sec, "unit": "pairs/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": "theory-cfg1-100k-d128", "n": cfg.n, "d": cfg.d, "nq": int(qt.shape[0]), "K": K,
                   "grid": GRID, "timing": "host API call (H2D of the dataset and queries inside)"},
        "rows": [r._asdict() for r in rows],
        "clocks": clk,
        "e2e": {"value": pairs / sec, "unit": "pairs/s", "h2d_bytes_per_step": int(t.nbytes + qt.nbytes),
                "d2h_bytes_per_step": 0},
        # per call: brute-force distances + select (one batch), kth distance, theory kernel
        "gpu_launches": 4 * args.steps,
    }
    from oracle import load_ref, ref_available

    if ref_available():
        ns = max(8, min(qt.shape[0], int(os.environ.get("ADS_THEORY_REF_Q", "100"))))
        t0 = time.perf_counter()
        eps, fr, ad, fails, pos = load_ref().verify_theory(t, qt[:ns], K, GRID)
        rsec = time.perf_counter() - t0
        sub = ads.verify_theory(t, qt[:ns], K, GRID)
        same = all((r.epsilon0, r.failure_rate, r.avg_dims, r.failures, r.positives) ==
                   (eps[g], fr[g], ad[g], int(fails[g]), int(pos[g])) for g, r in enumerate(sub))
        res["cpu_baseline"] = {"value": float(cfg.n) * ns / rsec, "unit": "pairs/s", "cores": os.cpu_count(),
                               "kind": "reference", "sample": f"first {ns} of {qt.shape[0]} queries, "
                               "adsann::verify_theory (parallel_chunks over queries)"}
        res["parity_with_reference_sample"] = bool(same)
        log(f"verify_theory: GPU {sec * 1e3:.1f} ms for {qt.shape[0]} queries; reference {rsec:.2f} s for {ns}; "
            f"rows identical on the sample: {same}")
    return res

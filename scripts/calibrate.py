"""Calibrate a config's within-component spread (BASELINE.md §3 rule): pick sigma
so FDScanning recall@K at the smallest swept nprobe lands in ~0.80-0.95.

    python scripts/calibrate.py --config 2 --sigmas 24 48 72 96 --nq 1000
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2303_09855_b200 as ads  # noqa: E402
from paper_2303_09855_b200 import configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--sigmas", type=float, nargs="+", required=True)
    ap.add_argument("--ranges", type=str, nargs="+", default=[""], help="lo:hi centre ranges")
    ap.add_argument("--nq", type=int, default=1000)
    ap.add_argument("--init", type=int, default=1)
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    for rg in args.ranges:
      for sigma in args.sigmas:
        cfg = configs.CONFIGS[args.config]
        cfg.sigma = sigma
        if rg:
            cfg.center_lo, cfg.center_hi = (float(v) for v in rg.split(":"))
        t0 = time.time()
        base, q = configs.generate(cfg, nq=args.nq)
        m = ads.generate_orthogonal(cfg.d, cfg.seed)
        t = ads.apply_dataset(m, base)
        t1 = time.time()
        idx = ads.build_ivf(base, t, m, cfg.nlist, cfg.seed, ads.IvfLayout.kSplit, 32,
                            max_iters=args.iters, init=args.init)
        t2 = time.time()
        gt = ads.brute_force_knn(base, q, cfg.K)
        t3 = time.time()
        row = {"range": rg, "sigma": sigma, "gen_s": round(t1 - t0, 1), "build_s": round(t2 - t1, 1),
               "gt_s": round(t3 - t2, 1)}
        sizes = np.diff(idx.export()["list_off"])
        row["list_sizes"] = [int(sizes.min()), float(sizes.mean()), int(sizes.max())]
        for np_ in cfg.sweep:
            fd = ads.ivf_query_batch(idx, None, q, cfg.K, np_, ads.IvfMode.kFd)
            ad = ads.ivf_query_batch(idx, None, q, cfg.K, np_, ads.IvfMode.kAdSplit)
            row[f"np{np_}"] = {"fd_recall": round(ads.recall_batch(fd.ids, gt, cfg.K), 4),
                               "ad_recall": round(ads.recall_batch(ad.ids, gt, cfg.K), 4),
                               "ad_dims_frac": round(float(ad.dims.sum()) / float(fd.dims.sum()), 4),
                               "cand": float(ad.candidates.mean())}
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()

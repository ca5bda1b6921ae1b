"""Same-box A/B of scan variants on one built index (bench.py's setup and measure):
python tools/ab_scan.py --config 5 --variants dense,nodense --steps 10 --reps 2"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--variants", default="dense,nodense")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    args = argparse.Namespace(config=a.config, nq=0, kmeans_iters=0, kmeans_init=-1, cfg_override="", step=0,
                              warps=0, query_order=2, ctas_per_sm=0, warmup=3, no_dense=False, walk=0)
    D = bench.Dist()
    log = lambda *x: print(*x, file=sys.stderr, flush=True)  # noqa: E731
    cfg = bench.config_for(args)
    S = bench.setup(cfg, D, log)
    out = []
    for rep in range(a.reps):
        for v in a.variants.split(","):
            # variant: comma-free tokens joined by '+', e.g. dense+step=512, nodense+warps=8
            args.no_dense = "nodense" in v
            args.step = int(v.split("step=")[1].split("+")[0]) if "step=" in v else 0
            args.warps = int(v.split("warps=")[1].split("+")[0]) if "warps=" in v else 0
            args.walk = 2 if "f32" in v else (1 if "exact" in v else 0)
            args.lag = -1 if "nolag" in v else (1 if "lag" in v else 0)
            M = bench.measure(S, cfg, cfg.nprobe, args, D, log, a.steps)
            row = {"variant": v, "rep": rep, "qps": M["value"], "scan_ms": M["stages_ms"]["scan"],
                   "frac": M["roofline"]["frac"], "sm_mhz": M["clocks"]["sm_mhz"],
                   "recall": M["recall_at_k"], "dims": M["dims_per_query"]}
            log(json.dumps(row))
            out.append(row)
    print(json.dumps({"config": cfg.key, "rows": out}))


if __name__ == "__main__":
    main()

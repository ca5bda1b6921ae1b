"""What list sharding costs at N ranks, measured on one GPU: the index is cut into
N list shards (LPT on list sizes, as bench.py's sharded path does) and each shard's
search, the work one rank would do, is run in turn on the same queries.  Reports
the scanned dims summed over shards (looser local thresholds inflate them) and the
slowest shard's scan time (the step's critical path), next to the unsharded search.
No rank waits on another, so one GPU measures each shard's work exactly.

    python tools/shard_inflation.py [config] [N ...] [walk=W]   (W: ads_search_opts.walk, 0 = engine's pick)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    import paper_2303_09855_b200 as ads
    from paper_2303_09855_b200 import configs
    from paper_2303_09855_b200.shard import partition_lists, shard_index

    argv = [a for a in sys.argv[1:] if not a.startswith("walk=")]
    walk = int(next((a.split("=")[1] for a in sys.argv[1:] if a.startswith("walk=")), 0))
    cfgid = int(argv[0]) if argv else 2
    ns = [int(v) for v in argv[1:]] or [2, 4, 8]
    cfg = configs.CONFIGS[cfgid]
    log = lambda *a: print(*a, file=sys.stderr, flush=True)  # noqa: E731
    S = bench.setup(cfg, bench.Dist(), log)
    ctx, q, idx = S["ctx"], S["q"], S["idx"]
    K, nprobe = cfg.K, cfg.nprobe
    opts = ads.search_opts(time_stages=True, walk=walk)
    print(f"walk option {walk} (engine's pick unsharded: {ads.search_plan(idx, K, nprobe, ads.IvfMode.kAdSplit, opts=opts)})")

    def run(index, reps=3):
        best, dims = None, None
        for _ in range(reps):
            ctx.flush_l2()
            r = ads.ivf_query_batch(index, None, q, K, nprobe, ads.IvfMode.kAdSplit, opts=opts)
            ms = float(index.last_timings()[3])
            best = ms if best is None else min(best, ms)
            dims = float(r.dims.astype(np.float64).sum())
        return best, dims

    base_ms, base_dims = run(idx)
    print(f"config {cfgid}: unsharded scan {base_ms:.2f} ms, dims {base_dims:.4g}")
    sizes = np.diff(idx.list_offsets())
    rows = []
    for n in ns:
        owner = partition_lists(sizes, n)
        shard_ms, shard_dims = [], []
        for rank in range(n):
            local = shard_index(idx, owner, rank)
            ms, dims = run(local)
            shard_ms.append(ms)
            shard_dims.append(dims)
            del local
        infl = sum(shard_dims) / base_dims
        crit = max(shard_ms)
        rows.append((n, infl, crit, base_ms / crit / n))
        print(f"N={n}: dims summed over shards x{infl:.3f} of unsharded; slowest shard scan {crit:.2f} ms "
              f"(unsharded {base_ms:.2f}); list-sharded weak-scaling efficiency on the scan "
              f"{base_ms / crit:.2f}/{n} = {base_ms / crit / n:.2f} of ideal")
        # two waves with the threshold exchange: probe ranks [0, w) on every shard, R = min over
        # shards of the wave-1 K-th distances (an upper bound on the global K-th distance), then
        # [w, nprobe) from r0 = R
        w = max(1, nprobe // 8)
        locals_ = [shard_index(idx, owner, rank) for rank in range(n)]
        print(f"N={n}: rank 0's plan {ads.search_plan(locals_[0], K, nprobe, ads.IvfMode.kAdSplit, opts=opts)}")
        w1 = []
        for loc in locals_:
            best = None
            for _ in range(3):
                ctx.flush_l2()
                r1 = ads.ivf_query_batch(loc, None, q, K, w, ads.IvfMode.kAdSplit, opts=opts)
                ms1 = float(loc.last_timings()[3])
                best = ms1 if best is None else min(best, ms1)
            w1.append((best, r1))
        kth = np.stack([np.where(r.counts == K, r.dists[:, K - 1], np.inf) for _, r in w1])
        R = np.nan_to_num(kth, nan=np.inf).min(axis=0)
        t2, d2 = [], []
        for (ms1, r1), loc in zip(w1, locals_):
            o2 = ads.search_opts(time_stages=True, probe_lo=w, r0=R, walk=walk)
            best = None
            for _ in range(3):
                ctx.flush_l2()
                r2 = ads.ivf_query_batch(loc, None, q, K, nprobe, ads.IvfMode.kAdSplit, opts=o2)
                ms2 = float(loc.last_timings()[3])
                best = ms2 if best is None else min(best, ms2)
            t2.append(ms1 + best)
            d2.append(float(r1.dims.astype(np.float64).sum()) + float(r2.dims.astype(np.float64).sum()))
        del locals_
        crit2 = max(t2)
        print(f"N={n} two waves (w={w}, R = min over shards): dims x{sum(d2) / base_dims:.3f}; slowest shard "
              f"scan {crit2:.2f} ms; efficiency {base_ms / crit2 / n:.2f} of ideal")
    return rows


if __name__ == "__main__":
    main()

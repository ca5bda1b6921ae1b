import sys; sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2303_09855_b200 as ads
from paper_2303_09855_b200 import configs
cfg = configs.CONFIGS[2]
base, q = configs.generate(cfg, nq=int(sys.argv[1]) if len(sys.argv) > 1 else 10000)
m = ads.generate_orthogonal(128, 0)
t = ads.apply_dataset(m, base)
idx = ads.build_ivf(base, t, m, 4096, 0, ads.IvfLayout.kSplit, 32, max_iters=3, init=1)
for qg in (1, 2, 8):
    o = ads.search_opts(first=1, step=8, scheduler=1, warps_per_cta=8, tile=64, queries_per_cta=qg, time_stages=True)
    r = ads.ivf_query_batch(idx, None, q, 100, 64, ads.IvfMode.kAdSplit, opts=o)
    print("qg", qg, "ok", float(r.dims.mean()), idx.last_timings(), flush=True)

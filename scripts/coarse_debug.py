import sys; sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2303_09855_b200 as ads
from paper_2303_09855_b200 import configs
cfg = configs.CONFIGS[int(sys.argv[1])]
base, q = configs.generate(cfg, nq=2000)
m = ads.generate_orthogonal(cfg.d, 0)
t = ads.apply_dataset(m, base)
idx = ads.build_ivf(base, t, m, cfg.nlist, 0, ads.IvfLayout.kSplit, 32, max_iters=3, init=1)
qt = ads.apply_dataset(m, q)
p = idx.probe_order(qt, 64)
print("done", p.shape, flush=True)

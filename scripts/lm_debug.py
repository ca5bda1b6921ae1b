import sys; sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import paper_2303_09855_b200 as eng
from oracle import load_oracle
from helpers import make_fixture, oracle_index, gpu_index
orc = load_oracle()
raw, t, qr, qt, P = make_fixture(orc, 500, 64, 4, 3, 1)
lay = oracle_index(orc, raw, t, P, 8, 2, d1=32)
idx = gpu_index(eng, lay, P)
o = eng.search_opts(first=1, step=1, scheduler=1, warps_per_cta=4, tile=64)
res = eng.ivf_query_batch(idx, qt, qr, 5, 3, eng.IvfMode.kAdSplit, opts=o)
print(res.ids)

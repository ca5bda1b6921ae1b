# How many centroids pass the certified prefilter (a <= T + 2E) under the fp32-FMA
# bound vs a 3xTF32 tensor-core bound (accumulation modelled as truncating, 3D terms).
import sys, numpy as np, torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2303_09855_b200 as ads
from paper_2303_09855_b200 import configs
cfgid = int(sys.argv[1])
cfg = configs.CONFIGS[cfgid]
import bench
ads_, ctx_, base, t, q, m, idx, gt = bench.setup(cfg, 0, 0, lambda *x: None)
exp = idx.export()
C = exp["centroids_t"].astype(np.float64)
qt = ads.apply_dataset(m, q).astype(np.float64)
mu = C.mean(0)
Cc = torch.tensor((C - mu).astype(np.float32), device="cuda")
Qc = torch.tensor((qt - mu).astype(np.float32), device="cuda")
cn2 = (Cc.double() ** 2).sum(1).float(); qn2 = (Qc.double() ** 2).sum(1).float()
torch.backends.cuda.matmul.allow_tf32 = False
approx = (qn2[:, None] + cn2[None, :] - 2 * (Qc @ Cc.T)).double()
D = C.shape[1]
s = Qc.double().norm(dim=1) + Cc.double().norm(dim=1).max()
nprobe = cfg.nprobe
T = approx.kthvalue(nprobe, dim=1).values
for name, u, terms, extra in (("fp32 FMA", 2.0**-24, D, 0.0), ("3xTF32 TC", 2.0**-23, 3 * D, 3 * 2.0**-22),
                              ("1xTF32 TC", 2.0**-23, D, 2 * 2.0**-11 + 2.0**-22),
                              ("1xBF16 TC", 2.0**-23, D, 2 * 2.0**-8 + 2.0**-16)):
    gamma = terms * u / (1 - terms * u) + 4 * 2.0**-24 + extra
    delta = 2 * 2.0**-24 * s
    E = 1.01 * (gamma * s * s + 2 * s * delta + delta * delta)
    n = (approx <= (T + 2 * E)[:, None]).sum(1).double()
    print(f"cfg{cfgid} {name}: gamma {gamma:.3e}, candidates/query mean {n.mean():.1f} p99 {n.quantile(0.99):.0f} max {n.max():.0f} (cap {4*nprobe+256})")

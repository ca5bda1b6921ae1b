"""Writes tests/golden/cfg5_centroids.npy: config 5's 16 384 IVF centroids, the
sampled k-means (seeded sample init, 10 Lloyd iterations, fp64 sums) of the GPU
engine over every 50th of the 1e8 rotated rows — exactly what
build_ivf_streamed trains for config 5.

Run on a B200 (python tests/golden/make_cfg5_centroids.py [out.npy]).  The bench's
reference arm builds its reference IvfIndex around these centroids (the k-means
itself would take hours of reference CPU time), and bench.py's GPU arm asserts on
every config-5 run that the centroids it trains are bit-identical to this file.
The k-means is pinned to the oracle's restatement (orc_kmeans_init) at small
sizes by tests/test_gpu_build_shard.py."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def train(cfg, ctx=None):
    import paper_2303_09855_b200 as ads
    from paper_2303_09855_b200 import configs

    ctx = ctx or ads.Context.default()
    m = ads.generate_orthogonal(cfg.d, cfg.seed)
    sample = cfg.extra["sample"]
    xs = configs.row_source(cfg)(0, sample, cfg.n // sample)
    dS = ads.DeviceArray.from_host(ctx, xs)
    dT = ads.DeviceArray(ctx, xs.shape, np.float32)
    ads.Transform(m, ctx).apply_dataset_device(dS, dT)
    b = ads.IvfBuilder(cfg.n, cfg.d, m, cfg.nlist, cfg.seed, 32, ctx)
    b.train_device(dT, cfg.kmeans_iters)
    return b.centroids()


if __name__ == "__main__":
    from paper_2303_09855_b200 import configs

    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "tests", "golden", "cfg5_centroids.npy")
    c = train(configs.CONFIGS[5])
    np.save(out, c)
    print(f"wrote {out}: {c.shape} float32")

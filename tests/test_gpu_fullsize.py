"""Parity at BASELINE.json's full sizes: config 2's 1 M x 128 index (4096 lists,
k-means++ + 25 Lloyd iterations) and config 3's 1 M x 960 index (8-warp CTAs,
30 segments per walk), built on the GPU, exported and searched by the C oracle
for a subset of queries, bit for bit: ids, distances and dims under the
engine's default batched refresh schedule, and under the reference's
per-candidate schedule (first = step = 1)."""
import numpy as np
import pytest

from helpers import MODE_ID

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.parametrize("cfgid,nq", [(2, 64), (3, 24)])
def test_full_size_vs_oracle(eng, orc, cfgid, nq):
    from paper_2303_09855_b200 import configs

    cfg = configs.CONFIGS[cfgid]
    base, q = configs.generate(cfg, nq=nq)
    m = eng.generate_orthogonal(cfg.d, cfg.seed)
    t = eng.apply_dataset(m, base)
    idx = eng.build_ivf(base, t, m, cfg.nlist, cfg.seed, eng.IvfLayout.kSplit, 32,
                        max_iters=cfg.kmeans_iters, init=cfg.kmeans_init)
    ex = idx.export()
    lay = {"n": cfg.n, "d": cfg.d, "k": cfg.nlist, "d1": 32, "split": True,
           "centroids_t": ex["centroids_t"], "centroids_raw": ex["centroids_raw"],
           "list_off": ex["list_off"], "ids_flat": ex["ids_flat"], "a1_t": ex["a1_t"], "a2_t": ex["a2_t"],
           "a1_raw": ex["a1_raw"], "a2_raw": ex["a2_raw"],
           # contiguous bucket-major copies (FD and the non-split modes read these)
           "vec_t": np.ascontiguousarray(np.hstack([ex["a1_t"], ex["a2_t"]])),
           "vec_raw": np.ascontiguousarray(np.hstack([ex["a1_raw"], ex["a2_raw"]]))}
    qt = eng.apply_dataset(m, q)
    K, nprobe = cfg.K, cfg.nprobe
    for mode in ("ad-split", "fd"):
        res = eng.ivf_query_batch(idx, qt, q, K, nprobe, eng.IvfMode(MODE_ID[mode]))
        plan = eng.search_plan(idx, K, nprobe, eng.IvfMode(MODE_ID[mode]))
        step, lag = plan["step"], (2 if plan["lag"] else 0)  # overlapped chunks == the oracle's lag 2
        for i in range(q.shape[0]):
            ids, dists, stats = orc.ivf_query(lay, qt[i], q[i], K, nprobe, mode, 2.1, 32, K, step, lag=lag)
            c = int(res.counts[i])
            assert c == len(ids)
            np.testing.assert_array_equal(res.ids[i, :c], ids, err_msg=f"{mode} q={i}")
            np.testing.assert_array_equal(res.dists[i, :c], dists, err_msg=f"{mode} q={i}")
            assert int(res.dims[i]) == int(stats[0]), (mode, i)
    ref = eng.ivf_query_batch(idx, qt[:8], q[:8], K, nprobe, eng.IvfMode.kAdSplit, first=1, step=1)
    for i in range(8):
        ids, dists, stats = orc.ivf_query(lay, qt[i], q[i], K, nprobe, "ad-split", 2.1, 32, 1, 1)
        np.testing.assert_array_equal(ref.ids[i, :len(ids)], ids)
        np.testing.assert_array_equal(ref.dists[i, :len(ids)], dists)
        assert int(ref.dims[i]) == int(stats[0])

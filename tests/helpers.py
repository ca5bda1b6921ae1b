"""Shared fixtures for the parity tests (test infrastructure)."""
import numpy as np

MODES = ("fd", "pd", "ad", "ad-split", "pd-split")
MODE_ID = {"fd": 0, "pd": 1, "ad": 2, "ad-split": 3, "pd-split": 4}


def make_fixture(orc, n, d, blobs, nq, seed, center_scale=10.0, sigma=1.0):
    """Gaussian blobs (numpy-seeded) + the reference's P; transformed by the oracle."""
    rng = np.random.default_rng(seed)
    centers = rng.normal(0.0, center_scale, (blobs, d))
    comp = rng.integers(0, blobs, n + nq)
    X = (centers[comp] + rng.normal(0.0, sigma, (n + nq, d))).astype(np.float32)
    raw, qr = X[:n].copy(), X[n:].copy()
    P = orc.generate_orthogonal(d, seed + 1)
    t = orc.apply_dataset(P, raw)
    qt = orc.apply_dataset(P, qr)
    return raw, t, qr, qt, P


def oracle_index(orc, raw, t, P, k, seed, d1=32, iters=10, split=True):
    cent, asg, _, _ = orc.kmeans(t, k, iters, seed)
    lay = orc.ivf_layout(raw, t, P, cent, asg, k, d1, split)
    lay["assignment"] = asg
    return lay


def gpu_index(ads, lay, P, with_raw=True):
    return ads.IvfIndex.from_arrays(
        n=lay["n"], d=lay["d"], k_clusters=lay["k"], d1=lay["d1"], layout=int(lay["split"]),
        centroids_t=lay["centroids_t"], list_off=lay["list_off"], ids_flat=lay["ids_flat"],
        vec_t=lay["vec_t"], a1_t=lay.get("a1_t"), a2_t=lay.get("a2_t"),
        centroids_raw=lay["centroids_raw"] if with_raw else None,
        vec_raw=lay["vec_raw"] if with_raw else None,
        a1_raw=lay.get("a1_raw") if with_raw else None,
        a2_raw=lay.get("a2_raw") if with_raw else None, P=P)


def assert_same_results(gpu_batch, orc, lay, qt, qr, K, nprobe, mode, eps0, dd, first, step):
    """GPU batch == oracle per query: ids, dists (bit-exact), dims, candidates."""
    for qi in range(qt.shape[0]):
        ids, dists, stats = orc.ivf_query(lay, qt[qi], qr[qi], K, nprobe, mode, eps0, dd, first, step)
        c = int(gpu_batch.counts[qi])
        assert c == len(ids), (mode, nprobe, qi, c, len(ids))
        np.testing.assert_array_equal(gpu_batch.ids[qi, :c], ids, err_msg=f"{mode} np={nprobe} q={qi}")
        np.testing.assert_array_equal(gpu_batch.dists[qi, :c], dists, err_msg=f"{mode} np={nprobe} q={qi}")
        assert int(gpu_batch.dims[qi]) == int(stats[0]), (mode, nprobe, qi, gpu_batch.dims[qi], stats[0])
        assert int(gpu_batch.candidates[qi]) == int(stats[2])

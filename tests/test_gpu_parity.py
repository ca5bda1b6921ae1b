"""GPU parity: the sm_100a kernels (through the C ABI) against the oracle.

The oracle is the C restatement pinned bit-for-bit to the reference
(test_oracle_pins.py).  Because the kernels use the reference's fp64
operation order, every comparison here is EXACT (decisions, dims,
distances, ids) — stricter than the north star's 1e-5 boundary band.
"""
import math

import numpy as np
import pytest

from helpers import MODES, MODE_ID, assert_same_results, gpu_index, make_fixture, oracle_index

pytestmark = pytest.mark.gpu


# ------------------------------------------------------------------ transform
@pytest.mark.parametrize("d,n", [(1, 5), (7, 33), (64, 1000), (128, 517), (200, 64), (960, 700), (30, 2049),
                                 (96, 1300)])
def test_apply_dataset_bitexact(eng, orc, d, n):
    """Tile edges in both dimensions (D not a multiple of the 64-row tile or the
    32-column stage, ragged vector counts) and apply_transpose over a dataset."""
    rng = np.random.default_rng(d * 7 + n)
    X = rng.normal(0, 3, (n, d)).astype(np.float32)
    m = eng.generate_orthogonal(d, 11)
    assert np.array_equal(m.entries, orc.generate_orthogonal(d, 11))
    Y = eng.apply_dataset(m, X)
    np.testing.assert_array_equal(Y, orc.apply_dataset(m.entries, X))
    yt = eng.apply_transpose(m, X[0])
    np.testing.assert_array_equal(yt, orc.apply_transpose(m.entries, X[0]))
    np.testing.assert_array_equal(eng.apply_prefix(m, X[1], d // 2),
                                  orc.apply_prefix(m.entries, X[1], d // 2))
    if n >= 512:  # apply_transpose over a whole dataset (the same kernels on P^T)
        yT = eng.Transform(m).apply_transpose_dataset(X)
        for i in range(0, n, max(1, n // 17)):
            np.testing.assert_array_equal(yT[i], orc.apply_transpose(m.entries, X[i]))


# ------------------------------------------------------------------ fixed-threshold DCOs
@pytest.mark.parametrize("D,dd,eps,kind", [
    (128, 32, 2.1, "ad"), (256, 32, 2.1, "ad"), (96, 32, 2.1, "ad"), (960, 32, 2.1, "ad"),
    (128, 16, 1.5, "ad"), (48, 48, 2.1, "ad"), (100, 20, 2.1, "ad"),   # partial last block
    (30, 7, 2.0, "ad"), (161, 1, 0.7, "ad"), (13, 13, 1e6, "ad"),      # 4-byte gather path
    (128, 32, 2.1, "pd"), (40, 9, 2.1, "pd"), (64, 32, 2.1, "fd"), (33, 1, 2.1, "fd"),
])
def test_dco_fixed_bitexact(eng, orc, D, dd, eps, kind):
    rng = np.random.default_rng(D * 1000 + dd)
    n, nq, per = 700, 9, 300
    X = rng.normal(0, 1, (n, D)).astype(np.float32)
    Q = rng.normal(0, 1, (nq, D)).astype(np.float32)
    rows = rng.integers(0, n, nq * per).astype(np.int64)
    off = np.arange(0, nq * per + 1, per, dtype=np.int64)
    # thresholds around the typical distance so decisions are mixed; include r=0 and r=inf
    r = np.sqrt(2.0 * D) * rng.uniform(0.7, 1.05, nq)
    r[0] = 0.0
    r[1] = math.inf
    cfg = eng.DcoConfig(eps, dd)
    res = eng.dco_fixed(X, Q, r, cand_off=off, cand_rows=rows, kind=kind, cfg=cfg)
    qidx = np.repeat(np.arange(nq, dtype=np.int32), per)
    pos, dims, dsq, obs = orc.ad_scan_pairs(X, Q, rows, qidx, np.repeat(r, per), eps, dd,
                                            pd_mode=(kind == "pd"))
    if kind == "fd":  # l2_sq + sqrt(s) <= r (dco.cpp:70-81)
        s = np.array([orc.scan_kernel(1, X[rw], Q[q], D, 0, 0.0, math.inf, eps, D, False)[1]
                      for rw, q in zip(rows, qidx)])
        obs = np.sqrt(s)
        pos = (obs <= np.repeat(r, per)).astype(np.uint8)
        dims = np.full(len(rows), D, np.int32)
        dsq = np.where(pos == 1, s, np.nan)
    np.testing.assert_array_equal(res.positive.astype(np.uint8), pos)
    np.testing.assert_array_equal(res.dims, dims)
    np.testing.assert_array_equal(res.observed, obs)
    np.testing.assert_array_equal(np.isnan(res.dist_sq), np.isnan(dsq))
    ok = ~np.isnan(dsq)
    np.testing.assert_array_equal(res.dist_sq[ok], dsq[ok])
    per_q = dims.reshape(nq, per).sum(axis=1).astype(np.uint64)
    np.testing.assert_array_equal(res.dims_per_query, per_q)


def test_dco_fixed_windows(eng, orc):
    """Config-4 style windows (wrapping row ranges) == explicit rows."""
    rng = np.random.default_rng(5)
    n, D, nq, win = 5000, 256, 6, 1777
    X = rng.normal(0, 1, (n, D)).astype(np.float32)
    Q = rng.normal(0, 1, (nq, D)).astype(np.float32)
    start = rng.integers(0, n, nq).astype(np.int64)
    r = np.full(nq, np.sqrt(2 * D) * 0.93)
    a = eng.dco_fixed(X, Q, r, win_start=start, win_len=win)
    rows = ((start[:, None] + np.arange(win)[None, :]) % n).reshape(-1)
    qidx = np.repeat(np.arange(nq, dtype=np.int32), win)
    pos, dims, dsq, obs = orc.ad_scan_pairs(X, Q, rows, qidx, np.repeat(r, win), 2.1, 32)
    np.testing.assert_array_equal(a.positive.astype(np.uint8), pos)
    np.testing.assert_array_equal(a.dims, dims)
    np.testing.assert_array_equal(a.observed, obs)


def test_single_dco_kats(eng, orc):
    """test_dco.cpp KATs through the validated single-DCO API."""
    o, q = [3.0, 4.0], [0.0, 0.0]
    hit = eng.fd_scan(o, q, 5.0)
    assert hit.positive and hit.distance == 5.0 and hit.dims_used == 2
    miss = eng.fd_scan(o, q, 4.9)
    assert not miss.positive and miss.distance is None and miss.observed == 5.0
    pd = eng.pd_scan(o, q, 2.0, 1)
    assert not pd.positive and pd.dims_used == 1 and pd.observed == 3.0
    m = eng.generate_orthogonal(64, 19)
    rng = np.random.default_rng(23)
    a = eng.apply(m, rng.normal(size=64))
    b = eng.apply(m, rng.normal(size=64))
    z = eng.ad_sampling(a, b, 0.0, eng.DcoConfig(2.1, 16))
    assert not z.positive and z.dims_used == 16
    s = eng.ad_sampling(a, a, 0.0, eng.DcoConfig(2.1, 16))
    assert s.positive and s.distance == 0.0 and s.dims_used == 64
    for kind, args in (("ad", (2.1, 16)), ("pd", (2.1, 8)), ("fd", (2.1, 1))):
        for r in (0.0, 3.0, 11.3, 50.0):
            out = {"ad": lambda: eng.ad_sampling(a, b, r, eng.DcoConfig(*args)),
                   "pd": lambda: eng.pd_scan(a, b, r, args[1]),
                   "fd": lambda: eng.fd_scan(a, b, r)}[kind]()
            exp = orc.dco(kind, a, b, r, *args)
            assert (out.positive, out.distance, out.observed, out.dims_used) == exp
    with pytest.raises(ValueError):
        eng.fd_scan([1.0, 2.0], [1.0], 1.0)
    with pytest.raises(ValueError):
        eng.fd_scan([1.0, 2.0], [1.0, 2.0], -1.0)
    with pytest.raises(ValueError):
        eng.pd_scan([1.0, 2.0], [1.0, 2.0], 1.0, 3)
    with pytest.raises(ValueError):
        eng.ad_sampling([1.0, 2.0], [1.0, 2.0], 1.0, eng.DcoConfig(0.0, 1))
    with pytest.raises(ValueError):
        eng.ad_sampling([1.0, 2.0], [1.0, 2.0], 1.0, eng.DcoConfig(2.1, 0))


# ------------------------------------------------------------------ IVF search
CASES = [
    # n, d, blobs, k, d1, dd, K
    (2000, 64, 16, 40, 32, 32, 10),
    (3000, 128, 32, 50, 32, 32, 20),
    (1500, 48, 8, 20, 16, 16, 5),     # persistence-test shape
    (1200, 30, 8, 12, 10, 7, 7),      # unaligned -> 4-byte gathers
    (1000, 96, 8, 16, 40, 24, 9),     # d1 != delta_d
]


@pytest.mark.parametrize("case", CASES)
def test_ivf_reference_schedule_bitexact(eng, orc, case):
    """first=step=1 (r re-read before every candidate) == adsann::ivf_query exactly."""
    n, d, blobs, k, d1, dd, K = case
    raw, t, qr, qt, P = make_fixture(orc, n, d, blobs, 25, 57 + d)
    lay = oracle_index(orc, raw, t, P, k, 59, d1=d1)
    idx = gpu_index(eng, lay, P)
    cfg = eng.DcoConfig(2.1, dd)
    for mode in MODES:
        for nprobe in (1, 5, k):
            res = eng.ivf_query_batch(idx, qt, qr, K, nprobe, eng.IvfMode(MODE_ID[mode]), cfg,
                                      first=1, step=1)
            assert_same_results(res, orc, lay, qt, qr, K, nprobe, mode, 2.1, dd, 1, 1)


@pytest.mark.parametrize("eps,dd", [(0.5, 32), (4.0, 32), (1e6, 32), (2.1, 64), (2.1, 8), (0.2, 16)])
def test_ivf_epsilon_and_delta_d(eng, orc, eps, dd):
    """ADSampling knobs beyond the defaults (dco.cpp:32-37: eps0 > 0, 1 <= delta_d <= D):
    a tight eps0 (many rejections), a loose one, eps0 = 1e6 (never rejects,
    test_dco.cpp:166-178), and delta_d below / above d1, in both refresh schedules."""
    raw, t, qr, qt, P = make_fixture(orc, 3000, 128, 24, 21, 301)
    lay = oracle_index(orc, raw, t, P, 30, 302, d1=32)
    idx = gpu_index(eng, lay, P)
    cfg = eng.DcoConfig(eps, dd)
    for mode in ("ad-split", "ad"):
        for first, step in ((1, 1), (10, 256)):
            res = eng.ivf_query_batch(idx, qt, qr, 10, 6, eng.IvfMode(MODE_ID[mode]), cfg, first=first, step=step)
            assert_same_results(res, orc, lay, qt, qr, 10, 6, mode, eps, dd, first, step)


@pytest.mark.parametrize("first,step", [(0, 256), (0, 64), (1, 1000), (37, 5)])
def test_ivf_batched_schedule_bitexact(eng, orc, first, step):
    """Batched threshold refresh == the oracle's same schedule, bit for bit."""
    raw, t, qr, qt, P = make_fixture(orc, 4000, 64, 16, 40, 91)
    lay = oracle_index(orc, raw, t, P, 50, 93, d1=32)
    idx = gpu_index(eng, lay, P)
    K = 10
    for mode in ("ad-split", "ad", "pd-split", "fd"):
        for nprobe in (3, 17):
            res = eng.ivf_query_batch(idx, qt, qr, K, nprobe, eng.IvfMode(MODE_ID[mode]),
                                      eng.DcoConfig(), first=first, step=step)
            f = first if first > 0 else K
            assert_same_results(res, orc, lay, qt, qr, K, nprobe, mode, 2.1, 32, f, step)


@pytest.mark.parametrize("K,first,step", [(10, 0, 256), (10, 1, 1), (25, 0, 16), (7, 3, 5)])
def test_ivf_duplicate_vectors_ties(eng, orc, K, first, step):
    """Exact duplicates (equal distances, distinct ids) drive the top-K's tie
    rules (strict '<' at the max, (dist, id) pop order) through both the
    CTA-wide rank merge and its sequential fallback."""
    raw, t, qr, qt, P = make_fixture(orc, 1200, 64, 8, 30, 401)
    rng = np.random.default_rng(402)
    src = rng.integers(0, 1200, 1800)
    raw = np.concatenate([raw, raw[src], raw[src[:300]]]).astype(np.float32)  # 1-3 copies
    t = orc.apply_dataset(P, raw)
    qr = np.concatenate([qr, raw[src[:10]]]).astype(np.float32)  # queries on duplicated points
    qt = orc.apply_dataset(P, qr)
    lay = oracle_index(orc, raw, t, P, 24, 403, d1=32)
    idx = gpu_index(eng, lay, P)
    for mode in ("ad-split", "fd", "pd"):
        for nprobe in (2, 9, 24):
            res = eng.ivf_query_batch(idx, qt, qr, K, nprobe, eng.IvfMode(MODE_ID[mode]),
                                      eng.DcoConfig(), first=first, step=step)
            f = first if first > 0 else K
            assert_same_results(res, orc, lay, qt, qr, K, nprobe, mode, 2.1, 32, f, step)


def test_ivf_rotation_on_device(eng, orc):
    """Q_t omitted -> queries rotated on the GPU with P: rotate_mode 0 (exact fp64) gives
    results identical to the oracle-rotated queries; the default (2) rotates batches of
    >= 64 queries on the tensor cores (== rotate_mode 1) and small batches exactly."""
    raw, t, qr, qt, P = make_fixture(orc, 2000, 64, 16, 80, 7)
    lay = oracle_index(orc, raw, t, P, 30, 8, d1=32)
    idx = gpu_index(eng, lay, P)
    b = eng.ivf_query_batch(idx, qt, qr, 10, 6, eng.IvfMode.kAdSplit)
    a = eng.ivf_query_batch(idx, None, qr, 10, 6, eng.IvfMode.kAdSplit, opts=eng.search_opts(rotate_mode=0))
    np.testing.assert_array_equal(a.ids, b.ids)
    np.testing.assert_array_equal(a.dists, b.dists)
    np.testing.assert_array_equal(a.dims, b.dims)
    small = eng.ivf_query_batch(idx, None, qr[:30], 10, 6, eng.IvfMode.kAdSplit)  # < 64: exact
    np.testing.assert_array_equal(small.ids, b.ids[:30])
    np.testing.assert_array_equal(small.dists, b.dists[:30])
    dflt = eng.ivf_query_batch(idx, None, qr, 10, 6, eng.IvfMode.kAdSplit)
    tc = eng.ivf_query_batch(idx, None, qr, 10, 6, eng.IvfMode.kAdSplit, opts=eng.search_opts(rotate_mode=1))
    np.testing.assert_array_equal(dflt.ids, tc.ids)
    np.testing.assert_array_equal(dflt.dists, tc.dists)
    np.testing.assert_array_equal(dflt.dims, tc.dims)
    # within the north star's tolerance of the exact rotation's distances
    m = np.isfinite(dflt.dists) & np.isfinite(b.dists) & (dflt.ids == b.ids)
    assert np.all(np.abs(dflt.dists[m] - b.dists[m]) <= 1e-5 * np.abs(b.dists[m]) + 1e-12)


def test_probe_order_bitexact(eng, orc):
    raw, t, qr, qt, P = make_fixture(orc, 3000, 64, 8, 40, 3)
    lay = oracle_index(orc, raw, t, P, 300, 4, d1=32, iters=3)
    idx = gpu_index(eng, lay, P)
    for nprobe in (1, 7, 64, 300):
        got = idx.probe_order(qt, nprobe, transformed=True)
        for qi in range(qt.shape[0]):
            np.testing.assert_array_equal(got[qi], orc.probe_order(lay["centroids_t"], qt[qi], nprobe))
    got = idx.probe_order(qr, 9, transformed=False)
    for qi in range(qr.shape[0]):
        np.testing.assert_array_equal(got[qi], orc.probe_order(lay["centroids_raw"], qr[qi], 9))


def test_ivf_validation(eng, orc):
    raw, t, qr, qt, P = make_fixture(orc, 100, 8, 2, 1, 73)
    lay = oracle_index(orc, raw, t, P, 5, 75, split=False)
    idx = gpu_index(eng, lay, P)
    M = eng.IvfMode
    with pytest.raises(ValueError):
        eng.ivf_query(idx, None, qr[0], 0, 1, M.kFd)
    with pytest.raises(ValueError):
        eng.ivf_query(idx, None, qr[0], 1, 0, M.kFd)
    with pytest.raises(ValueError):
        eng.ivf_query(idx, None, qr[0], 1, 6, M.kFd)
    with pytest.raises(ValueError):
        eng.ivf_query(idx, None, qr[0], 1, 1, M.kAdSplit)
    idx_noP = eng.IvfIndex.from_arrays(n=lay["n"], d=lay["d"], k_clusters=lay["k"], d1=lay["d1"],
                                       layout=0, centroids_t=lay["centroids_t"],
                                       list_off=lay["list_off"], ids_flat=lay["ids_flat"],
                                       vec_t=lay["vec_t"])
    with pytest.raises(ValueError):
        eng.ivf_query(idx_noP, None, qr[0], 1, 1, M.kAd)


# ------------------------------------------------------------------ build side
@pytest.mark.parametrize("n,d,k,iters,seed", [(500, 12, 10, 25, 21), (20, 8, 20, 25, 7),
                                               (100, 6, 1, 25, 9), (3000, 64, 37, 10, 5)])
def test_kmeans_bitexact(eng, orc, n, d, k, iters, seed):
    rng = np.random.default_rng(seed)
    X = rng.normal(0, 3, (n, d)).astype(np.float32)
    got = eng.kmeans(X, k, iters, seed)
    cent, asg, obj, it = orc.kmeans(X, k, iters, seed)
    np.testing.assert_array_equal(got.centroids, cent)
    np.testing.assert_array_equal(got.assignment, asg)
    assert got.objective == obj and got.iterations == it


def test_build_ivf_matches_reference_layout(eng, orc):
    raw, t, qr, qt, P = make_fixture(orc, 2500, 32, 8, 10, 45)
    m = eng.TransformMatrix(32, 46, P)
    idx = eng.build_ivf(raw, t, m, 20, 47, eng.IvfLayout.kSplit, 8, max_iters=25)
    ex = idx.export()
    cent, asg, _, _ = orc.kmeans(t, 20, 25, 47)
    lay = orc.ivf_layout(raw, t, P, cent, asg, 20, 8, True)
    for nm in ("centroids_t", "centroids_raw", "list_off", "ids_flat", "a1_t", "a2_t", "a1_raw", "a2_raw"):
        np.testing.assert_array_equal(ex[nm], lay[nm], err_msg=nm)
    with pytest.raises(ValueError):
        eng.build_ivf(raw, t, m, 20, 1, eng.IvfLayout.kSplit, 0)
    with pytest.raises(ValueError):
        eng.build_ivf(raw, t, m, 20, 1, eng.IvfLayout.kSplit, 32)


@pytest.mark.parametrize("n,d,nq,K", [(3000, 64, 30, 10), (500, 17, 5, 500), (2000, 128, 12, 100)])
def test_brute_force_knn_bitexact(eng, orc, n, d, nq, K):
    rng = np.random.default_rng(n + d)
    base = rng.normal(0, 1, (n, d)).astype(np.float32)
    base[7] = base[3]  # exact duplicate -> tie broken by id
    q = rng.normal(0, 1, (nq, d)).astype(np.float32)
    q[0] = base[3]
    np.testing.assert_array_equal(eng.brute_force_knn(base, q, K), orc.brute_force_knn(base, q, K))
    with pytest.raises(ValueError):
        eng.brute_force_knn(base, q, n + 1)


def test_ivf_scheduler_1_is_rejected(eng, orc):
    """The list-major scheduler was removed (slower than query-major)."""
    raw, t, qr, qt, P = make_fixture(orc, 500, 32, 4, 4, 5)
    lay = oracle_index(orc, raw, t, P, 8, 6, d1=16)
    idx = gpu_index(eng, lay, P)
    with pytest.raises(ValueError):
        eng.ivf_query_batch(idx, qt, qr, 5, 2, eng.IvfMode.kAdSplit, opts=eng.search_opts(scheduler=1))


def test_coarse_prefilter_adversarial_ties(eng, orc):
    """Certified prefilter == exact probe_order with exact and near-duplicate centroids."""
    rng = np.random.default_rng(12)
    d, L = 96, 300
    base = rng.normal(0, 1, (L, d)).astype(np.float32)
    base[1] = base[0]                              # exact duplicate centroid
    base[2] = base[0] + np.float32(1e-6)           # near duplicates
    base[3] = np.nextafter(base[0], np.float32(np.inf))
    base[10:20] = base[9]                          # a block of identical centroids
    n = L  # one point per list: point i == centroid i
    P = orc.generate_orthogonal(d, 3)
    lay = {"n": n, "d": d, "k": L, "d1": 32, "split": True, "centroids_t": base,
           "centroids_raw": base, "list_off": np.arange(L + 1, dtype=np.int64),
           "ids_flat": np.arange(n, dtype=np.int32), "vec_t": base, "vec_raw": base,
           "a1_t": base[:, :32].copy(), "a2_t": base[:, 32:].copy(), "a1_raw": base[:, :32].copy(),
           "a2_raw": base[:, 32:].copy()}
    idx = gpu_index(eng, lay, P)
    Q = np.concatenate([base[:12] + rng.normal(0, 1e-7, (12, d)).astype(np.float32),
                        rng.normal(0, 1, (20, d)).astype(np.float32)])
    for nprobe in (1, 2, 3, 5, 13, 64, L):
        got = idx.probe_order(Q, nprobe)
        for qi in range(Q.shape[0]):
            np.testing.assert_array_equal(got[qi], orc.probe_order(base, Q[qi], nprobe))
    a = eng.ivf_query_batch(idx, Q, Q, 5, 13, eng.IvfMode.kAdSplit, opts=eng.search_opts(coarse_mode=0))
    b = eng.ivf_query_batch(idx, Q, Q, 5, 13, eng.IvfMode.kAdSplit, opts=eng.search_opts(coarse_mode=1))
    np.testing.assert_array_equal(a.ids, b.ids)
    np.testing.assert_array_equal(a.dims, b.dims)


@pytest.mark.parametrize("d,L,nprobe", [(128, 512, 16), (96, 300, 64), (960, 256, 32), (30, 200, 8)])
def test_coarse_prefilter_gemm_paths(eng, orc, d, L, nprobe):
    """The tcgen05 TF32 prefilter (default; fp32 FMA when d % 4 != 0), the fp32-FMA
    prefilter (coarse_mode 2) and exact scoring (coarse_mode 1) give the same probes;
    the certified window stays tight (a wrong GEMM would show up here as many
    rescored centroids or fallbacks, which the exact fallback would otherwise hide)."""
    raw, t, qr, qt, P = make_fixture(orc, 6 * L, d, 64, 300, 5 + d, center_scale=3.0)
    lay = oracle_index(orc, raw, t, P, L, 7, d1=32 if d > 32 else 16, iters=4)
    idx = gpu_index(eng, lay, P)
    res = {}
    for mode in (0, 2, 1):
        r = eng.ivf_query_batch(idx, qt, qr, 10, nprobe, eng.IvfMode.kAdSplit,
                                eng.DcoConfig(2.1, min(32, d)), opts=eng.search_opts(coarse_mode=mode))
        res[mode] = r
        if mode != 1:
            st = idx.coarse_stats()
            assert st["queries"] == qt.shape[0] and st["fallbacks"] == 0, (mode, st)
            assert st["rescored"] <= qt.shape[0] * (3 * nprobe + 16), (mode, st)
    for mode in (0, 2):
        np.testing.assert_array_equal(res[mode].ids, res[1].ids)
        np.testing.assert_array_equal(res[mode].dims, res[1].dims)
    got = idx.probe_order(qt, nprobe)
    for qi in range(0, qt.shape[0], 37):
        np.testing.assert_array_equal(got[qi], orc.probe_order(lay["centroids_t"], qt[qi], nprobe))


@pytest.mark.parametrize("n,d", [(1000, 128), (777, 960), (300, 96), (129, 32), (5000, 256), (70000, 128)])
def test_transform_tensor_cores(eng, orc, n, d):
    """apply_dataset_tc (tcgen05 3xTF32) vs the exact fp64 rotation: elementwise
    within 1e-6 |x| (SURVEY §8c's transform budget) up to D = 256 and 2e-6 |x| at
    D = 960 (fp32 tensor-core accumulation over 3 D products; measured max 1.24e-6),
    norms preserved to 1e-5."""
    rng = np.random.default_rng(d + n)
    X = rng.normal(0, 3, (n, d)).astype(np.float32)
    m = eng.generate_orthogonal(d, 5)
    exact = orc.apply_dataset(m.entries, X).astype(np.float64)
    tc = eng.apply_dataset_tc(m, X).astype(np.float64)
    xn = np.linalg.norm(X.astype(np.float64), axis=1)
    err = np.abs(tc - exact).max(axis=1) / xn
    assert err.max() <= (1e-6 if d <= 256 else 2e-6), err.max()
    np.testing.assert_allclose(np.linalg.norm(tc, axis=1), xn, rtol=1e-5)
    with pytest.raises(ValueError):
        eng.apply_dataset_tc(eng.generate_orthogonal(6, 1), rng.normal(size=(3, 6)).astype(np.float32))


def test_tc_rotation_kernels_agree(eng, tmp_path):
    """The persistent tcgen05 rotation with the TF32 split fused (default) is bit-identical
    to the first tiled kernel on a pre-split X (ADS_TC_ROTATE=0, run in a subprocess):
    same products, same K order, same cvt.rna split; shapes cover every N-tile width
    (96, 128, 192, 256, and the D = 32 fallback) and row tails."""
    import os
    import subprocess
    import sys

    shapes = [(300, 96), (1000, 128), (129, 32), (777, 960), (5000, 256), (1, 960), (4099, 192)]
    code = (
        "import sys, numpy as np\n"
        f"sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})\n"
        "import paper_2303_09855_b200 as ads\n"
        "out = {}\n"
        f"for n, d in {shapes!r}:\n"
        "    X = np.random.default_rng(n + d).normal(0, 3, (n, d)).astype(np.float32)\n"
        "    out[f'{n}x{d}'] = ads.apply_dataset_tc(ads.generate_orthogonal(d, 5), X)\n"
        f"np.savez({str(tmp_path / 'tiled.npz')!r}, **out)\n")
    env = dict(os.environ, ADS_TC_ROTATE="0")
    subprocess.run([sys.executable, "-c", code], env=env, check=True, timeout=600)
    ref = np.load(tmp_path / "tiled.npz")
    for n, d in shapes:
        X = np.random.default_rng(n + d).normal(0, 3, (n, d)).astype(np.float32)
        got = eng.apply_dataset_tc(eng.generate_orthogonal(d, 5), X)
        np.testing.assert_array_equal(got, ref[f"{n}x{d}"], err_msg=f"{n}x{d}")


def test_ivf_tensor_core_query_rotation(eng, orc):
    """rotate_mode 1 (queries rotated by the 3xTF32 tensor-core transform on the GPU)
    == the oracle run on the same TC-rotated queries, bit for bit."""
    raw, t, qr, qt, P = make_fixture(orc, 3000, 128, 16, 40, 77)
    lay = oracle_index(orc, raw, t, P, 40, 78, d1=32)
    idx = gpu_index(eng, lay, P)
    m = eng.TransformMatrix(128, 0, np.asarray(P, np.float64))
    qt_tc = eng.apply_dataset_tc(m, qr)
    assert not np.array_equal(qt_tc, qt)  # a different (fp32-accurate) rotation
    for mode in ("ad-split", "ad"):
        res = eng.ivf_query_batch(idx, None, qr, 10, 7, eng.IvfMode(MODE_ID[mode]),
                                  opts=eng.search_opts(rotate_mode=1))
        assert_same_results(res, orc, lay, qt_tc, qr, 10, 7, mode, 2.1, 32, 10, 256)


@pytest.mark.parametrize("n,d,nq,K,grid", [(1500, 48, 12, 20, [1e6]),
                                           (2000, 64, 10, 50, [2.5, 0.5, 1.0, 2.0, 1.5, 3.0]),
                                           (800, 30, 7, 1, [2.1, 2.1, 0.2]),
                                           (3000, 128, 20, 100, [0.3, 1.0, 2.1, 4.0])])
def test_verify_theory_bitexact(eng, orc, n, d, nq, K, grid):
    """verify_theory (bench.cpp:303-392) on the GPU == the oracle: counts exact,
    ratios bit-identical (formed like the reference)."""
    _, t, _, qt, _ = make_fixture(orc, n, d, 8, nq, 31 + d)
    if n == 3000:  # duplicated rows: ties at the K-th distance
        t = np.concatenate([t, t[:400]]).astype(np.float32)
    rows = eng.verify_theory(t, qt, K, grid)
    eps, fr, ad, fails, pos = orc.verify_theory(t, qt, K, grid)
    assert len(rows) == len(grid)
    for g, r in enumerate(rows):
        assert (r.epsilon0, r.failures, r.positives) == (eps[g], int(fails[g]), int(pos[g])), g
        assert r.failure_rate == fr[g] and r.avg_dims == ad[g], g
    with pytest.raises(ValueError):
        eng.verify_theory(t, qt, 0, grid)
    with pytest.raises(ValueError):
        eng.verify_theory(t, qt, t.shape[0] + 1, grid)
    with pytest.raises(ValueError):
        eng.verify_theory(t, qt, K, [0.0])


@pytest.mark.parametrize("K", [200, 256, 300, 1000])
def test_ivf_large_k_merge_paths(eng, orc, K):
    """K = 200 / 256 fit the CTA rank merge (heap <= 2 x blockDim), 300 / 1000 take
    the one-warp sequential offers; all bit-exact, including partial (count < K) results."""
    raw, t, qr, qt, P = make_fixture(orc, 4000, 64, 16, 12, 91 + K)
    lay = oracle_index(orc, raw, t, P, 30, 93, d1=32)
    idx = gpu_index(eng, lay, P)
    for mode in ("ad-split", "fd"):
        for nprobe in (2, 11, 30):
            res = eng.ivf_query_batch(idx, qt, qr, K, nprobe, eng.IvfMode(MODE_ID[mode]), first=0, step=128)
            assert_same_results(res, orc, lay, qt, qr, K, nprobe, mode, 2.1, 32, K, 128)


def test_ivf_empty_lists_and_empty_streams(eng, orc):
    """Many empty lists (k close to n): queries whose probed lists hold nothing
    return count 0 (ids -1, NaN dists); the rest stay bit-exact."""
    raw, t, qr, qt, P = make_fixture(orc, 150, 32, 4, 20, 5)
    k = 120
    cent = t[:k].copy()
    asg = np.zeros(150, np.int32)  # everything in 3 lists, 117 lists empty
    asg[50:100] = 1
    asg[100:] = 2
    lay = orc.ivf_layout(raw, t, P, cent, asg, k, 16, True)
    idx = gpu_index(eng, lay, P)
    for nprobe in (1, 3, 40, k):
        res = eng.ivf_query_batch(idx, qt, qr, 5, nprobe, eng.IvfMode.kAdSplit, eng.DcoConfig(2.1, 16))
        assert_same_results(res, orc, lay, qt, qr, 5, nprobe, "ad-split", 2.1, 16, 5, 256)
        empty = res.counts == 0
        if nprobe == 1:
            assert empty.any()
        assert (res.ids[empty] == -1).all() and np.isnan(res.dists[empty]).all()


def test_ivf_query_order_invariant(eng, orc):
    """The order in which a batch's queries are served (input, L2 chain, longest first
    (the default)) changes nothing: ids, dists, dims and candidates are identical, and
    the default order matches the oracle."""
    raw, t, qr, qt, P = make_fixture(orc, 6000, 96, 24, 61, 91)
    lay = oracle_index(orc, raw, t, P, 48, 92, d1=32)
    idx = gpu_index(eng, lay, P)
    res = {qo: eng.ivf_query_batch(idx, qt, qr, 10, 9, eng.IvfMode.kAdSplit, opts=eng.search_opts(query_order=qo))
           for qo in (0, 1, 2)}
    for qo in (1, 2):
        for f in ("ids", "dists", "counts", "dims", "candidates"):
            np.testing.assert_array_equal(getattr(res[qo], f), getattr(res[0], f), err_msg=f"order {qo} {f}")
    assert_same_results(res[2], orc, lay, qt, qr, 10, 9, "ad-split", 2.1, 32, 10, 256)


@pytest.mark.parametrize("probe_lo,rscale", [(0, 1.0), (3, 1.0), (3, 0.5), (5, 2.0), (17, 1.3), (0, 0.0)])
def test_ivf_probe_range_and_initial_radius(eng, orc, probe_lo, rscale):
    """probe_lo / r0 (the sharded search's second wave): only probe ranks
    [probe_lo, nprobe) are scanned and r starts at r0[q] == the oracle, bit for bit."""
    raw, t, qr, qt, P = make_fixture(orc, 4000, 64, 16, 30, 191)
    lay = oracle_index(orc, raw, t, P, 40, 193, d1=32)
    idx = gpu_index(eng, lay, P)
    K, nprobe = 10, 17
    full = eng.ivf_query_batch(idx, qt, qr, K, nprobe, eng.IvfMode.kAdSplit, first=0, step=64)
    r0 = np.where(full.counts == K, full.dists[:, K - 1], np.inf) * rscale
    r0 = np.where(np.isnan(r0), np.inf, r0)
    for mode in ("ad-split", "ad", "fd", "pd-split"):
        res = eng.ivf_query_batch(idx, qt, qr, K, nprobe, eng.IvfMode(MODE_ID[mode]),
                                  opts=eng.search_opts(first=0, step=64, probe_lo=probe_lo, r0=r0))
        for i in range(qt.shape[0]):
            ids, dists, stats = orc.ivf_query(lay, qt[i], qr[i], K, nprobe, mode, 2.1, 32, K, 64,
                                              probe_lo=probe_lo, r0=float(r0[i]))
            c = int(res.counts[i])
            assert c == len(ids), (mode, i)
            np.testing.assert_array_equal(res.ids[i, :c], ids, err_msg=f"{mode} q={i}")
            np.testing.assert_array_equal(res.dists[i, :c], dists)
            assert int(res.dims[i]) == int(stats[0]), (mode, i)
    with pytest.raises(ValueError):
        eng.ivf_query_batch(idx, qt, qr, K, nprobe, eng.IvfMode.kAdSplit, opts=eng.search_opts(probe_lo=nprobe + 1))


@pytest.mark.parametrize("case", [(6000, 96, 24, 40, 8), (3000, 128, 16, 30, 32), (2500, 200, 12, 20, 48),
                                  (4000, 64, 40, 64, 16), (5000, 192, 16, 24, 32)])
def test_ivf_dense_prefix_phase_bitexact(eng, orc, case, monkeypatch):
    """IVF++ with a 32-float A1: the dense prefix phase (interleaved A1 copy, built here
    for short lists with ADS_DENSE_MIN_LIST=0; default opts) == the lane walk without it
    (opts.tile = -1) == the oracle, at the batched and the reference schedules, with Δd
    below, at and above d1."""
    monkeypatch.setenv("ADS_DENSE_MIN_LIST", "0")
    n, d, blobs, k, dd = case
    raw, t, qr, qt, P = make_fixture(orc, n, d, blobs, 24, 300 + d)
    lay = oracle_index(orc, raw, t, P, k, 301, d1=32)
    idx = gpu_index(eng, lay, P)
    cfg = eng.DcoConfig(2.1, dd)
    for first, step in ((1, 1), (10, 64), (10, 7)):
        for nprobe in (1, 5, k):
            b = eng.ivf_query_batch(idx, qt, qr, 10, nprobe, eng.IvfMode.kAdSplit, cfg,
                                    opts=eng.search_opts(first=first, step=step, tile=-1))
            for tile in (64,):
                a = eng.ivf_query_batch(idx, qt, qr, 10, nprobe, eng.IvfMode.kAdSplit, cfg,
                                        opts=eng.search_opts(first=first, step=step, tile=tile))
                np.testing.assert_array_equal(a.ids, b.ids)
                np.testing.assert_array_equal(a.dims, b.dims)
                np.testing.assert_array_equal(np.nan_to_num(a.dists, nan=-1), np.nan_to_num(b.dists, nan=-1))
            assert_same_results(b, orc, lay, qt, qr, 10, nprobe, "ad-split", 2.1, dd, first, step)


@pytest.mark.parametrize("case", [(6000, 96, 24, 40, 32), (3000, 128, 16, 30, 32), (2500, 256, 12, 20, 32),
                                  (4000, 64, 40, 64, 32)])
@pytest.mark.parametrize("K", [1, 10, 100])
def test_ivf_certified_f32_walk_bitexact(eng, orc, case, K, monkeypatch):
    """walk = 2 (certified fp32 walk + exact fp64 re-walk of undecided / possibly
    positive candidates) == the exact walk == the oracle, at the reference schedule
    and batched schedules, including the first chunk at r = +inf and an initial
    radius r0 (the sharded second wave); with and without the dense prefix phase (the
    interleaved A1 copy built with ADS_DENSE_MIN_LIST=0)."""
    monkeypatch.setenv("ADS_DENSE_MIN_LIST", "0")
    n, d, blobs, k, dd = case
    raw, t, qr, qt, P = make_fixture(orc, n, d, blobs, 24, 400 + d)
    lay = oracle_index(orc, raw, t, P, k, 401, d1=32)
    idx = gpu_index(eng, lay, P)
    cfg = eng.DcoConfig(2.1, dd)
    for first, step in ((1, 1), (K, 64), (K, 7)):
        for nprobe in (1, 5, k):
            b = eng.ivf_query_batch(idx, qt, qr, K, nprobe, eng.IvfMode.kAdSplit, cfg,
                                    opts=eng.search_opts(first=first, step=step, walk=1, tile=-1))
            for tile in (-1, 64):
                a = eng.ivf_query_batch(idx, qt, qr, K, nprobe, eng.IvfMode.kAdSplit, cfg,
                                        opts=eng.search_opts(first=first, step=step, walk=2, tile=tile))
                np.testing.assert_array_equal(a.ids, b.ids)
                np.testing.assert_array_equal(a.dims, b.dims)
                np.testing.assert_array_equal(np.nan_to_num(a.dists, nan=-1), np.nan_to_num(b.dists, nan=-1))
            assert_same_results(b, orc, lay, qt, qr, K, nprobe, "ad-split", 2.1, dd, first, step)
    r0 = np.full(qt.shape[0], 0.5 * float(np.median(np.linalg.norm(t[:50] - qt[0], axis=1))))
    a = eng.ivf_query_batch(idx, qt, qr, K, k, eng.IvfMode.kAdSplit, cfg,
                            opts=eng.search_opts(first=K, step=64, walk=2, probe_lo=2, r0=r0))
    b = eng.ivf_query_batch(idx, qt, qr, K, k, eng.IvfMode.kAdSplit, cfg,
                            opts=eng.search_opts(first=K, step=64, walk=1, probe_lo=2, r0=r0))
    np.testing.assert_array_equal(a.ids, b.ids)
    np.testing.assert_array_equal(a.dims, b.dims)


@pytest.mark.parametrize("case", [(2500, 960, 12, 16, 32, 32),   # config 3's plan: 30 full segments
                                  (2500, 300, 12, 16, 32, 32),   # ragged last segment (12 floats)
                                  (3000, 256, 16, 20, 32, 16),   # 16-float segments (half lines)
                                  (2000, 512, 8, 12, 64, 48)])   # d1 != delta_d, ragged
@pytest.mark.parametrize("warps", [0, 4, 8])
def test_ivf_deep_tail_steps_bitexact(eng, orc, case, warps, monkeypatch):
    """Long walks (>= 8 segments) run the kernel with deep tail steps: a warp left with
    <= 16 live candidates fetches 2 or 4 consecutive segments of each per step and tests
    after every one.  Ids, distances, dims and candidate counts == the oracle at the
    reference schedule and at batched schedules whose chunks are mostly tail (7, 64) or
    mostly body (1000); all AD/PD modes; with and without the dense prefix phase."""
    monkeypatch.setenv("ADS_DENSE_MIN_LIST", "0")
    n, d, blobs, k, d1, dd = case
    raw, t, qr, qt, P = make_fixture(orc, n, d, blobs, 12, 700 + d)
    lay = oracle_index(orc, raw, t, P, k, 701, d1=d1)
    idx = gpu_index(eng, lay, P)
    cfg = eng.DcoConfig(2.1, dd)
    K = 10
    for mode in ("ad-split", "ad", "pd-split"):
        for first, step in ((1, 1), (K, 64), (K, 7), (K, 1000)):
            for nprobe in (2, k):
                for tile in ((-1, 64) if (mode == "ad-split" and d1 == 32) else (-1,)):
                    res = eng.ivf_query_batch(idx, qt, qr, K, nprobe, eng.IvfMode(MODE_ID[mode]), cfg,
                                              opts=eng.search_opts(first=first, step=step, tile=tile,
                                                                   warps_per_cta=warps, walk=1))
                    assert_same_results(res, orc, lay, qt, qr, K, nprobe, mode, 2.1, dd, first, step)


@pytest.mark.parametrize("case", [(2500, 960, 12, 16, 32, 32),   # config 3's plan: 30 full segments
                                  (2500, 300, 12, 16, 32, 32),   # ragged last segment
                                  (3000, 128, 16, 20, 32, 32),   # config 2's plan: 4 segments
                                  (2000, 512, 8, 12, 64, 16)])   # 16-float segments, d1 = 64
@pytest.mark.parametrize("warps", [0, 4])
def test_ivf_overlapped_chunks_bitexact(eng, orc, case, warps):
    """opts.lag = 1: lanes that find a chunk's stream exhausted start on the next chunk;
    chunk c >= 2 is tested against the thresholds after chunk c - 2, chunk 1 against chunk
    0's, with the merges in chunk order.  The oracle replays that schedule (lag = 2): ids,
    distances, dims and candidate counts are bit-exact, at schedules from one candidate per
    chunk to one chunk per query, and the plan reports the overlap."""
    n, d, blobs, k, d1, dd = case
    raw, t, qr, qt, P = make_fixture(orc, n, d, blobs, 12, 800 + d)
    lay = oracle_index(orc, raw, t, P, k, 801, d1=d1)
    idx = gpu_index(eng, lay, P)
    cfg = eng.DcoConfig(2.1, dd)
    K = 10
    for mode in ("ad-split", "ad", "pd-split"):
        for first, step in ((1, 1), (K, 64), (K, 7), (K, 5000), (3, 50), (K, 0)):
            for nprobe in (2, k):
                opts = eng.search_opts(first=first, step=step, tile=-1, warps_per_cta=warps, walk=1, lag=1)
                plan = eng.search_plan(idx, K, nprobe, eng.IvfMode(MODE_ID[mode]), cfg, opts=opts)
                # plans with an untested prefix (d1 spanning several segments) keep the
                # pre-walk and the plain schedule; the plan says which one runs
                assert plan["first"] == first and (plan["lag"] == 1 or d1 > dd)
                res = eng.ivf_query_batch(idx, qt, qr, K, nprobe, eng.IvfMode(MODE_ID[mode]), cfg, opts=opts)
                for qi in range(qt.shape[0]):
                    ids, dists, stats = orc.ivf_query(lay, qt[qi], qr[qi], K, nprobe, mode, 2.1, dd,
                                                      plan["first"], plan["step"], lag=2 if plan["lag"] else 0)
                    c = int(res.counts[qi])
                    assert c == len(ids), (mode, first, step, nprobe, qi)
                    np.testing.assert_array_equal(res.ids[qi, :c], ids, err_msg=f"{mode} {first}/{step} np={nprobe} q={qi}")
                    np.testing.assert_array_equal(res.dists[qi, :c], dists)
                    assert int(res.dims[qi]) == int(stats[0]), (mode, first, step, nprobe, qi)
                    assert int(res.candidates[qi]) == int(stats[2])
    # where the plan cannot overlap (the FD walk pre-walks its untested prefix) lag is ignored
    plan = eng.search_plan(idx, K, 2, eng.IvfMode.kFd, cfg, opts=eng.search_opts(lag=1))
    assert plan["lag"] == 0
    # default options: overlapped from 8 segments when the engine also picks the schedule;
    # a pinned schedule, a probe range or lag = -1 keep the plain one
    auto = eng.search_plan(idx, K, k, eng.IvfMode.kAdSplit, cfg)["lag"]
    assert auto == (1 if (d1 <= dd and (d + dd - 1) // dd >= 8) else 0)
    assert eng.search_plan(idx, K, k, eng.IvfMode.kAdSplit, cfg, opts=eng.search_opts(step=64))["lag"] == 0
    assert eng.search_plan(idx, K, k, eng.IvfMode.kAdSplit, cfg, opts=eng.search_opts(lag=-1))["lag"] == 0
    assert eng.search_plan(idx, K, k, eng.IvfMode.kAdSplit, cfg, opts=eng.search_opts(probe_lo=1))["lag"] == 0


def test_ivf_long_lists_default_path_bitexact(eng, orc):
    """The default path at config 5's shape of work: 6 250-row lists (the interleaved A1
    copy and its dense prefix phase) and 100 000 candidates per query (the certified fp32
    walk), both picked automatically, == the exact walk without the dense phase == the
    oracle on the exported index, at the batched schedule."""
    n, d, k, nq, K, nprobe = 400_000, 96, 64, 24, 100, 16
    m = eng.generate_orthogonal(d, 7)

    def rows(lo, count, stride=1):
        return eng.synth_rows(n, d, 256, 7, 1, lo, count, stride, kind=3, sigma=1.4)

    idx, _, _ = eng.build_ivf_streamed(rows, n, d, m, k, 7, 32, 4, 40_000, chunk=100_000)
    q = eng.synth_rows(1000, d, 256, 7, 2, 0, nq, 1, kind=3, sigma=1.4)
    qt = eng.apply_dataset(m, q)
    plan = eng.search_plan(idx, K, nprobe, eng.IvfMode.kAdSplit)
    assert plan["walk"] == 2 and plan["dense"]  # the default path at config 5's shape
    step = plan["step"]
    a = eng.ivf_query_batch(idx, qt, None, K, nprobe, eng.IvfMode.kAdSplit)
    b = eng.ivf_query_batch(idx, qt, None, K, nprobe, eng.IvfMode.kAdSplit,
                            opts=eng.search_opts(walk=1, tile=-1, step=step))
    assert float(a.candidates.mean()) >= 100_000
    np.testing.assert_array_equal(a.ids, b.ids)
    np.testing.assert_array_equal(a.dims, b.dims)
    np.testing.assert_array_equal(a.dists, b.dists)
    for walk, tile in ((1, 64), (2, -1)):  # the dense phase with the exact walk, the fp32 walk alone
        c = eng.ivf_query_batch(idx, qt, None, K, nprobe, eng.IvfMode.kAdSplit,
                                opts=eng.search_opts(walk=walk, tile=tile, step=step))
        np.testing.assert_array_equal(c.ids, b.ids)
        np.testing.assert_array_equal(c.dims, b.dims)
        np.testing.assert_array_equal(c.dists, b.dists)
    # chunk-state edge shapes of the dense + fp32 kernel: odd chunk caps, and chunks too
    # long for the pending distances to live in the gather lines (8 * cap + 1 KiB > 16 KiB)
    for first, st in ((99, 333), (K, 2048), (K, 4099)):
        c = eng.ivf_query_batch(idx, qt, None, K, nprobe, eng.IvfMode.kAdSplit,
                                opts=eng.search_opts(first=first, step=st))
        e = eng.ivf_query_batch(idx, qt, None, K, nprobe, eng.IvfMode.kAdSplit,
                                opts=eng.search_opts(first=first, step=st, walk=1, tile=-1))
        np.testing.assert_array_equal(c.ids, e.ids)
        np.testing.assert_array_equal(c.dims, e.dims)
        np.testing.assert_array_equal(c.dists, e.dists)
    ex = idx.export()
    lay = {"n": idx.n, "d": d, "k": k, "d1": 32, "split": True, "centroids_t": ex["centroids_t"],
           "centroids_raw": ex["centroids_t"], "list_off": ex["list_off"], "ids_flat": ex["ids_flat"],
           "a1_t": ex["a1_t"], "a2_t": ex["a2_t"], "a1_raw": ex["a1_t"], "a2_raw": ex["a2_t"],
           "vec_t": None, "vec_raw": None}
    for i in range(nq):
        ids, dists, stats = orc.ivf_query(lay, qt[i], qt[i], K, nprobe, "ad-split", 2.1, 32, K, step)
        np.testing.assert_array_equal(a.ids[i], ids, err_msg=f"q={i}")
        np.testing.assert_array_equal(a.dists[i], dists, err_msg=f"q={i}")
        assert int(a.dims[i]) == int(stats[0]), i

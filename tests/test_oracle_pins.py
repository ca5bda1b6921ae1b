"""Pin the oracle restatement (oracle/adsann_oracle.c) before trusting it.

1. Against the committed golden vectors generated from the reference itself
   (tests/golden/make_golden.py) — always runs.
2. Against the reference library compiled from /root/reference
   (oracle/_ref) on randomized inputs — runs wherever that library exists.
Every comparison is bit-exact.
"""
import math

import numpy as np
import pytest

from helpers import MODES

# ------------------------------------------------------------------ golden


def test_golden_rng_transform(orc, golden):
    for kind in range(4):
        np.testing.assert_array_equal(orc.rng_draw(42, 0x1234ABCD, kind, 257, arg=1000),
                                      golden[f"rng_k{kind}"])
    np.testing.assert_array_equal(orc.rng_draw(7, 0, 2, 65, use_stream=False), golden["rng_plain_normal"])
    for d in (1, 2, 16, 64):
        np.testing.assert_array_equal(orc.generate_orthogonal(d, 5), golden[f"P{d}"])
    P = golden["P64"]
    X = golden["apply_X"]
    np.testing.assert_array_equal(orc.apply_dataset(P, X), golden["apply_Y"])
    np.testing.assert_array_equal(orc.apply_transpose(P, X[3]), golden["apply_T"])
    np.testing.assert_array_equal(orc.apply_prefix(P, X[5], 17), golden["apply_prefix"])


def test_golden_dco(orc, golden):
    np.testing.assert_array_equal(orc.ad_context(2.1, 32, 128), golden["factor_128"])
    np.testing.assert_array_equal(orc.ad_context(1.5, 16, 80), golden["factor_80"])
    args = [golden[k] for k in ("dco_X", "dco_Q", "dco_rows", "dco_qidx", "dco_r")]
    for nm, pdm, eps, dd in (("ad", False, 2.1, 16), ("pd", True, 2.1, 8), ("ad7", False, 0.9, 7)):
        pos, dims, dsq, obs = orc.ad_scan_pairs(*args, eps, dd, pd_mode=pdm)
        np.testing.assert_array_equal(pos, golden[f"dco_{nm}_pos"])
        np.testing.assert_array_equal(dims, golden[f"dco_{nm}_dims"])
        np.testing.assert_array_equal(dsq, golden[f"dco_{nm}_dsq"])
        np.testing.assert_array_equal(obs, golden[f"dco_{nm}_obs"])


def test_golden_kmeans_bruteforce(orc, golden):
    cent, asg, obj, it = orc.kmeans(golden["km_X"], 7, 25, 3)
    np.testing.assert_array_equal(cent, golden["km_cent"])
    np.testing.assert_array_equal(asg, golden["km_asg"])
    assert obj == float(golden["km_obj"]) and it == int(golden["km_it"])
    np.testing.assert_array_equal(orc.brute_force_knn(golden["bf_base"], golden["bf_q"], 9),
                                  golden["bf_ids"])


def test_golden_ivf(orc, golden):
    g = golden
    lay = orc.ivf_layout(g["ivf_raw"], g["ivf_t"], g["ivf_P"], g["ivf_centroids_t"],
                         g["ivf_assignment"], 12, 8, True)
    for nm in ("centroids_raw", "list_off", "ids_flat"):
        np.testing.assert_array_equal(lay[nm], g[f"ivf_{nm}"])
    for mode in MODES:
        for np_ in (1, 4, 12):
            key = f"ivfq_{mode}_{np_}"
            for qi in range(5):
                ids, dists, stats = orc.ivf_query(lay, g["ivf_qt"][qi], g["ivf_qr"][qi], 5, np_,
                                                  mode, 2.1, 8)
                c = len(ids)
                np.testing.assert_array_equal(ids, g[key + "_ids"][qi, :c])
                np.testing.assert_array_equal(dists, g[key + "_dists"][qi, :c])
                assert int(stats[0]) == int(g[key + "_dims"][qi])


# ------------------------------------------------------------------ reference itself


def test_ref_rng_and_transform(orc, ref):
    for kind in range(4):
        for seed, tag in ((0, 0), (42, 0x9d5c41cf0f5e6a31), (2**63 + 5, 77)):
            np.testing.assert_array_equal(orc.rng_draw(seed, tag, kind, 333, arg=97),
                                          ref.rng_draw(seed, tag, kind, 333, arg=97))
    for d in (1, 3, 31, 96, 130):
        np.testing.assert_array_equal(orc.generate_orthogonal(d, d + 2), ref.generate_orthogonal(d, d + 2))
    with pytest.raises(ValueError):
        orc.generate_orthogonal(0, 1)
    with pytest.raises(ValueError):
        ref.generate_orthogonal(0, 1)
    rng = np.random.default_rng(1)
    for d in (5, 128):
        P = ref.generate_orthogonal(d, 9)
        X = rng.normal(0, 10, (50, d)).astype(np.float32)
        np.testing.assert_array_equal(orc.apply_dataset(P, X), ref.apply_dataset(P, X))
        np.testing.assert_array_equal(orc.apply_transpose(P, X[0]), ref.apply_transpose(P, X[0]))
        for p in (0, 1, d // 2, d):
            np.testing.assert_array_equal(orc.apply_prefix(P, X[1], p), ref.apply_prefix(P, X[1], p))


def test_ref_dco_api(orc, ref):
    rng = np.random.default_rng(4242)
    for d in (1, 2, 7, 33, 128):
        assert orc.threshold_multiplier(d, 2.1) == ref.threshold_multiplier(d, 2.1)
    for eps, dd, D in ((2.1, 32, 128), (0.3, 1, 7), (5.0, 9, 100)):
        np.testing.assert_array_equal(orc.ad_context(eps, dd, D), ref.ad_context(eps, dd, D))
    for _ in range(3000):
        d = int(rng.integers(1, 161))
        dd = int(rng.integers(1, d + 1))
        eps = float(rng.uniform(0.1, 4.0))
        o = rng.normal(0, 2, d).astype(np.float32)
        q = rng.normal(0, 2, d).astype(np.float32)
        r = float(np.linalg.norm(o.astype(np.float64) - q) * rng.uniform(0.05, 1.5))
        for kind in ("fd", "pd", "ad"):
            assert orc.dco(kind, o, q, r, eps, dd) == ref.dco(kind, o, q, r, eps, dd)
        d0 = int(rng.integers(0, d))
        s0 = float(rng.uniform(0, 50))
        for kernel in (0, 1):
            for tas in (False, True):
                a = orc.scan_kernel(kernel, o[d0:], q[d0:], d, d0, s0, r, eps, dd, tas)
                b = ref.scan_kernel(kernel, o[d0:], q[d0:], d, d0, s0, r, eps, dd, tas)
                assert a == b
    # argument validation (test_dco.cpp:392-401)
    a, b = [1.0, 2.0], [1.0]
    for lib in (orc, ref):
        for call in (lambda: lib.dco("fd", a, b, 1.0), lambda: lib.dco("fd", a, a, -1.0),
                     lambda: lib.dco("pd", a, a, 1.0, 2.1, 0), lambda: lib.dco("pd", a, a, 1.0, 2.1, 3),
                     lambda: lib.dco("ad", a, a, 1.0, 0.0, 1), lambda: lib.dco("ad", a, a, 1.0, 2.1, 0),
                     lambda: lib.dco("fd", a, a, math.inf)):
            with pytest.raises(ValueError):
                call()


@pytest.mark.parametrize("n,d,k,iters,seed", [(20, 8, 20, 25, 7), (100, 6, 1, 25, 9),
                                               (500, 12, 10, 25, 21), (2000, 32, 40, 10, 3)])
def test_ref_kmeans(orc, ref, n, d, k, iters, seed):
    X = np.random.default_rng(seed).normal(0, 3, (n, d)).astype(np.float32)
    a = orc.kmeans(X, k, iters, seed)
    b = ref.kmeans(X, k, iters, seed)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])
    assert a[2:] == b[2:]
    with pytest.raises(ValueError):
        orc.kmeans(X, n + 1, 5, 1)


def test_ref_brute_force(orc, ref):
    rng = np.random.default_rng(8)
    base = rng.integers(0, 4, (700, 9)).astype(np.float32)  # many exact ties
    q = rng.integers(0, 4, (10, 9)).astype(np.float32)
    for K in (1, 10, 700):
        np.testing.assert_array_equal(orc.brute_force_knn(base, q, K), ref.brute_force_knn(base, q, K))


@pytest.mark.parametrize("split,d1,dd", [(True, 32, 32), (True, 8, 16), (False, 32, 32), (True, 20, 12)])
def test_ref_ivf_all_modes(orc, ref, split, d1, dd):
    from helpers import make_fixture

    raw, t, qr, qt, P = make_fixture(orc, 1500, 64, 8, 12, 57)
    idx = ref.build_ivf(raw, t, P, 20, 59, split=split, d1=d1)
    ex = idx.export()
    asg = np.empty(raw.shape[0], np.int32)
    for c in range(20):
        asg[ex["ids_flat"][ex["list_off"][c]:ex["list_off"][c + 1]]] = c
    lay = orc.ivf_layout(raw, t, P, ex["centroids_t"], asg, 20, d1, split)
    for nm in ("ids_flat", "vec_t", "vec_raw", "centroids_raw") + (("a1_t", "a2_t", "a1_raw", "a2_raw") if split else ()):
        np.testing.assert_array_equal(lay[nm], ex[nm], err_msg=nm)
    modes = MODES if split else ("fd", "pd", "ad")
    for mode in modes:
        for np_ in (1, 5, 20):
            for qi in range(qt.shape[0]):
                a = orc.ivf_query(lay, qt[qi], qr[qi], 10, np_, mode, 2.1, dd)
                b = idx.query(qt[qi], qr[qi], 10, np_, mode, 2.1, dd)
                for x, y in zip(a, b):
                    np.testing.assert_array_equal(x, y)
    if not split:
        with pytest.raises(ValueError):
            orc.ivf_query(lay, qt[0], qr[0], 10, 3, "ad-split")
        with pytest.raises(ValueError):
            idx.query(qt[0], qr[0], 10, 3, "ad-split")


def test_oracle_batched_schedule_semantics(orc):
    """first=step=1 is the reference; batching only loosens r, never changes exactness."""
    from helpers import make_fixture, oracle_index

    raw, t, qr, qt, P = make_fixture(orc, 3000, 64, 16, 20, 5)
    lay = oracle_index(orc, raw, t, P, 40, 6)
    gt = orc.brute_force_knn(t, qt, 10)
    for qi in range(qt.shape[0]):
        a = orc.ivf_query(lay, qt[qi], qr[qi], 10, 40, "ad-split")
        b = orc.ivf_query(lay, qt[qi], qr[qi], 10, 40, "ad-split", first=10, step=256)
        c = orc.ivf_query(lay, qt[qi], qr[qi], 10, 40, "ad-split", first=10**9, step=1)
        # with r = +inf throughout nothing is rejected: exact top-10 over everything
        assert int(c[2][0]) == int(c[2][2]) * 64
        np.testing.assert_array_equal(np.sort(c[0]), np.sort(gt[qi]))
        assert int(b[2][0]) >= int(a[2][0]) * 0.95
        assert len(set(a[0]) & set(gt[qi])) <= 10


@pytest.mark.parametrize("n,d,nq,K,grid", [(1500, 48, 12, 20, [1e6]),
                                           (2000, 64, 10, 50, [2.5, 0.5, 1.0, 2.0, 1.5, 3.0]),
                                           (800, 30, 7, 1, [2.1, 2.1, 0.2])])
def test_ref_verify_theory(orc, ref, n, d, nq, K, grid):
    """orc_verify_theory == adsann::verify_theory (bench.cpp:303-392), every field exact."""
    from helpers import make_fixture

    _, t, _, qt, _ = make_fixture(orc, n, d, 8, nq, 31 + d)
    a = orc.verify_theory(t, qt, K, grid)
    b = ref.verify_theory(t, qt, K, grid)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
    with pytest.raises(ValueError):
        orc.verify_theory(t, qt, 0, grid)
    with pytest.raises(ValueError):
        orc.verify_theory(t, qt, n + 1, grid)


def test_oracle_rejects_layouts_missing_mode_arrays(orc):
    """A layout without the arrays a mode reads is an error, not a crash."""
    from helpers import make_fixture, oracle_index

    raw, t, qr, qt, P = make_fixture(orc, 500, 32, 4, 2, 3)
    lay = oracle_index(orc, raw, t, P, 8, 4, d1=16)
    lay = dict(lay, vec_raw=None, vec_t=None)
    orc.ivf_query(lay, qt[0], qr[0], 5, 2, "ad-split", 2.1, 16)  # split arrays present
    with pytest.raises(ValueError):
        orc.ivf_query(lay, qt[0], qr[0], 5, 2, "fd")


def test_oracle_lag_schedule(orc):
    """orc_ivf_query_lag: with a single chunk the lag changes nothing; with short
    chunks it still returns K exact (dist, id) pairs sorted ascending, each distance
    the exact fp64 distance of its id, and it never scans fewer dims than lag 0
    (a staler radius only rejects later)."""
    from helpers import make_fixture, oracle_index

    raw, t, qr, qt, P = make_fixture(orc, 2000, 64, 12, 6, 41)
    lay = oracle_index(orc, raw, t, P, 20, 42, d1=32)
    for qi in range(qt.shape[0]):
        a = orc.ivf_query(lay, qt[qi], qr[qi], 10, 6, "ad-split", 2.1, 32, 10**9, 1)
        b = orc.ivf_query(lay, qt[qi], qr[qi], 10, 6, "ad-split", 2.1, 32, 10**9, 1, lag=1)
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[1], b[1])
        assert int(a[2][0]) == int(b[2][0])
        c0 = orc.ivf_query(lay, qt[qi], qr[qi], 10, 6, "ad-split", 2.1, 32, 10, 16)
        c1 = orc.ivf_query(lay, qt[qi], qr[qi], 10, 6, "ad-split", 2.1, 32, 10, 16, lag=1)
        assert len(c1[0]) == 10 and np.all(np.diff(c1[1]) >= 0)
        exact = np.sqrt(((t[c1[0]].astype(np.float64) - qt[qi].astype(np.float64)) ** 2).sum(axis=1))
        np.testing.assert_allclose(c1[1], exact, rtol=1e-12)
        assert int(c1[2][0]) >= int(c0[2][0])

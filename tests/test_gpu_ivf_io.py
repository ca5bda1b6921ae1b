"""On-disk index interop (save_ivf / load_ivf, ivf.hpp:91-92, ivf.cpp:423-501)
through the C ABI: a directory written by the reference (oracle/_ref, the
reference compiled from its sources) loads into the engine bit-identically and
searches exactly like the reference; a directory written by the engine loads into
the reference and searches the same; a raw-less (config-5 style) index
round-trips through the engine."""
import numpy as np
import pytest

from helpers import MODE_ID, make_fixture

pytestmark = pytest.mark.gpu


def _same_layout(ex, rx, with_raw=True):
    np.testing.assert_array_equal(ex["centroids_t"], rx["centroids_t"])
    np.testing.assert_array_equal(ex["list_off"], rx["list_off"])
    np.testing.assert_array_equal(ex["ids_flat"], rx["ids_flat"])
    np.testing.assert_array_equal(ex["a1_t"], rx["a1_t"])
    np.testing.assert_array_equal(ex["a2_t"], rx["a2_t"])
    if with_raw:
        np.testing.assert_array_equal(ex["centroids_raw"], rx["centroids_raw"])
        np.testing.assert_array_equal(ex["a1_raw"], rx["a1_raw"])
        np.testing.assert_array_equal(ex["a2_raw"], rx["a2_raw"])


@pytest.mark.parametrize("split", [True, False])
def test_reference_directory_loads_into_engine(eng, orc, ref, tmp_path, split):
    raw, t, qr, qt, P = make_fixture(orc, 3000, 48, 12, 20, 31)
    h = ref.build_ivf(raw, t, P, 24, 32, split=split, d1=16)
    h.save(tmp_path / "idx")
    m = eng.TransformMatrix(48, 31, P)
    idx = eng.load_ivf(tmp_path / "idx", m)
    rx = h.export()
    assert (idx.n, idx.d, idx.k_clusters, idx.d1, int(idx.layout), idx.seed) == (
        rx["n"], rx["d"], rx["k"], rx["d1"], int(split), 32)
    ex = idx.export()
    if split:
        _same_layout(ex, rx)
    else:  # contiguous: the engine re-blocks vec_* into its 32-float A1 | A2 streams
        np.testing.assert_array_equal(np.hstack([ex["a1_t"], ex["a2_t"]]), rx["vec_t"])
        np.testing.assert_array_equal(np.hstack([ex["a1_raw"], ex["a2_raw"]]), rx["vec_raw"])
    modes = ("fd", "pd", "ad", "ad-split", "pd-split") if split else ("fd", "pd", "ad")
    for mode in modes:
        res = eng.ivf_query_batch(idx, qt, qr, 10, 6, eng.IvfMode(MODE_ID[mode]), first=1, step=1)
        for i in range(qt.shape[0]):
            ids, dists, stats = h.query(qt[i], qr[i], 10, 6, mode)
            c = int(res.counts[i])
            np.testing.assert_array_equal(res.ids[i, :c], ids, err_msg=f"{mode} {i}")
            np.testing.assert_array_equal(res.dists[i, :c], dists, err_msg=f"{mode} {i}")
            assert int(res.dims[i]) == int(stats[0])


def test_engine_directory_loads_into_reference(eng, orc, ref, tmp_path):
    raw, t, qr, qt, P = make_fixture(orc, 4000, 64, 16, 16, 33)
    m = eng.TransformMatrix(64, 33, P)
    idx = eng.build_ivf(raw, t, m, 40, 34, eng.IvfLayout.kSplit, 32, max_iters=10)
    eng.save_ivf(idx, tmp_path / "e")
    h = ref.load_ivf(tmp_path / "e")
    rx = h.export()
    _same_layout(idx.export(), rx)
    np.testing.assert_array_equal(rx["vec_t"], np.hstack([rx["a1_t"], rx["a2_t"]]))
    for mode in ("fd", "ad", "ad-split", "pd-split"):
        res = eng.ivf_query_batch(idx, qt, qr, 10, 8, eng.IvfMode(MODE_ID[mode]), first=1, step=1)
        for i in range(qt.shape[0]):
            ids, dists, stats = h.query(qt[i], qr[i], 10, 8, mode)
            np.testing.assert_array_equal(res.ids[i, :len(ids)], ids)
            np.testing.assert_array_equal(res.dists[i, :len(ids)], dists)
            assert int(res.dims[i]) == int(stats[0])
    # and back: engine -> disk -> engine is the identity
    again = eng.load_ivf(tmp_path / "e", m)
    _same_layout(again.export(), idx.export())


def test_rawless_index_roundtrip(eng, ref, tmp_path):
    """A config-5 style index (transformed vectors only) round-trips through the engine;
    the reference's format cannot express it, so its loader refuses the directory."""
    n, d, k = 30_000, 96, 64
    m = eng.generate_orthogonal(d, 5)

    def rows(lo, count, stride=1):
        return eng.synth_rows(n, d, 40, 5, 1, lo, count, stride, kind=3, sigma=1.4)

    idx, _, _ = eng.build_ivf_streamed(rows, n, d, m, k, 5, 32, 4, 3000, chunk=8000)
    eng.save_ivf(idx, tmp_path / "c5")
    back = eng.load_ivf(tmp_path / "c5", m)
    assert not back.has_raw
    _same_layout(back.export(), idx.export(), with_raw=False)
    q = eng.synth_rows(100, d, 40, 5, 2, 0, 12, 1, kind=3, sigma=1.4)
    a = eng.ivf_query_batch(idx, None, q, 20, 8, eng.IvfMode.kAdSplit)
    b = eng.ivf_query_batch(back, None, q, 20, 8, eng.IvfMode.kAdSplit)
    np.testing.assert_array_equal(a.ids, b.ids)
    np.testing.assert_array_equal(a.dims, b.dims)
    with pytest.raises((RuntimeError, ValueError)):  # "cannot open .../centroids_raw.fvecs"
        ref.load_ivf(tmp_path / "c5")


def test_load_errors(eng, tmp_path):
    with pytest.raises(RuntimeError):
        eng.load_ivf(tmp_path / "missing")

"""HNSW+/HNSW++ through the facade: graph construction on the
host and every query-time DCO batched per hop on the B200, against the reference
itself (oracle/_ref: adsann::build_hnsw / save_hnsw / hnsw_query compiled from
/root/reference).  The facade and the reference define the same adsann:: symbols,
so the facade runs in its own process (tests/cpp/_bin/facade_hnsw_tool) and the
two meet through the reference's on-disk graph format (hnsw.cpp:381-456).

* construction (CPU): the facade's graph directory is byte-identical to the
  reference's for the same data and seed;
* queries (GPU): on the reference's graph, every mode returns the reference's
  ids, distances (bit-exact), dims_evaluated, DCO count and hop count."""
import os
import subprocess

import numpy as np
import pytest

from helpers import make_fixture

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "tests", "cpp", "_bin", "facade_hnsw_tool")


def _fvecs(path, X):
    X = np.ascontiguousarray(X, np.float32)
    n, d = X.shape
    rec = np.empty((n, d + 1), np.float32)
    rec[:, 0] = np.frombuffer(np.int32(d).tobytes(), np.float32)[0]
    rec[:, 1:] = X
    rec.tofile(path)


def _tool(*args):
    if not os.path.exists(TOOL):
        pytest.skip("facade_hnsw_tool not built (make -C tests/cpp)")
    p = subprocess.run([TOOL, *map(str, args)], capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr


@pytest.fixture(scope="module")
def graphs(tmp_path_factory, request):
    from oracle import load_oracle, load_ref, ref_available

    if not ref_available():
        pytest.skip("oracle/_ref not built")
    orc, ref = load_oracle(), load_ref()
    base = tmp_path_factory.mktemp("hnsw")
    out = {}
    for name, (n, d, blobs, nq, seed, M, ef) in {"a": (2500, 48, 10, 24, 41, 8, 60),
                                                 "b": (1200, 20, 6, 16, 43, 4, 16)}.items():
        raw, t, qr, qt, P = make_fixture(orc, n, d, blobs, nq, seed)
        files = {}
        for nm, X in (("raw", raw), ("t", t), ("qr", qr), ("qt", qt)):
            files[nm] = base / f"{name}_{nm}.fvecs"
            _fvecs(files[nm], X)
        h = ref.hnsw_build(raw, t, M, ef, seed + 1)
        ref.hnsw_save(h, base / f"{name}_ref")
        out[name] = dict(raw=raw, t=t, qr=qr, qt=qt, files=files, h=h, dir=base / f"{name}_ref",
                         M=M, ef=ef, seed=seed + 1, base=base)
    yield ref, out
    for g in out.values():
        ref.hnsw_free(g["h"])


@pytest.mark.parametrize("name", ["a", "b"])
def test_facade_graph_construction_is_the_reference_graph(graphs, name):
    ref, gs = graphs
    g = gs[name]
    fdir = g["base"] / f"{name}_facade"
    _tool("build", g["files"]["raw"], g["files"]["t"], g["M"], g["ef"], g["seed"], fdir)
    for fn in ("meta.txt", "levels.ivecs", "links.ivecs"):
        assert (fdir / fn).read_bytes() == (g["dir"] / fn).read_bytes(), fn


@pytest.mark.gpu
@pytest.mark.parametrize("name,K,nef,eps0,dd", [("a", 10, 40, 2.1, 32), ("a", 5, 12, 0.8, 8),
                                                ("b", 10, 30, 2.1, 4), ("b", 3, 3, 1e6, 20)])
def test_facade_queries_match_reference(graphs, eng, name, K, nef, eps0, dd):
    ref, gs = graphs
    g = gs[name]
    nq = g["qr"].shape[0]
    for mode in range(4):  # plain, pd, plus, plusplus
        out = g["base"] / f"{name}_q{mode}_{K}_{nef}_{dd}.bin"
        _tool("query", g["dir"], g["files"]["raw"], g["files"]["t"], g["files"]["qr"], g["files"]["qt"], K, nef,
              mode, eps0, dd, out)
        rec = np.dtype([("cnt", "<i4"), ("ids", "<i4", K), ("dists", "<f8", K), ("st", "<u8", 4)])
        got = np.fromfile(out, rec)
        assert got.shape[0] == nq
        for i in range(nq):
            ids, dists, st = ref.hnsw_query(g["h"], g["qt"][i], g["qr"][i], K, nef, mode, eps0, dd)
            c = int(got["cnt"][i])
            assert c == len(ids), (mode, i)
            np.testing.assert_array_equal(got["ids"][i, :c], ids, err_msg=f"mode {mode} q {i}")
            np.testing.assert_array_equal(got["dists"][i, :c], dists, err_msg=f"mode {mode} q {i}")
            np.testing.assert_array_equal(got["st"][i], st, err_msg=f"mode {mode} q {i} stats")

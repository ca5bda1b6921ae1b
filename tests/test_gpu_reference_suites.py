"""The REFERENCE's own doctest suites (test_dco.cpp, test_ivf.cpp,
test_transform.cpp, test_vecio.cpp, test_bench.cpp, test_hnsw.cpp from
/root/reference/proj/tests), compiled unchanged against the adsann C++ facade of
the B200 engine (tests/cpp/Makefile, doctest shim tests/cpp/doctest.h), run on
the GPU.  Every DCO, transform, k-means, build_ivf, ivf_query, brute_force_knn,
sweep_ivf and hnsw_query comparison in them executes on the B200 through
include/adsann_b200.h (HNSW: graph build and walk on the host, every query-time
DCO batched per hop on the GPU).  facade_theory_test is this repo's own doctest
file for the facade's verify_theory."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_bin")


@pytest.mark.parametrize("suite", ["test_dco", "test_transform", "test_vecio", "test_ivf", "test_bench",
                                   "test_hnsw", "facade_theory_test"])
def test_reference_suite_passes_on_b200(eng, suite):
    exe = os.path.join(BIN, suite)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (needs /root/reference at build time: make -C tests/cpp)")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    tail = "\n".join(p.stderr.strip().splitlines()[-40:])
    assert p.returncode == 0, f"{suite} failed:\n{tail}"
    assert "failed: 0" in p.stderr, tail

"""The C-ABI boundary without a GPU: the library loads, exports every symbol the
header declares, and its host-side entry points match the oracle bit for bit.
No GPU compute is called here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "adsann_b200.h")


def header_symbols():
    return sorted(set(re.findall(r"\b(ads_[a-z0-9_]+)\s*\(", open(HEADER).read())))


def test_library_exports_every_header_symbol():
    from paper_2303_09855_b200 import _lib

    syms = header_symbols()
    assert len(syms) >= 40
    missing = [s for s in syms if not hasattr(_lib.lib, s)]
    assert not missing, missing


def test_header_cites_reference_interfaces():
    text = open(HEADER).read()
    for cite in ("ivf.cpp:296-419", "dco.hpp:86-177", "dco.cpp:70-110", "transform.cpp:47-97",
                 "bench.cpp:31-61", "ivf.hpp:55-74"):
        assert cite in text, cite


def test_host_rng_matches_oracle(orc):
    import paper_2303_09855_b200 as ads

    for kind in range(4):
        for seed, tag in ((0, 0), (42, 0x1234), (7, 0x9d5c41cf0f5e6a31)):
            np.testing.assert_array_equal(ads.rng_draw(seed, tag, kind, 501, arg=13),
                                          orc.rng_draw(seed, tag, kind, 501, arg=13))


@pytest.mark.parametrize("dim", [1, 2, 5, 64, 128, 200])
def test_generate_orthogonal_matches_oracle(orc, dim):
    import paper_2303_09855_b200 as ads

    m = ads.generate_orthogonal(dim, 3 + dim)
    np.testing.assert_array_equal(m.entries, orc.generate_orthogonal(dim, 3 + dim))


def test_dco_host_tables_and_validation(orc):
    import paper_2303_09855_b200 as ads

    for d in (1, 2, 7, 1 << 20):
        assert ads.threshold_multiplier(d, ads.DcoConfig(2.1, 32)) == orc.threshold_multiplier(d, 2.1)
    assert abs(ads.threshold_multiplier(1, ads.DcoConfig(2.1, 32)) - 3.1) < 1e-12
    assert abs(ads.threshold_multiplier(4, ads.DcoConfig(2.0, 32)) - 2.0) < 1e-12
    for eps, dd, D in ((2.1, 32, 128), (0.5, 1, 9), (3.0, 7, 100)):
        np.testing.assert_array_equal(ads.ad_context_factor(ads.DcoConfig(eps, dd), D),
                                      orc.ad_context(eps, dd, D))
    with pytest.raises(ValueError):
        ads.threshold_multiplier(0, ads.DcoConfig())
    with pytest.raises(ValueError):
        ads.ad_context_factor(ads.DcoConfig(0.0, 32), 64)
    with pytest.raises(ValueError):
        ads.ad_context_factor(ads.DcoConfig(2.1, 65), 64)
    with pytest.raises(ValueError):
        ads.generate_orthogonal(0, 1)


def test_synth_is_deterministic_across_thread_counts():
    import paper_2303_09855_b200 as ads

    a = ads.synth(10_000, 24, 16, 5, 1, kind=1, center_lo=100, center_hi=150, sigma=9,
                  decay=True, threads=1)
    b = ads.synth(10_000, 24, 16, 5, 1, kind=1, center_lo=100, center_hi=150, sigma=9,
                  decay=True, threads=7)
    np.testing.assert_array_equal(a, b)
    assert np.all(a == np.round(a)) and a.min() >= 0 and a.max() <= 255
    u = ads.synth(5000, 16, 8, 5, 2, kind=2, center_lo=0.2, center_hi=0.8, sigma=0.3)
    assert u.min() >= 0.0 and u.max() <= 1.0
    s = ads.synth(5000, 16, 8, 5, 2, kind=3, sigma=0.25)
    np.testing.assert_allclose(np.linalg.norm(s.astype(np.float64), axis=1), 1.0, atol=1e-6)
    q1 = ads.synth(100, 16, 8, 5, 2)
    q2 = ads.synth(100, 16, 8, 5, 3)
    assert not np.array_equal(q1, q2)  # distinct roles -> distinct streams


def test_configs_match_baseline_shapes():
    from paper_2303_09855_b200 import configs

    c1, c2, c3 = configs.CONFIGS[1], configs.CONFIGS[2], configs.CONFIGS[3]
    assert (c1.n, c1.d, c1.nq, c1.components, c1.nlist, c1.K, c1.nprobe) == (100_000, 128, 1000, 64, 256, 20, 16)
    assert (c2.n, c2.d, c2.nq, c2.components, c2.nlist, c2.K) == (1_000_000, 128, 10_000, 1024, 4096, 100)
    assert (c3.n, c3.d, c3.nq, c3.components, c3.nlist, c3.K) == (1_000_000, 960, 10_000, 1024, 4096, 100)
    assert c2.sweep == (8, 16, 32, 64, 128)


def test_gpu_entry_points_fail_loudly_without_device():
    import paper_2303_09855_b200 as ads

    if ads.device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(RuntimeError):
        ads.Context(0)
    with pytest.raises(RuntimeError):
        ads.fd_scan([3.0, 4.0], [0.0, 0.0], 5.0)

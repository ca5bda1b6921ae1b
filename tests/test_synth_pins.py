"""The benchmark configs' mixture generator, host side (no GPU): the engine's
ads_synth / ads_synth_rows and the oracle's restated orc_synth_rows give the same
bits for any row set and thread count.  The bench's reference arm generates its
data with the oracle copy, so it never maps libadsann_b200.so; this pin is what
makes its workload the same as the GPU arm's."""
import numpy as np
import pytest

KINDS = [  # (kind, extra kwargs) as the configs use them
    (0, dict(center_scale=10.0, sigma=1.0)),
    (1, dict(center_lo=112.0, center_hi=144.0, sigma=21.0, decay=True)),
    (2, dict(center_lo=0.47, center_hi=0.53, sigma=0.12, decay=True)),
    (3, dict(center_scale=1.0, sigma=1.4)),
]


@pytest.mark.parametrize("kind,kw", KINDS)
def test_synth_rows_equal_full_generation_and_oracle(orc, kind, kw):
    import paper_2303_09855_b200 as ads

    n, d, comps = 20_000, 37, 50
    full = ads.synth(n, d, comps, 5, 1, kind=kind, **kw)
    for lo, count, stride in ((0, n, 1), (123, 4321, 1), (7, 1500, 13), (n - 1, 1, 1), (0, 0, 1)):
        rows = ads.synth_rows(n, d, comps, 5, 1, lo, count, stride, kind=kind, **kw)
        np.testing.assert_array_equal(rows, full[lo:lo + count * stride:stride][:count])
        for threads in (1, 3):
            o = orc.synth_rows(n, d, comps, 5, 1, lo, count, stride, kind=kind, threads=threads, **kw)
            np.testing.assert_array_equal(o, rows)


def test_synth_rows_component_major_and_roles(orc):
    import paper_2303_09855_b200 as ads

    n, d, comps = 9_000, 96, 64
    for role in (1, 2, 3):
        full = ads.synth(n, d, comps, 0, role, kind=3, sigma=1.4, assign_mode=1)
        o = orc.synth_rows(n, d, comps, 0, role, 100, 8000, 1, kind=3, sigma=1.4, assign_mode=1)
        np.testing.assert_array_equal(o, full[100:8100])


def test_synth_rows_range_errors(orc):
    import paper_2303_09855_b200 as ads

    with pytest.raises(ValueError):
        ads.synth_rows(100, 8, 4, 0, 1, 90, 11, 1)
    with pytest.raises(ValueError):
        orc.synth_rows(100, 8, 4, 0, 1, 0, 50, 3)
    with pytest.raises(ValueError):
        ads.synth_rows(100, 8, 4, 0, 1, 0, 10, 0)

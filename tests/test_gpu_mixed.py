"""The mixed scan (ADS_SCAN_MIXED=1: certified fp32 walkers + one exact fp64 warp,
lag-1 merge) against the oracle's lag-1 schedule (orc_ivf_query_lag), bit for bit:
ids, dists, dims, under several refresh schedules and both split modes."""
import os

import numpy as np
import pytest

from helpers import MODE_ID, make_fixture, oracle_index, gpu_index

pytestmark = pytest.mark.gpu


@pytest.fixture
def mixed_env():
    old = os.environ.get("ADS_SCAN_MIXED")
    os.environ["ADS_SCAN_MIXED"] = "1"
    yield
    if old is None:
        del os.environ["ADS_SCAN_MIXED"]
    else:
        os.environ["ADS_SCAN_MIXED"] = old


@pytest.mark.parametrize("n,d,k,K,nprobe", [(3000, 128, 40, 10, 7), (2500, 64, 30, 20, 9), (4000, 96, 50, 5, 12)])
@pytest.mark.parametrize("first,step", [(0, 256), (10, 64), (1, 1), (37, 5)])
def test_mixed_scan_matches_lag1_oracle(eng, orc, mixed_env, n, d, k, K, nprobe, first, step):
    raw, t, qr, qt, P = make_fixture(orc, n, d, 16, 23, 700 + d)
    lay = oracle_index(orc, raw, t, P, k, 701, d1=32)
    idx = gpu_index(eng, lay, P)
    f = first if first else K
    for mode in ("ad-split", "pd-split"):
        res = eng.ivf_query_batch(idx, qt, qr, K, nprobe, eng.IvfMode(MODE_ID[mode]),
                                  opts=eng.search_opts(first=first, step=step, warps_per_cta=4))
        for qi in range(qt.shape[0]):
            ids, dists, stats = orc.ivf_query(lay, qt[qi], qr[qi], K, nprobe, mode, 2.1, 32, f, step, lag=1)
            c = int(res.counts[qi])
            assert c == len(ids), (mode, qi)
            np.testing.assert_array_equal(res.ids[qi, :c], ids, err_msg=f"{mode} q={qi}")
            np.testing.assert_array_equal(res.dists[qi, :c], dists, err_msg=f"{mode} q={qi}")
            assert int(res.dims[qi]) == int(stats[0]), (mode, qi, int(res.dims[qi]), int(stats[0]))

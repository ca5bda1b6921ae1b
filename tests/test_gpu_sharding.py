"""GPU pieces of the list-sharded path: ads_ivf_subset, per-shard search and the
merge kernel, each bit-exact against the oracle / reference merge.  Ranks are
emulated one after another on one GPU (no cross-rank waiting)."""
import numpy as np
import pytest

from helpers import gpu_index, make_fixture, oracle_index
from shard_helpers import merge_ref, numpy_subset, shard_search_oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3, 8])
def test_shards_search_and_merge_bitexact(eng, orc, world):
    from paper_2303_09855_b200.shard import merge_topk, partition_lists, shard_index

    raw, t, qr, qt, P = make_fixture(orc, 4000, 64, 16, 30, 11)
    lay = oracle_index(orc, raw, t, P, 48, 12, d1=32)
    idx = gpu_index(eng, lay, P)
    owner = partition_lists(np.diff(lay["list_off"]), world)
    K, nprobe = 10, 16
    all_i = np.full((world, qt.shape[0], K), -1, np.int32)
    all_d = np.full((world, qt.shape[0], K), np.nan)
    for rank in range(world):
        sh = shard_index(idx, owner, rank)
        ref = numpy_subset(lay, owner, rank)
        ex = sh.export()
        np.testing.assert_array_equal(ex["list_off"], ref["list_off"])
        np.testing.assert_array_equal(ex["ids_flat"], ref["ids_flat"])
        np.testing.assert_array_equal(ex["a1_t"], ref["a1_t"])
        np.testing.assert_array_equal(ex["a2_raw"], ref["a2_raw"])
        res = eng.ivf_query_batch(sh, qt, qr, K, nprobe, eng.IvfMode.kAdSplit, first=K, step=64)
        ids, dists, dims = shard_search_oracle(orc, ref, qt, qr, K, nprobe, "ad-split", K, 64)
        np.testing.assert_array_equal(res.ids, ids)
        np.testing.assert_array_equal(np.nan_to_num(res.dists, nan=-1), np.nan_to_num(dists, nan=-1))
        np.testing.assert_array_equal(res.dims, dims)
        all_i[rank], all_d[rank] = res.ids, res.dists
    mi, md, mc = merge_topk(all_d, all_i, K)
    ri, rd = merge_ref(all_d, all_i, K)
    np.testing.assert_array_equal(mi, ri)
    np.testing.assert_array_equal(np.nan_to_num(md, nan=-1), np.nan_to_num(rd, nan=-1))
    assert np.array_equal(mc, (ri >= 0).sum(axis=1))

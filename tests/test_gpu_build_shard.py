"""Config 5's build and sharded search on the GPU, bit-exact against the oracle:

* the seeded-sample k-means init (ads_kmeans init 1) against orc_kmeans_init;
* the streamed builder (ads_ivf_builder_*: k-means on the strided sample, the
  certified nprobe-1 assignment of every row, the bucket layout, the keep mask of
  a shard) against the oracle's sample k-means, exact fp64 argmin and ivf_layout;
* ads_ivf_build_sampled_device (the one-piece form) against the streamed builder;
* a config-5-shaped index (unit sphere, D 96, 16 384 lists, 2 M rows) searched at
  nprobe 64 against orc_ivf_query on the exported index;
* the product's two-wave sharded step (shard.ShardedIvf: probe_lo / r0 waves, a real
  1-rank NCCL group, all-gather, merge kernel) against the oracle's restricted
  searches merged by (dist, id).
"""
import os
import socket

import numpy as np
import pytest

from shard_helpers import kth_distance, merge_ref, numpy_subset, shard_search_oracle

pytestmark = pytest.mark.gpu

SPHERE = dict(kind=3, center_scale=1.0, sigma=1.4)


def _gen(eng, n, d, comps, seed):
    def rows(lo, count, stride=1):
        return eng.synth_rows(n, d, comps, seed, 1, lo, count, stride, **SPHERE)
    return rows


def _lay_from_export(ex, n, d, k, d1=32):
    return {"n": n, "d": d, "k": k, "d1": d1, "split": True, "centroids_t": ex["centroids_t"],
            "centroids_raw": ex["centroids_t"], "list_off": ex["list_off"], "ids_flat": ex["ids_flat"],
            "a1_t": ex["a1_t"], "a2_t": ex["a2_t"], "a1_raw": ex["a1_t"], "a2_raw": ex["a2_t"],
            "vec_t": None, "vec_raw": None}


@pytest.mark.parametrize("n,d,k,iters,seed", [(3000, 24, 17, 8, 3), (20000, 96, 200, 5, 0)])
def test_kmeans_sample_init_bitexact(eng, orc, n, d, k, iters, seed):
    X = eng.synth(n, d, 40, seed, 1, **SPHERE)
    got = eng.kmeans(X, k, iters, seed, init=1)
    cent, asg, obj, it = orc.kmeans_init(X, k, iters, seed, 1)
    np.testing.assert_array_equal(got.centroids, cent)
    np.testing.assert_array_equal(got.assignment, asg)
    assert got.objective == obj and got.iterations == it


def test_streamed_build_matches_oracle(eng, orc):
    from paper_2303_09855_b200.shard import partition_lists

    n, d, comps, k, sample, iters, seed = 50_000, 96, 64, 100, 5_000, 6, 0
    m = eng.generate_orthogonal(d, seed)
    rows = _gen(eng, n, d, comps, seed)
    idx, sizes, cent = eng.build_ivf_streamed(rows, n, d, m, k, seed, 32, iters, sample, chunk=7_000)
    # oracle: the same rows from the restated generator, rotated by the oracle
    stride = n // sample
    S = orc.apply_dataset(m.entries, orc.synth_rows(n, d, comps, seed, 1, 0, sample, stride, **SPHERE))
    ocent, _, _, _ = orc.kmeans_init(S, k, iters, seed, 1)
    np.testing.assert_array_equal(cent, ocent)
    T = orc.apply_dataset(m.entries, orc.synth_rows(n, d, comps, seed, 1, 0, n, 1, **SPHERE))
    asg = orc.assign(T, ocent)
    np.testing.assert_array_equal(sizes, np.bincount(asg, minlength=k))
    lay = orc.ivf_layout(T, T, m.entries, ocent, asg, k, 32, True)
    ex = idx.export()
    for nm in ("centroids_t", "list_off", "ids_flat", "a1_t", "a2_t"):
        np.testing.assert_array_equal(ex[nm], lay[nm], err_msg=nm)
    # a shard's keep mask lays out exactly the owned lists (== ads_ivf_subset)
    owner = partition_lists(sizes, 3)
    for rank in range(3):
        sh, _, _ = eng.build_ivf_streamed(rows, n, d, m, k, seed, 32, iters, sample, chunk=11_000,
                                          owner=lambda s: partition_lists(s, 3), rank=rank)
        sub = numpy_subset(lay, owner, rank)
        es = sh.export()
        assert sh.n == sub["n"]
        for nm in ("list_off", "ids_flat", "a1_t", "a2_t"):
            np.testing.assert_array_equal(es[nm], sub[nm], err_msg=f"rank {rank} {nm}")


def test_build_sampled_device_equals_streamed(eng):
    n, d, comps, k, sample, iters, seed = 40_000, 96, 50, 80, 4_000, 4, 1
    m = eng.generate_orthogonal(d, seed)
    rows = _gen(eng, n, d, comps, seed)
    a, _, _ = eng.build_ivf_streamed(rows, n, d, m, k, seed, 32, iters, sample, chunk=9_999)
    ctx = eng.Context.default()
    dX = eng.DeviceArray.from_host(ctx, rows(0, n))
    dT = eng.DeviceArray(ctx, (n, d), np.float32)
    eng.Transform(m, ctx).apply_dataset_device(dX, dT)
    b = eng.build_ivf_sampled_device(dT, m, k, seed, 32, iters, sample, ctx=ctx)
    ea, eb = a.export(), b.export()
    for nm in ("centroids_t", "list_off", "ids_flat", "a1_t", "a2_t"):
        np.testing.assert_array_equal(ea[nm], eb[nm], err_msg=nm)
    with pytest.raises(ValueError):
        eng.build_ivf_sampled_device(dT, m, k, seed, 32, iters, k - 1, ctx=ctx)


@pytest.mark.slow
def test_config5_shape_search_vs_oracle(eng, orc):
    """Config 5's shape at 2 M rows: unit sphere, D 96, 16 384 lists (122 rows per list),
    nprobe 64, K 100, IVF++ at the engine's batched schedule (48 queries) and the
    reference's per-candidate schedule (6 queries), bit-exact."""
    from paper_2303_09855_b200 import configs

    cfg = configs.CONFIGS[5]
    n, d, k, nq = 2_000_000, cfg.d, cfg.nlist, 48
    m = eng.generate_orthogonal(d, cfg.seed)
    rows = _gen(eng, n, d, cfg.components, cfg.seed)
    idx, _, _ = eng.build_ivf_streamed(rows, n, d, m, k, cfg.seed, 32, 4, 400_000, chunk=500_000)
    q = eng.synth_rows(cfg.nq, d, cfg.components, cfg.seed, 2, 0, nq, 1, **SPHERE)
    qt = eng.apply_dataset(m, q)
    lay = _lay_from_export(idx.export(), idx.n, d, k)
    K, nprobe = cfg.K, cfg.nprobe
    res = eng.ivf_query_batch(idx, qt, None, K, nprobe, eng.IvfMode.kAdSplit)
    step = eng.search_plan(idx, K, nprobe, eng.IvfMode.kAdSplit)["step"]
    for i in range(nq):
        ids, dists, stats = orc.ivf_query(lay, qt[i], qt[i], K, nprobe, "ad-split", 2.1, 32, K, step)
        c = int(res.counts[i])
        assert c == len(ids) == K
        np.testing.assert_array_equal(res.ids[i, :c], ids, err_msg=f"q={i}")
        np.testing.assert_array_equal(res.dists[i, :c], dists, err_msg=f"q={i}")
        assert int(res.dims[i]) == int(stats[0]), i
    ref = eng.ivf_query_batch(idx, qt[:6], None, K, nprobe, eng.IvfMode.kAdSplit, first=1, step=1)
    for i in range(6):
        ids, dists, stats = orc.ivf_query(lay, qt[i], qt[i], K, nprobe, "ad-split", 2.1, 32, 1, 1)
        np.testing.assert_array_equal(ref.ids[i], ids)
        np.testing.assert_array_equal(ref.dists[i], dists)
        assert int(ref.dims[i]) == int(stats[0])


def _one_rank_nccl():
    import torch.distributed as dist

    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=None)
    return dist.group.WORLD


@pytest.mark.parametrize("waves", [0, 2, 5])
def test_sharded_step_world1_vs_oracle(eng, orc, waves):
    """The product's sharded step at world 1 over a real NCCL group: wave 1 over probe
    ranks [0, w), all-reduce (min) of the K-th distances, wave 2 from that bound, the
    all-gather and the merge kernel == the oracle's two restricted searches merged."""
    import torch

    from helpers import make_fixture, oracle_index
    from paper_2303_09855_b200.shard import ShardedIvf, partition_lists, shard_index

    torch.cuda.set_device(0)
    group = _one_rank_nccl()
    raw, t, qr, qt, P = make_fixture(orc, 5000, 64, 20, 40, 21)
    lay = oracle_index(orc, raw, t, P, 60, 22, d1=32)
    from helpers import gpu_index

    idx = gpu_index(eng, lay, P)
    owner = partition_lists(np.diff(lay["list_off"]), 1)
    sh = shard_index(idx, owner, 0)
    K, nprobe, step = 10, 16, 64
    S = ShardedIvf.on_device(sh, qt.shape[0], K, nprobe, 1, 0, group, waves=waves, step=step)
    dq = torch.from_numpy(qt).cuda()
    S.step(dq)
    sh.ctx.sync()
    w = S.w
    assert w == (waves if 0 < waves < nprobe else 0)
    if w:
        i1, d1, m1 = shard_search_oracle(orc, lay, qt, qr, K, w, "ad-split", K, step)
        R = kth_distance(d1, K)
        i2, d2, m2 = shard_search_oracle(orc, lay, qt, qr, K, nprobe, "ad-split", K, step, probe_lo=w, r0=R)
        np.testing.assert_array_equal(S.rb.cpu().numpy(), R)
        ei, ed = merge_ref(np.stack([d1, d2]), np.stack([i1, i2]), K)
        np.testing.assert_array_equal(S.lm.cpu().numpy().sum(axis=0), (m1 + m2).astype(np.int64))
    else:
        ei, ed, m = shard_search_oracle(orc, lay, qt, qr, K, nprobe, "ad-split", K, step)
    np.testing.assert_array_equal(S.oi.cpu().numpy(), ei)
    np.testing.assert_array_equal(np.nan_to_num(S.od.cpu().numpy(), nan=-1), np.nan_to_num(ed, nan=-1))


@pytest.mark.parametrize("waves", [0, 3])
def test_sharded_step_two_gpus(eng, orc, tmp_path, waves):
    """The product's sharded step across two GPUs over NCCL (runs when a 2-GPU lease
    exists; this pool's gpurun leases one GPU) == the oracle's per-shard restricted
    searches, the all-reduced bound and the (dist, id) merge."""
    import subprocess
    import sys

    from helpers import make_fixture, oracle_index
    from paper_2303_09855_b200.shard import partition_lists

    if eng.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    procs = [subprocess.Popen([sys.executable, os.path.join(root, "tests", "dist_gpu_shard_worker.py"), str(r), "2",
                               str(port), str(tmp_path), str(waves)]) for r in range(2)]
    for p in procs:
        assert p.wait(timeout=600) == 0
    g0, g1 = np.load(tmp_path / "g0.npz"), np.load(tmp_path / "g1.npz")
    np.testing.assert_array_equal(g0["ids"], g1["ids"])
    raw, t, qr, qt, P = make_fixture(orc, 6000, 64, 20, 40, 51)
    lay = oracle_index(orc, raw, t, P, 64, 52, d1=32)
    owner = partition_lists(np.diff(lay["list_off"]), 2)
    w = int(g0["w"])
    parts_i, parts_d, R = [], [], np.full(qt.shape[0], np.inf)
    subs = [numpy_subset(lay, owner, r) for r in range(2)]
    if w:
        for sub in subs:
            _, d1, _ = shard_search_oracle(orc, sub, qt, qr, 10, w, "ad-split", 10, 64)
            R = np.minimum(R, kth_distance(d1, 10))
        np.testing.assert_array_equal(g0["R"], R)
    for sub in subs:
        if w:
            i1, d1, _ = shard_search_oracle(orc, sub, qt, qr, 10, w, "ad-split", 10, 64)
            i2, d2, _ = shard_search_oracle(orc, sub, qt, qr, 10, 16, "ad-split", 10, 64, probe_lo=w, r0=R)
            parts_i += [i1, i2]
            parts_d += [d1, d2]
        else:
            i1, d1, _ = shard_search_oracle(orc, sub, qt, qr, 10, 16, "ad-split", 10, 64)
            parts_i.append(i1)
            parts_d.append(d1)
    ei, ed = merge_ref(np.stack(parts_d), np.stack(parts_i), 10)
    np.testing.assert_array_equal(g0["ids"], ei)
    np.testing.assert_array_equal(np.nan_to_num(g0["dists"], nan=-1), np.nan_to_num(ed, nan=-1))

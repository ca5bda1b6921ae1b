"""One rank of the 2-process gloo test of the list-sharded search (CPU).
Per-rank search runs on the oracle (test infrastructure); the product pieces
under test are the partition (shard.partition_lists), the restricted-stream
semantics of a shard, and the orchestration of the product's sharded step
(shard.ShardedIvf: two waves, all-reduce of the bound, all-gather, merge)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def run(rank, world, port, outdir):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from helpers import make_fixture, oracle_index
    from oracle import load_oracle
    from paper_2303_09855_b200.shard import partition_lists
    from shard_helpers import numpy_subset, shard_search_oracle

    orc = load_oracle()
    raw, t, qr, qt, P = make_fixture(orc, 3000, 32, 12, 24, 17)
    lay = oracle_index(orc, raw, t, P, 40, 18, d1=8)
    owner = partition_lists(np.diff(lay["list_off"]), world)
    sub = numpy_subset(lay, owner, rank)
    K, nprobe = 10, 12
    ids, dists, dims = shard_search_oracle(orc, sub, qt, qr, K, nprobe, "ad-split", K, 64)
    gi = [torch.zeros(ids.shape, dtype=torch.int32) for _ in range(world)]
    gd = [torch.zeros(dists.shape, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gi, torch.from_numpy(ids))
    dist.all_gather(gd, torch.from_numpy(dists))
    all_ids = np.stack([x.numpy() for x in gi])
    all_d = np.stack([x.numpy() for x in gd])
    # the product's list-sharded step (shard.ShardedIvf: wave 1 over probe ranks [0, w),
    # all-reduce (min) of the K-th distances, wave 2 over [w, nprobe) from that bound,
    # all-gather + merge), driven here with gloo and an oracle-backed per-rank search
    from paper_2303_09855_b200.shard import ShardedIvf
    from shard_helpers import OracleShardSearch

    be = OracleShardSearch(orc, sub, qt, qr, K, K, 64)
    one = ShardedIvf(be, qt.shape[0], qt.shape[1], K, nprobe, world, rank, dist.group.WORLD, waves=0)
    one.step(None)
    two = ShardedIvf(be, qt.shape[0], qt.shape[1], K, nprobe, world, rank, dist.group.WORLD, waves=3)
    two.step(None)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), ids=all_ids, dists=all_d, owner=owner,
             dims=dims, R=two.rb.numpy(), wave_ids=two.gi.numpy(), wave_dists=two.gd.numpy(),
             wave_dims=two.lm.numpy().sum(axis=0), one_ids=one.oi.numpy(), one_dists=one.od.numpy(),
             two_ids=two.oi.numpy(), two_dists=two.od.numpy())
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    run(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4])

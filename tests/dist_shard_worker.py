"""One rank of the 2-process gloo test of the list-sharded search (CPU).
Per-rank search runs on the oracle (test infrastructure); the product pieces
under test are the partition (shard.partition_lists), the restricted-stream
semantics of a shard and the all-gather -> (dist, id) merge contract."""
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
    # the threshold exchange (bench.py's list-sharded step for N > 1): wave 1 over probe
    # ranks [0, w), all-reduce (min) of the K-th distances, wave 2 over [w, nprobe) from it
    from shard_helpers import kth_distance

    w = 3
    i1, d1, m1 = shard_search_oracle(orc, sub, qt, qr, K, w, "ad-split", K, 64)
    R = torch.from_numpy(kth_distance(d1, K))
    dist.all_reduce(R, op=dist.ReduceOp.MIN)
    i2, d2, m2 = shard_search_oracle(orc, sub, qt, qr, K, nprobe, "ad-split", K, 64, probe_lo=w, r0=R.numpy())
    wi = [torch.zeros((2,) + ids.shape, dtype=torch.int32) for _ in range(world)]
    wd = [torch.zeros((2,) + dists.shape, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(wi, torch.from_numpy(np.stack([i1, i2])))
    dist.all_gather(wd, torch.from_numpy(np.stack([d1, d2])))
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), ids=all_ids, dists=all_d, owner=owner,
             dims=dims, R=R.numpy(), wave_ids=np.stack([x.numpy() for x in wi]).reshape(-1, *ids.shape),
             wave_dists=np.stack([x.numpy() for x in wd]).reshape(-1, *dists.shape),
             wave_dims=m1 + m2)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    run(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4])

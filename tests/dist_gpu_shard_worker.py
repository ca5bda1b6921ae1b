"""One rank of the 2-GPU NCCL test of the product's list-sharded step
(tests/test_gpu_build_shard.py::test_sharded_step_two_gpus): every rank builds the
same small index on its own GPU, keeps its lists (partition_lists + shard_index),
runs shard.ShardedIvf over a real NCCL group and saves the merged result."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def run(rank, world, port, outdir, waves):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    import paper_2303_09855_b200 as ads
    from helpers import make_fixture, oracle_index
    from oracle import load_oracle
    from paper_2303_09855_b200.shard import ShardedIvf, partition_lists, shard_index

    orc = load_oracle()
    raw, t, qr, qt, P = make_fixture(orc, 6000, 64, 20, 40, 51)
    lay = oracle_index(orc, raw, t, P, 64, 52, d1=32)
    ctx = ads.Context.default(rank)
    idx = ads.IvfIndex.from_arrays(
        n=lay["n"], d=lay["d"], k_clusters=lay["k"], d1=lay["d1"], layout=1, centroids_t=lay["centroids_t"],
        list_off=lay["list_off"], ids_flat=lay["ids_flat"], vec_t=lay["vec_t"], a1_t=lay["a1_t"],
        a2_t=lay["a2_t"], P=P, ctx=ctx)
    owner = partition_lists(np.diff(lay["list_off"]), world)
    sh = shard_index(idx, owner, rank)
    S = ShardedIvf.on_device(sh, qt.shape[0], 10, 16, world, rank, dist.group.WORLD, waves=waves, step=64)
    S.step(torch.from_numpy(qt).cuda())
    torch.cuda.synchronize()
    np.savez(os.path.join(outdir, f"g{rank}.npz"), ids=S.oi.cpu().numpy(), dists=S.od.cpu().numpy(),
             R=S.rb.cpu().numpy(), owner=owner, w=S.w)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    run(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5]))

"""Worker for tests/test_gpu_multiproc.py (launched by torch.distributed.run, gloo, every rank on
cuda:0): the fused cfg5 exchange across real processes -- CUDA IPC receive buffers mapped by
PeerBuffers, every rank's scatter storing straight into its owners' buffers -- against the
all-to-all order computed on the host from every rank's keys."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def splitmix_keys(i0, n):
    x = np.arange(i0, i0 + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9e3779b97f4a7c15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xbf58476d1ce4e5b9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94d049bb133111eb)
        x = x ^ (x >> np.uint64(31))
    return (x >> np.uint64(32)).astype(np.uint32)


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    import paper_1507_01391_b200 as dmm
    from paper_1507_01391_b200.distributed import PeerBuffers, bucket_owner, global_partition_p2p, p2p_capacity
    sizes = [300000 + 12345 * r for r in range(world)]  # ragged shards
    starts = np.concatenate([[0], np.cumsum(sizes)])
    keys = dmm.gen_keys(int(starts[rank]), sizes[rank])
    peers = PeerBuffers(p2p_capacity(max(sizes), world))
    ok = True
    for rep in range(3):  # the buffers are reused across calls
        peers.local.fill_(-1)
        dist.barrier()
        got, counts = global_partition_p2p(keys, peers)
        host = dmm.as_uint32(got)
        exp = []
        for s in range(world):
            h = splitmix_keys(int(starts[s]), sizes[s])
            lab = h >> 29
            loc = h[np.argsort(lab, kind="stable")]
            own = [b for b in range(8) if bucket_owner(b, 8, world) == rank]
            exp.append(loc[np.isin(loc >> 29, own)])
        exp = np.concatenate(exp)
        ok = ok and host.shape == exp.shape and bool((host == exp).all())
        ok = ok and int(counts.sum()) == sum(sizes)
    res = torch.tensor([int(ok)])
    dist.all_reduce(res, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("P2P_MULTIPROC", "ok" if int(res) else "FAIL", world)
    dist.barrier()
    dist.destroy_process_group()
    return 0 if int(res) else 1


if __name__ == "__main__":
    sys.exit(main())

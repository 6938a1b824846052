"""CPU (gloo, world_size 2) tests of the multi-GPU host logic: instance sharding, max-over-ranks
timing and cfg5's all-to-all exchange of a bucket-major partition (the GPU path runs the same
functions over NCCL)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1507_01391_b200.distributed import (bucket_owner, exchange_partitioned, max_over_ranks, send_splits,
                                               shard_range)


def test_shard_range_covers_everything_once():
    for total in (0, 1, 7, 65536, 2 ** 18 + 3):
        for world in (1, 2, 4, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and b - a >= d - c >= b - a - 1


def test_send_splits_and_owners():
    assert [bucket_owner(b, 8, 8) for b in range(8)] == list(range(8))
    assert [bucket_owner(b, 8, 2) for b in range(8)] == [0, 0, 0, 0, 1, 1, 1, 1]
    assert send_splits([1, 2, 3, 4, 5, 6, 7, 8], 2) == [10, 26]
    assert send_splits([1, 2, 3, 4, 5, 6, 7, 8], 1) == [36]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(100 + rank)
    keys = rng.integers(0, 2 ** 32, size=n, dtype=np.uint64).astype(np.uint32)
    labels = keys >> 29
    order = np.argsort(labels, kind="stable")  # reference-free restatement of the local step
    local = keys[order]
    counts = np.bincount(labels, minlength=8).tolist()
    out = exchange_partitioned(torch.from_numpy(local.view(np.int32)), counts)
    t = max_over_ranks(float(rank + 1))
    q.put((rank, out.numpy().view(np.uint32).copy(), t))
    dist.destroy_process_group()


def test_global_partition_exchange_gloo_world2():
    world, n = 2, 5000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, out, t = q.get(timeout=120)
        res[r] = (out, t)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    allkeys = np.concatenate([np.random.default_rng(100 + r).integers(0, 2 ** 32, size=n, dtype=np.uint64)
                              .astype(np.uint32) for r in range(world)])
    for r in range(world):
        out, t = res[r]
        assert t == float(world)  # max over ranks
        labels = out >> 29
        assert all(bucket_owner(int(b), 8, world) == r for b in np.unique(labels))
        # stable by (source rank, source index) within each label
        exp = []
        for src in range(world):
            k = np.random.default_rng(100 + src).integers(0, 2 ** 32, size=n, dtype=np.uint64).astype(np.uint32)
            lab = k >> 29
            keep = np.array([bucket_owner(int(b), 8, world) == r for b in lab])
            sel = k[keep]
            exp.append(sel[np.argsort(sel >> 29, kind="stable")])
        assert (out == np.concatenate(exp)).all()
    assert sum(len(res[r][0]) for r in range(world)) == len(allkeys)


def _simulate_fused_scatter(keys_by_rank, world, nb=8, shift=29):
    """Numpy model of dmm_multisplit_scatter_to driven by p2p_destinations: every rank writes its
    bucket-b keys (stable) to owner(b)'s buffer from dst_base[b] on."""
    from paper_1507_01391_b200.distributed import p2p_destinations, recv_counts
    counts = torch.from_numpy(np.stack([np.bincount(k >> shift, minlength=nb) for k in keys_by_rank]).astype(np.int64))
    recv = recv_counts(counts).tolist()
    bufs = [np.full(recv[r], -1, dtype=np.int64) for r in range(world)]
    for s, k in enumerate(keys_by_rank):
        base = p2p_destinations(counts, s).tolist()
        lab = k >> shift
        for b in range(nb):
            mine = k[lab == b]
            o = bucket_owner(b, nb, world)
            assert (bufs[o][base[b]: base[b] + len(mine)] == -1).all()  # no overlap
            bufs[o][base[b]: base[b] + len(mine)] = mine
    assert all((b >= 0).all() for b in bufs)  # every slot written
    return bufs


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_fused_exchange_positions_match_all_to_all_order(world):
    # the fused scatter's destinations reproduce the all-to-all's (source rank, source index)
    # order exactly, for any world size
    rng = np.random.default_rng(world)
    keys = [rng.integers(0, 2 ** 32, size=int(rng.integers(0, 3000)), dtype=np.uint64).astype(np.uint32)
            for _ in range(world)]
    bufs = _simulate_fused_scatter(keys, world)
    for r in range(world):
        exp = []
        for k in keys:
            lab = k >> 29
            loc = k[np.argsort(lab, kind="stable")]
            exp.append(loc[[bucket_owner(int(x), 8, world) == r for x in (loc >> 29)]])
        assert (bufs[r] == np.concatenate(exp).astype(np.int64)).all()


def _worker_fused(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1507_01391_b200.distributed import p2p_destinations, recv_counts
    rng = np.random.default_rng(200 + rank)
    keys = rng.integers(0, 2 ** 32, size=n + 37 * rank, dtype=np.uint64).astype(np.uint32)
    counts = torch.tensor(np.bincount(keys >> 29, minlength=8), dtype=torch.int64)
    gathered = [torch.empty_like(counts) for _ in range(world)]
    dist.all_gather(gathered, counts)  # the count exchange of global_partition_p2p
    all_counts = torch.stack(gathered)
    base = p2p_destinations(all_counts, rank)
    recv = recv_counts(all_counts)
    # the reference exchange (all-to-all) this rank would receive
    local = keys[np.argsort(keys >> 29, kind="stable")]
    out = exchange_partitioned(torch.from_numpy(local.view(np.int32)), counts.tolist())
    q.put((rank, base.numpy(), recv.numpy(), out.numpy().view(np.uint32).copy()))
    dist.destroy_process_group()


def test_fused_exchange_offsets_gloo_world2():
    world, n = 2, 4000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_fused, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, base, recv, out = q.get(timeout=120)
        res[r] = (base, recv, out)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    keys = [np.random.default_rng(200 + r).integers(0, 2 ** 32, size=n + 37 * r, dtype=np.uint64).astype(np.uint32)
            for r in range(world)]
    bufs = _simulate_fused_scatter(keys, world)
    for r in range(world):
        base, recv, out = res[r]
        assert recv[r] == len(out)
        # what the fused scatter puts in rank r's buffer == what the all-to-all delivered
        assert (bufs[r] == out.astype(np.int64)).all()

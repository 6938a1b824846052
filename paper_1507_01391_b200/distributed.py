"""Multi-GPU plumbing, one process per GPU over torch.distributed.

* Batched configs (cfg1-cfg4): instances are independent, so each rank takes a contiguous
  instance range (`shard_range`) and there is no collective in the data path; only the
  timing uses a barrier + max-over-ranks reduction (`max_over_ranks`).
* cfg5, the global w-way partition of one large array: every rank stably partitions its
  keys into `nbuckets` label buckets on its GPU (dmm_multisplit), then one all-to-all
  (NCCL over NVLink on GPUs; gloo in the CPU tests) sends bucket j to the rank that owns
  label j.  Rank r receives its labels ordered by (source rank, source index).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) share of `total` units for `rank` (sizes differ by at most one)."""
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank float (device timing) over the group; identity without one."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def bucket_owner(bucket: int, nbuckets: int, world: int) -> int:
    """Rank that owns label `bucket` (contiguous label ranges per rank)."""
    return bucket * world // nbuckets


def send_splits(bucket_counts: list[int], world: int) -> list[int]:
    """Keys this rank sends to each rank, given its per-bucket counts (buckets are bucket-major
    and owners are monotone in the bucket index, so each destination's keys are contiguous)."""
    nb = len(bucket_counts)
    out = [0] * world
    for b, c in enumerate(bucket_counts):
        out[bucket_owner(b, nb, world)] += int(c)
    return out


def exchange_partitioned(local: torch.Tensor, bucket_counts: list[int], group=None) -> torch.Tensor:
    """All-to-all of a bucket-major locally partitioned array: returns the keys of every rank
    whose labels this rank owns, ordered by (source rank, source order)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return local
    splits = send_splits(bucket_counts, world)
    dev = local.device
    send_t = torch.tensor(splits, dtype=torch.int64, device=dev)
    recv_t = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_to_all_single(recv_t, send_t, group=group)
    recv = recv_t.tolist()
    out = torch.empty(sum(recv), dtype=local.dtype, device=dev)
    dist.all_to_all_single(out, local, output_split_sizes=recv, input_split_sizes=splits, group=group)
    return out


def global_partition(keys: torch.Tensor, nbuckets: int = 8, shift: int = 29, group=None):
    """cfg5 on GPUs: local stable multisplit (libdmm_b200) + NCCL all-to-all.
    Returns (received keys, local bucket counts)."""
    from . import dmm
    local, starts = dmm.multisplit(keys, nbuckets, shift)
    s = starts.tolist() + [keys.numel()]
    counts = [s[b + 1] - s[b] for b in range(nbuckets)]
    return exchange_partitioned(local, counts, group), counts

"""Multi-GPU plumbing, one process per GPU over torch.distributed.

* Batched configs (cfg1-cfg4): instances are independent, so each rank takes a contiguous
  instance range (`shard_range`) and there is no collective in the data path; only the
  timing uses a barrier + max-over-ranks reduction (`max_over_ranks`).
* cfg5, the global w-way partition of one large array: every rank stably partitions its
  keys into `nbuckets` label buckets on its GPU (dmm_multisplit), then one all-to-all
  (NCCL over NVLink on GPUs; gloo in the CPU tests) sends bucket j to the rank that owns
  label j.  Rank r receives its labels ordered by (source rank, source index).
* cfg5 fused (`global_partition_p2p`): the exchange is folded into the partition's scatter --
  after a tiny all-gather of per-rank bucket counts, every rank's scatter kernel writes each
  key straight into its owner's receive buffer (peer memory over NVLink, mapped once with CUDA
  IPC by `PeerBuffers`) at the position the all-to-all would have put it; no local staging
  array, no second pass over the keys.  Same output as `global_partition`, key for key.
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


_OWNER_CACHE: dict = {}


def _owner_tables(nb: int, world: int, device):
    """(owner [nb], same-owner [nb, nb], same-owner-and-earlier [nb, nb]) int64 tensors, cached."""
    key = (nb, world, str(device))
    if key not in _OWNER_CACHE:
        owner = torch.tensor([bucket_owner(b, nb, world) for b in range(nb)], device=device)
        same = owner.view(-1, 1) == owner.view(1, -1)
        idx = torch.arange(nb, device=device)
        earlier = idx.view(1, -1) < idx.view(-1, 1)  # [b, b']: b' < b
        _OWNER_CACHE[key] = (owner, same.to(torch.int64), (same & earlier).to(torch.int64))
    return _OWNER_CACHE[key]


def p2p_destinations(all_counts: torch.Tensor, rank: int) -> torch.Tensor:
    """dst_base[b]: where this rank's bucket-b keys start in the receive buffer of the bucket's
    owner, given every rank's bucket counts C [world, nbuckets].  The owner's buffer holds the
    all-to-all order -- source rank by source rank, each source's buckets in bucket order:
    base = sum_{s < rank} sum_{b' owned by r} C[s, b'] + sum_{b' < b owned by r} C[rank, b']."""
    world, nb = all_counts.shape
    c = all_counts.to(torch.int64)
    _, same, same_earlier = _owner_tables(nb, world, c.device)
    from_lower_ranks = c[:rank].sum(dim=0)  # zeros for rank 0
    # (integer matrix-vector products as broadcast sums: CUDA has no int64 matmul)
    return (same * from_lower_ranks.view(1, -1)).sum(dim=1) + (same_earlier * c[rank].view(1, -1)).sum(dim=1)


def recv_counts(all_counts: torch.Tensor) -> torch.Tensor:
    """Keys each rank receives (int64 [world])."""
    world, nb = all_counts.shape
    owner, _, _ = _owner_tables(nb, world, all_counts.device)
    out = torch.zeros(world, dtype=torch.int64, device=all_counts.device)
    return out.index_add_(0, owner, all_counts.to(torch.int64).sum(dim=0))


last_launches = 0  # kernels the last global_partition_p2p call launched


def p2p_capacity(keys_per_rank: int, world: int, nbuckets: int = 8, slack: float = 1.05) -> int:
    """Receive-buffer size for uniformly distributed labels: the largest label share a rank owns
    times all keys, with slack (global_partition_p2p raises if a rank would receive more)."""
    owned = max(sum(1 for b in range(nbuckets) if bucket_owner(b, nbuckets, world) == r) for r in range(world))
    return int(keys_per_rank * world * owned / nbuckets * slack) + 4096


class PeerBuffers:
    """One receive buffer per rank (int32, `capacity` keys), mapped into every rank's address
    space: CUDA IPC handles of the caching allocator's block are exchanged once through the
    process group; `ptrs` (int64, device) holds every rank's buffer address as seen from this
    rank.  Peer access over NVLink is enabled by the IPC open."""

    def __init__(self, capacity: int, group=None, device=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.capacity = int(capacity)
        self.local = torch.empty(self.capacity, dtype=torch.int32, device=dev)
        self.peers = [None] * self.world
        self.peers[self.rank] = self.local
        if self.world > 1:
            st = self.local.untyped_storage()
            handle = st._share_cuda_()
            offset = self.local.storage_offset() * self.local.element_size()
            handles = [None] * self.world
            dist.all_gather_object(handles, (handle, offset), group=group)
            for r, (h, off) in enumerate(handles):
                if r == self.rank:
                    continue
                storage = torch.UntypedStorage._new_shared_cuda(*h)
                t = torch.empty(0, dtype=torch.int32, device=dev)
                t.set_(storage, off // 4, (self.capacity,))
                self.peers[r] = t
        self.ptrs = torch.tensor([p.data_ptr() for p in self.peers], dtype=torch.int64, device=dev)


def global_partition_p2p(keys: torch.Tensor, peers: PeerBuffers, nbuckets: int = 8, shift: int = 29,
                         group=None, workspace: torch.Tensor | None = None):
    """cfg5 with the all-to-all fused into the scatter (see module doc).  Returns (this rank's
    received keys -- a view of peers.local --, all ranks' bucket counts [world, nbuckets])."""
    from . import dmm
    k = keys.reshape(-1)
    n = k.numel()
    dev = k.device
    ws = workspace
    if ws is None or ws.numel() < int(dmm.lib().dmm_multisplit_workspace_bytes(n, nbuckets)):
        ws = torch.empty(int(dmm.lib().dmm_multisplit_workspace_bytes(n, nbuckets)), dtype=torch.uint8, device=dev)
    starts = torch.empty(nbuckets, dtype=torch.int64, device=dev)
    dmm.multisplit_count(k, nbuckets, shift, starts, ws)
    launches = int(dmm.lib().dmm_last_launch_count())
    counts = torch.empty_like(starts)
    counts[:-1] = starts[1:] - starts[:-1]
    counts[-1:] = n - starts[-1:]
    world = peers.world
    if world > 1:
        all_counts = torch.empty((world, nbuckets), dtype=torch.int64, device=dev)
        if dist.get_backend(group) == "gloo":  # host collective (several ranks on one GPU in tests)
            parts = [torch.empty(nbuckets, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(parts, counts.cpu(), group=group)
            all_counts.copy_(torch.stack(parts))
        else:
            dist.all_gather_into_tensor(all_counts, counts, group=group)
    else:
        all_counts = counts.view(1, -1)
    recv = recv_counts(all_counts).tolist()  # the one host sync: sizes for the capacity check
    if max(recv) > peers.capacity:
        raise RuntimeError(f"global_partition_p2p: a rank receives {max(recv)} keys, "
                           f"receive buffers hold {peers.capacity}")
    dst_base = p2p_destinations(all_counts, peers.rank)
    owner, _, _ = _owner_tables(nbuckets, world, dev)
    dst_ptrs = peers.ptrs[owner]
    dmm.multisplit_scatter_to(k, nbuckets, shift, dst_ptrs, dst_base, ws)
    global last_launches
    last_launches = launches + int(dmm.lib().dmm_last_launch_count())
    if world > 1:
        # every rank's stores into this rank's buffer have landed before it is read
        torch.cuda.current_stream().synchronize()
        dist.barrier(group=group)
    return peers.local[: recv[peers.rank]], all_counts

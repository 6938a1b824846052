"""Python mirror of the reference's hot-path API over the B200 C ABI.

Names and argument meaning follow /root/reference/proj/include/dmm/*.hpp
(partition_general, integer_sort_general, sort_tall, permute, to_column_major, ...);
the error behaviour mirrors the reference's exception hierarchy (core.hpp:59-78):
shape contracts raise before launch, data-dependent failures (PostconditionFailed,
InvalidInstance, KeyOutOfRange) raise after the batch completes, naming the
first failing instance.

Inputs are batches ``[count, w, m]`` (or a single ``[w, m]`` grid) of uint32 words
held as ``torch.int32`` on the GPU (numpy arrays are copied over).  Device memory
and streams come from PyTorch; every computation runs in libdmm_b200.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

_LIB: C.CDLL | None = None


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        _LIB = _lib.load()
    return _LIB


# --------------------------------------------------------------------------------------
# Errors (core.hpp:59-78)
# --------------------------------------------------------------------------------------
class Error(RuntimeError):
    status = 11


class ConflictViolation(Error):
    status = 13


class OverlappingViews(ConflictViolation):
    status = 10


class ShapeViolation(Error):
    status = 1


class InvalidInstance(Error):
    status = 2


class KeyOutOfRange(Error):
    status = 3


class DivisibilityViolation(Error):
    status = 4


class PostconditionFailed(Error):
    status = 5


class PackingOverflow(Error):
    status = 6


class CapacityExceeded(Error):
    status = 7


class NotSquare(Error):
    status = 8


class OutOfBounds(Error):
    status = 9


class NotBijective(Error):
    status = 12


class UnsupportedShape(Error):
    """The reference accepts the shape but no B200 kernel is built for it (no fallback)."""
    status = 64


class CudaError(Error):
    status = 66


_BY_STATUS = {c.status: c for c in (ShapeViolation, InvalidInstance, KeyOutOfRange, DivisibilityViolation,
                                     PostconditionFailed, PackingOverflow, CapacityExceeded, NotSquare,
                                     OutOfBounds, OverlappingViews, NotBijective, ConflictViolation,
                                     UnsupportedShape, CudaError)}
_BY_STATUS[11] = Error
_BY_STATUS[65] = ValueError

FLAG_EXT_PARTIAL_GROUPS = 1
FLAG_NONSTRICT = 2
FLAG_NO_ENFORCE_PRE = 4


def _check(status: int, where: str) -> None:
    if status != 0:
        cls = _BY_STATUS.get(status, Error)
        msg = lib().dmm_last_error().decode()
        raise cls(f"{where}: status {status}" + (f" ({msg})" if msg else ""))


# --------------------------------------------------------------------------------------
# Tensor plumbing
# --------------------------------------------------------------------------------------
def _as_batch(grid) -> tuple[torch.Tensor, bool]:
    """-> (contiguous int32 CUDA tensor [count, w, m], was_single_grid)."""
    if isinstance(grid, np.ndarray):
        a = np.ascontiguousarray(grid)
        if a.dtype != np.uint32:
            if a.size and (a.min() < 0 or a.max() >= 2 ** 32):
                raise KeyOutOfRange("words must fit in 32 bits (the B200 layout narrows the reference's u64 words)")
            a = a.astype(np.uint32)
        t = torch.from_numpy(a.view(np.int32)).cuda()
    elif isinstance(grid, torch.Tensor):
        t = grid
        if t.dtype in (torch.int64, torch.uint32):
            t = t.to(torch.int64)
            if t.numel() and (int(t.min()) < 0 or int(t.max()) >= 2 ** 32):
                raise KeyOutOfRange("words must fit in 32 bits")
            t = (t & 0xFFFFFFFF).to(torch.int64)
            t = torch.where(t >= 2 ** 31, t - 2 ** 32, t).to(torch.int32)
        elif t.dtype != torch.int32:
            raise TypeError(f"unsupported dtype {t.dtype}")
        if not t.is_cuda:
            t = t.cuda()
        t = t.contiguous()
    else:
        raise TypeError("grid must be a numpy array or a torch tensor")
    single = t.dim() == 2
    if single:
        t = t.unsqueeze(0)
    if t.dim() != 3:
        raise ShapeViolation("grid must be [w, m] or [count, w, m]")
    return t, single


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


def as_uint32(t: torch.Tensor) -> np.ndarray:
    """Device int32 tensor -> host numpy uint32 (bit reinterpretation)."""
    return t.detach().cpu().numpy().view(np.uint32)


def _raise_first(status: torch.Tensor, where: str) -> None:
    bad = torch.nonzero(status != 0)
    if bad.numel():
        k = int(bad[0, 0])
        s = int(status[k])
        cls = _BY_STATUS.get(s, Error)
        raise cls(f"{where}: instance {k} failed with status {s}")


@dataclass
class GeneralStats:
    """GeneralStats partition.hpp:292-295, per instance."""
    cleanup_retries: torch.Tensor  # int32 [count]
    sorted_raw: torch.Tensor       # int32 [count] (0 / 1 as written by the kernel)
    status: torch.Tensor           # uint8 [count] (dmm_status)
    # PartitionProbe capture (probe=True): [count, snaps, w, m] windows after every
    # after_balance / after_divide hook of the outer recursion, in hook order
    snapshots: torch.Tensor | None = None

    @property
    def sorted(self) -> torch.Tensor:  # bool [count]; computed on access (no extra kernel per call)
        return self.sorted_raw != 0


# --------------------------------------------------------------------------------------
# Instance generation (instance.hpp:48-76)
# --------------------------------------------------------------------------------------
KIND_SORT_U32, KIND_PARTITION, KIND_PERMUTE = 0, 1, 2


def gen_instances(kind: int, w: int, m: int, seed0: int, count: int, stream=None) -> torch.Tensor:
    """gen_instance(kind, w, m, seed0 + k) for k < count, on the device (bit-exact)."""
    out = torch.empty((count, w, m), dtype=torch.int32, device="cuda")
    _check(lib().dmm_gen_instances(kind, w, m, seed0, count, out.data_ptr(), _stream(stream)), "gen_instances")
    return out


def gen_keys(index0: int, n: int, stream=None) -> torch.Tensor:
    """cfg5 keys: splitmix64(index0 + i) >> 32 for i < n (uint32 bits in an int32 tensor)."""
    out = torch.empty((n,), dtype=torch.int32, device="cuda")
    _check(lib().dmm_gen_keys(index0, n, out.data_ptr(), _stream(stream)), "gen_keys")
    return out


# --------------------------------------------------------------------------------------
# Partition / integer sort (partition.hpp:436-456)
# --------------------------------------------------------------------------------------
def _general(fn_name: str, grid, domain: int | None, flags: int, out, stream, check: bool, probe: bool = False):
    t, single = _as_batch(grid)
    count, w, m = t.shape
    res = out if out is not None else torch.empty_like(t)
    stats = torch.empty((count, 2), dtype=torch.int32, device=t.device)
    status = torch.empty((count,), dtype=torch.uint8, device=t.device)
    L = lib()
    snaps = None
    if probe:
        ns = int(L.dmm_general_probe_snaps(w, m, flags))
        snaps = torch.zeros((count, ns, w, m), dtype=torch.int32, device=t.device)
        pp = snaps.data_ptr() if ns else None
    if fn_name == "partition_general":
        if probe:
            st = L.dmm_partition_general_probe(t.data_ptr(), res.data_ptr(), w, m, count, flags, stats.data_ptr(),
                                               status.data_ptr(), pp, ns, _stream(stream))
        else:
            st = L.dmm_partition_general(t.data_ptr(), res.data_ptr(), w, m, count, flags, stats.data_ptr(),
                                         status.data_ptr(), _stream(stream))
    else:
        if probe:
            st = L.dmm_integer_sort_general_probe(t.data_ptr(), res.data_ptr(), w, m, count, domain, flags,
                                                  stats.data_ptr(), status.data_ptr(), pp, ns, _stream(stream))
        else:
            st = L.dmm_integer_sort_general(t.data_ptr(), res.data_ptr(), w, m, count, domain, flags,
                                            stats.data_ptr(), status.data_ptr(), _stream(stream))
    _check(st, fn_name)
    gs = GeneralStats(stats[:, 0], stats[:, 1], status, snaps[0] if (single and snaps is not None) else snaps)
    if check:
        _raise_first(status, fn_name)
    return (res[0] if single else res), gs


def partition_general(grid, *, flags: int = 0, out=None, stream=None, check: bool = True, probe: bool = False):
    """GeneralStats partition_general(const MatrixView&)  partition.hpp:453-456.

    Labels in [0, w), m copies each.  Returns (partitioned grid(s), GeneralStats).
    flags: FLAG_EXT_PARTIAL_GROUPS accepts shapes like 32 x 8 that the reference's
    balance() rejects; FLAG_NONSTRICT = MachineConfig.strict false.
    """
    return _general("partition_general", grid, None, flags, out, stream, check, probe)


def integer_sort_general(grid, domain: int, *, enforce_analysis_pre: bool = True, flags: int = 0, out=None,
                         stream=None, check: bool = True, probe: bool = False):
    """GeneralStats integer_sort_general(view, domain, probe, enforce_analysis_pre)  partition.hpp:436-449.

    probe=True captures the PartitionProbe hook points (after_balance / after_divide of the
    outer recursion) as GeneralStats.snapshots."""
    if not enforce_analysis_pre:
        flags |= FLAG_NO_ENFORCE_PRE
    return _general("integer_sort_general", grid, domain, flags, out, stream, check, probe)


def _simple(fn_name: str, grid, *args, out=None, stream=None, w_arg_only: bool = False):
    t, single = _as_batch(grid)
    count, w, m = t.shape
    res = out if out is not None else torch.empty_like(t)
    fn = getattr(lib(), "dmm_" + fn_name)
    if w_arg_only:
        st = fn(t.data_ptr(), res.data_ptr(), w, count, *args, _stream(stream))
    else:
        st = fn(t.data_ptr(), res.data_ptr(), w, m, count, *args, _stream(stream))
    _check(st, fn_name)
    return res[0] if single else res


def _partition_entry(fn_name: str, grid, out, stream, check: bool):
    t, single = _as_batch(grid)
    res = out if out is not None else torch.empty_like(t)
    count, w, m = t.shape
    status = torch.empty((count,), dtype=torch.uint8, device=t.device)
    _check(getattr(lib(), "dmm_" + fn_name)(t.data_ptr(), res.data_ptr(), w, m, count, status.data_ptr(),
                                            _stream(stream)), fn_name)
    if check:
        _raise_first(status, fn_name)
    return res[0] if single else res


def partition_square(grid, *, out=None, stream=None, check: bool = True):
    """void partition_square(const MatrixView&)  partition.hpp:189-197 (w = m, m a perfect
    square; w < 32 machines run 32 / w per warp)."""
    return _partition_entry("partition_square", grid, out, stream, check)


def partition_short_wide(grid, *, out=None, stream=None, check: bool = True):
    """void partition_short_wide(const MatrixView&, hook)  partition.hpp:178-185 (w^2 <= m)."""
    return _partition_entry("partition_short_wide", grid, out, stream, check)


def short_wide_probe(grid, *, partition: bool, ascending: bool = True, stream=None, check: bool = True):
    """The ShortWideHook stages (sort.hpp:189-218) of partition_short_wide (partition=True) or
    sort_short_wide(ascending): -> (result [count, w, m], snapshots [count, 3, w, m]) with the
    machine after_first_convert, after_first_pass and done."""
    t, single = _as_batch(grid)
    count, w, m = t.shape
    res = torch.empty_like(t)
    snaps = torch.empty((count, 3, w, m), dtype=torch.int32, device=t.device)
    status = torch.zeros((count,), dtype=torch.uint8, device=t.device)
    _check(lib().dmm_short_wide_probe(t.data_ptr(), res.data_ptr(), w, m, count, int(partition), int(ascending),
                                      status.data_ptr(), snaps.data_ptr(), _stream(stream)), "short_wide_probe")
    if check:
        _raise_first(status, "short_wide_probe")
    return (res[0], snaps[0]) if single else (res, snaps)


# --------------------------------------------------------------------------------------
# Comparison sorts (sort.hpp) and layout primitives (layout.hpp)
# --------------------------------------------------------------------------------------
def sort_wide_any(grid, ascending: bool = True, **kw):
    """detail::sort_wide_any(view, asc)  sort.hpp:321-330 (w <= m, w | m)."""
    return _simple("sort_wide_any", grid, int(ascending), **kw)


def sort_tall(grid, **kw):
    """void sort_tall(const MatrixView&)  sort.hpp:352-374 (w >= m, m | w)."""
    return _simple("sort_tall", grid, **kw)


def sort_square(grid, ascending: bool = True, **kw):
    """void sort_square(view, ascending)  sort.hpp:337-346."""
    return _simple("sort_square", grid, int(ascending), **kw)


def sort_short_wide(grid, ascending: bool = True, **kw):
    """void sort_short_wide(view, ascending, hook)  sort.hpp:225-230."""
    return _simple("sort_short_wide", grid, int(ascending), **kw)


def transpose_square(grid, **kw):
    """transpose_square layout.hpp:24-61."""
    return _simple("transpose_square", grid, w_arg_only=True, **kw)


def to_column_major(grid, **kw):
    """to_column_major layout.hpp:397-399."""
    return _simple("to_column_major", grid, **kw)


def to_row_major(grid, **kw):
    """to_row_major layout.hpp:403-405."""
    return _simple("to_row_major", grid, **kw)


ORDER_ASC, ORDER_DESC, ORDER_ALT, ORDER_ALT_DESC = 0, 1, 2, 3


def sort_rows(grid, order: int = ORDER_ASC, domain: int = 0, *, out=None, stream=None, check: bool = True):
    """radix_sort_rows(view, domain, order) partition.hpp:94 / sort_rows(view, order) sort.hpp:76."""
    t, single = _as_batch(grid)
    count, w, m = t.shape
    res = out if out is not None else torch.empty_like(t)
    status = torch.empty((count,), dtype=torch.uint8, device=t.device)
    _check(lib().dmm_sort_rows(t.data_ptr(), res.data_ptr(), w, m, count, order, domain, status.data_ptr(),
                               _stream(stream)), "sort_rows")
    if check:
        _raise_first(status, "sort_rows")
    return res[0] if single else res


# --------------------------------------------------------------------------------------
# Randomized permutation (permute.hpp:545-628)
# --------------------------------------------------------------------------------------
@dataclass
class PermuteReports:
    """PermuteReport permute.hpp:62-72, per instance."""
    iterations: np.ndarray
    fallback: np.ndarray
    used_packing: np.ndarray
    packed_width: np.ndarray
    threshold: np.ndarray
    random_words: np.ndarray
    cleanup_retries: np.ndarray
    leftover_history: list
    shifts: np.ndarray
    status: np.ndarray

    def report(self, k: int) -> dict:
        return {"iterations": int(self.iterations[k]), "fallback": bool(self.fallback[k]),
                "used_packing": bool(self.used_packing[k]), "packed_width": int(self.packed_width[k]),
                "threshold": int(self.threshold[k]), "random_words": int(self.random_words[k]),
                "cleanup_retries": int(self.cleanup_retries[k]), "leftover_history": self.leftover_history[k],
                "shifts": self.shifts[k].tolist()}


def permute(grid, seeds, alpha: int = 4, iter_cap: int = 64, *, out=None, stream=None, check: bool = True):
    """PermuteReport permute(Machine&, Rng&, const PermuteParams&)  permute.hpp:545-628.

    grid: [count, w, m] label bijections; seeds: count seeds of each instance's Rng.
    Returns (output regions [count, w, m], PermuteReports).
    """
    t, single = _as_batch(grid)
    count, w, m = t.shape
    sd = torch.as_tensor(np.asarray(seeds, dtype=np.uint64).view(np.int64).reshape(-1), device="cuda")
    if sd.numel() != count:
        raise ValueError("one seed per instance")
    res = out if out is not None else torch.empty_like(t)
    reps = torch.zeros((count, 5), dtype=torch.int64, device="cuda")  # 40-byte dmm_permute_report
    hist = torch.zeros((count, 64), dtype=torch.int64, device="cuda")
    shifts = torch.zeros((count, w), dtype=torch.int32, device="cuda")
    status = torch.zeros((count,), dtype=torch.uint8, device="cuda")
    L = lib()
    ws = torch.empty((max(1, int(L.dmm_permute_workspace_bytes(w, m, count))),), dtype=torch.uint8, device="cuda")
    _check(L.dmm_permute(t.data_ptr(), res.data_ptr(), w, m, count, sd.data_ptr(), alpha, iter_cap, reps.data_ptr(),
                         hist.data_ptr(), shifts.data_ptr(), status.data_ptr(), ws.data_ptr(), _stream(stream)),
           "permute")
    if check:
        _raise_first(status, "permute")
    r = reps.cpu().numpy().view(np.uint32).reshape(count, 10)
    r64 = reps.cpu().numpy().view(np.uint64).reshape(count, 5)
    n_hist = r[:, 9]
    h = hist.cpu().numpy().view(np.uint64)
    rep = PermuteReports(iterations=r[:, 0], fallback=r[:, 1], used_packing=r[:, 2], packed_width=r[:, 3],
                         threshold=r64[:, 2], random_words=r64[:, 3], cleanup_retries=r[:, 8],
                         leftover_history=[h[k, : n_hist[k]].tolist() for k in range(count)],
                         shifts=shifts.cpu().numpy().view(np.uint32), status=status.cpu().numpy())
    return (res[0] if single else res), rep


def permute_steps(grid, seeds, alpha: int = 4, iter_cap: int = 64, stream=None) -> torch.Tensor:
    """Machine::steps() after permute(Machine&, Rng&) for each instance (what run_algorithm reports,
    instance.hpp:357): int64 [count] (0 where not modelled).  Off the hot path (dmm_permute_steps)."""
    t, _ = _as_batch(grid)
    count, w, m = t.shape
    sd = torch.as_tensor(np.asarray(seeds, dtype=np.uint64).astype(np.int64), device=t.device)
    steps = torch.zeros(count, dtype=torch.int64, device=t.device)
    _check(lib().dmm_permute_steps(t.data_ptr(), w, m, count, sd.data_ptr(), alpha, iter_cap, steps.data_ptr(),
                                   _stream(stream)), "permute_steps")
    return steps


def permute_into(src: torch.Tensor, dst: torch.Tensor, seeds, bufs: dict, alpha: int = 4, iter_cap: int = 64,
                 stream=None):
    """Allocation-free permute over device tensors (bench / pipelines): reports, history,
    shifts and status land in the reusable buffers of `bufs`; nothing is copied to the host.
    Returns the status tensor."""
    count, w, m = src.shape
    if "seeds" not in bufs or bufs["seeds"].numel() != count:
        bufs["seeds"] = torch.as_tensor(np.asarray(seeds, dtype=np.uint64).view(np.int64), device="cuda")
    if "reps" not in bufs or bufs["reps"].shape[0] != count:
        bufs["reps"] = torch.zeros((count, 5), dtype=torch.int64, device="cuda")
        bufs["hist"] = torch.zeros((count, 64), dtype=torch.int64, device="cuda")
        bufs["shifts"] = torch.zeros((count, w), dtype=torch.int32, device="cuda")
        bufs["status"] = torch.zeros((count,), dtype=torch.uint8, device="cuda")
    _check(lib().dmm_permute(src.data_ptr(), dst.data_ptr(), w, m, count, bufs["seeds"].data_ptr(), alpha, iter_cap,
                             bufs["reps"].data_ptr(), bufs["hist"].data_ptr(), bufs["shifts"].data_ptr(),
                             bufs["status"].data_ptr(), None, _stream(stream)), "permute")
    return None, bufs["status"]


def multisplit(keys: torch.Tensor, nbuckets: int = 8, shift: int = 29, out=None, stream=None):
    """Stable bucket-major partition of a flat key array by label (key >> shift) & (nbuckets-1)
    (the local step of the global w-way partition, cfg5).  Returns (out, bucket_starts[nbuckets])."""
    k = keys.reshape(-1)
    if k.dtype != torch.int32 or not k.is_cuda:
        raise TypeError("keys must be a CUDA int32 (uint32 bits) tensor")
    n = k.numel()
    res = out if out is not None else torch.empty_like(k)
    starts = torch.zeros((nbuckets,), dtype=torch.int64, device=k.device)
    ws = torch.empty((int(lib().dmm_multisplit_workspace_bytes(n, nbuckets)),), dtype=torch.uint8, device=k.device)
    _check(lib().dmm_multisplit(k.data_ptr(), n, shift, nbuckets, res.data_ptr(), starts.data_ptr(), ws.data_ptr(),
                                _stream(stream)), "multisplit")
    return res, starts


def multisplit_count(keys: torch.Tensor, nbuckets: int, shift: int, starts: torch.Tensor, workspace: torch.Tensor,
                     stream=None) -> None:
    """First half of the fused partition + exchange: bucket starts of the local bucket-major
    order into ``starts`` (int64 [nbuckets], device); the tile offsets stay in ``workspace``
    (dmm_multisplit_workspace_bytes) for multisplit_scatter_to."""
    k = keys.reshape(-1)
    _check(lib().dmm_multisplit_count(k.data_ptr(), k.numel(), shift, nbuckets, starts.data_ptr(),
                                      workspace.data_ptr(), _stream(stream)), "multisplit_count")


def multisplit_scatter_to(keys: torch.Tensor, nbuckets: int, shift: int, dst_ptrs: torch.Tensor,
                          dst_base: torch.Tensor, workspace: torch.Tensor, stream=None) -> None:
    """Second half: bucket b's keys (stable) to the device array at dst_ptrs[b] (int64 device
    pointers, e.g. peer receive buffers) from element dst_base[b] on."""
    k = keys.reshape(-1)
    _check(lib().dmm_multisplit_scatter_to(k.data_ptr(), k.numel(), shift, nbuckets, dst_ptrs.data_ptr(),
                                           dst_base.data_ptr(), workspace.data_ptr(), _stream(stream)),
           "multisplit_scatter_to")


def version() -> str:
    return lib().dmm_version().decode()


def supported(algorithm: str, w: int, m: int) -> bool:
    return bool(lib().dmm_supported(algorithm.encode(), w, m))

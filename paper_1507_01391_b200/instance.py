"""Instances, their text format and the run_algorithm dispatcher -- the Python mirror of
/root/reference/proj/include/dmm/instance.hpp (the layer the reference's CLI and acceptance
harness drive).

* ``Instance`` / ``gen_instance`` / ``validate_instance``   instance.hpp:38-100
* ``instance_to_text`` / ``instance_from_text`` / ``load_instance`` / ``save_instance``
  instance.hpp:102-142 (header ``"kind w m seed"``, then one row per line; parsing is
  whitespace-token based like the reference's ``operator>>``)
* ``Algorithm`` names, ``instance_kind_for``, ``RunReport`` (``summary``, ``csv_header``,
  ``csv_line``), ``run_algorithm``   instance.hpp:146-363

``run_algorithms`` is the batched form: every instance of one shape goes through ONE kernel
launch (the B200 way to run the reference's per-instance loop).  Verification follows the
reference's independent verifiers (instance.hpp:236-273) and runs on the device.

Differences from the reference, by construction: words are 32-bit on the device (a loaded
instance holding a word >= 2^32 raises KeyOutOfRange); ``gen_instance("sort", ...)`` emits
the uint32 sort tile of include/dmm_gpu.h (the reference's sort kind draws 64-bit words);
``RunReport.steps`` / ``work`` are the reference's exact counts where the schedule is
data-independent (``modelled_steps``), for the w <= m leaves of the general partition /
integer sort (``leaf_steps``), for the w > m recursion (``general_steps``, cleanup retries
included) and for the comparison sorts (``sort_steps``), all replayed on the device; 0 for the
permutation;
``record_trace=True`` raises TraceIncomplete.
"""
from __future__ import annotations

import io
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import dmm

KINDS = ("sort", "partition", "permute")
_KIND_ID = {"sort": dmm.KIND_SORT_U32, "partition": dmm.KIND_PARTITION, "permute": dmm.KIND_PERMUTE}

ALGORITHMS = ("sort_short_wide", "sort_square", "sort_tall", "partition_short_wide", "partition_square",
              "partition_general", "integer_sort_general", "permute")


class TraceIncomplete(dmm.Error):
    """core.hpp:69 -- raised for record_trace: the kernels record no DMM trace."""
    status = -2


@dataclass
class Instance:
    """struct Instance instance.hpp:38-44: kind name, shape, seed and the row-major grid."""
    kind: str = "sort"
    w: int = 1
    m: int = 1
    seed: int = 0
    grid: np.ndarray = field(default_factory=lambda: np.zeros((1, 1), dtype=np.uint64))

    def __post_init__(self):
        self.grid = np.asarray(self.grid, dtype=np.uint64).reshape(-1)


def kind_from_name(s: str) -> str:
    """kind_from_name instance.hpp:29-37."""
    if s not in KINDS:
        raise dmm.InvalidInstance("unknown instance kind: " + s)
    return s


def gen_instances(kind: str, w: int, m: int, seed0: int, count: int) -> list[Instance]:
    """gen_instance(kind, w, m, seed0 + k) for k < count (instance.hpp:48-76), generated on the
    device by the bit-exact generator of include/dmm_gpu.h and copied to the host."""
    if w < 1 or m < 1:
        raise dmm.ShapeViolation("instances need w >= 1, m >= 1")
    g = dmm.as_uint32(dmm.gen_instances(_KIND_ID[kind_from_name(kind)], w, m, seed0, count))
    return [Instance(kind, w, m, seed0 + k, g[k].astype(np.uint64)) for k in range(count)]


def gen_instance(kind: str, w: int, m: int, seed: int) -> Instance:
    return gen_instances(kind, w, m, seed, 1)[0]


def validate_instance(inst: Instance) -> None:
    """validate_instance instance.hpp:79-100 (raises InvalidInstance)."""
    g = inst.grid
    if g.size != inst.w * inst.m:
        raise dmm.InvalidInstance("grid size does not match w*m")
    if inst.kind == "partition":
        if g.size and int(g.max()) >= inst.w:
            raise dmm.InvalidInstance("partition label outside [0, w)")
        if (np.bincount(g.astype(np.int64), minlength=inst.w) != inst.m).any():
            raise dmm.InvalidInstance("partition labels are not m copies each")
    elif inst.kind == "permute":
        if g.size and int(g.max()) >= g.size:
            raise dmm.InvalidInstance("permute labels are not a bijection")
        if (np.bincount(g.astype(np.int64), minlength=g.size) != 1).any():
            raise dmm.InvalidInstance("permute labels are not a bijection")


def instance_to_text(inst: Instance) -> str:
    """instance_to_text instance.hpp:103-115."""
    rows = inst.grid.reshape(inst.w, inst.m)
    lines = [f"{inst.kind} {inst.w} {inst.m} {inst.seed}"]
    lines += [" ".join(str(int(x)) for x in r) for r in rows]
    return "\n".join(lines) + "\n"


def _u(tok: str, bits: int) -> int:
    v = int(tok)
    if v < 0 or v >= (1 << bits):
        raise ValueError(tok)
    return v


def instance_from_text(src) -> Instance:
    """instance_from_text instance.hpp:117-128; ``src`` is a string or a text stream."""
    toks = (src.read() if isinstance(src, io.TextIOBase) or hasattr(src, "read") else str(src)).split()
    try:
        kind, w, m, seed = toks[0], _u(toks[1], 32), _u(toks[2], 32), _u(toks[3], 64)
    except (IndexError, ValueError):
        raise dmm.InvalidInstance("malformed instance header") from None
    kind = kind_from_name(kind)
    n = w * m
    body = toks[4:4 + n]
    try:
        vals = [_u(t, 64) for t in body]
    except ValueError:
        vals = None
    if vals is None or len(vals) < n:
        raise dmm.InvalidInstance("instance grid truncated")
    return Instance(kind, w, m, seed, np.array(vals, dtype=np.uint64))


def load_instance(path: str | os.PathLike) -> Instance:
    """load_instance instance.hpp:130-135."""
    try:
        with open(path) as f:
            return instance_from_text(f)
    except OSError:
        raise dmm.Error(f"cannot open instance file: {path}") from None


def save_instance(inst: Instance, path: str | os.PathLike) -> None:
    """save_instance instance.hpp:137-142."""
    try:
        with open(path, "w") as f:
            f.write(instance_to_text(inst))
    except OSError:
        raise dmm.Error(f"cannot write instance file: {path}") from None


def instance_kind_for(alg: str) -> str:
    """instance_kind_for instance.hpp:188-201."""
    if alg.startswith("sort_"):
        return "sort"
    if alg.startswith("partition_"):
        return "partition"
    if alg in ("integer_sort_general", "permute"):
        return "permute"  # permutation labels double as integer keys
    raise ValueError(f"unknown algorithm {alg!r}")


@dataclass
class RunReport:
    """struct RunReport instance.hpp:211-231."""
    algorithm: str = ""
    w: int = 0
    m: int = 0
    seed: int = 0
    steps: int = 0
    work: int = 0
    conflicts: int = 0
    correct: bool = False
    iterations: int = 0
    fallback: bool = False
    cleanup_retries: int = 0

    def summary(self) -> str:
        return (f"algorithm={self.algorithm} w={self.w} m={self.m} seed={self.seed} steps={self.steps} "
                f"work={self.work} conflicts={self.conflicts} correct={int(self.correct)} "
                f"iterations={self.iterations} fallback={int(self.fallback)} "
                f"cleanup_retries={self.cleanup_retries}")


def csv_header() -> str:
    """csv_header instance.hpp:233-235."""
    return "algorithm,w,m,seed,steps,work,conflicts,correct,iterations,fallback"


def csv_line(r: RunReport) -> str:
    """csv_line instance.hpp:237-243."""
    return (f"{r.algorithm},{r.w},{r.m},{r.seed},{r.steps},{r.work},{r.conflicts},{int(r.correct)},"
            f"{r.iterations},{int(r.fallback)}")


@dataclass
class RunOutcome:
    """struct RunOutcome instance.hpp:277-281 (no trace); ``result`` is the final grid (the
    view snapshot, or the out region for permute) as uint64 [w, m]."""
    report: RunReport
    pipeline: dict | None = None
    result: np.ndarray | None = None


def modelled_steps(alg: str, w: int, m: int) -> int:
    """Machine::steps() of one run where the reference's count does not depend on the data
    (dmm_modelled_steps: radix leaves -- partition_short_wide, partition_square, and
    partition_general / integer_sort_general with w <= m on short-wide or square shapes);
    0 otherwise (merge segment sorts, cleanup retries, the permutation's iterations)."""
    return int(dmm.lib().dmm_modelled_steps(alg.encode(), w, m))


def leaf_metered(w: int, m: int) -> bool:
    """dmm_leaf_steps meters this w <= m leaf (shearsort, or square skeleton with w < m)."""
    if not (2 <= w <= 32 and m <= 128 and w <= m) or w * w <= m:
        return False
    h = int(round(m ** 0.5))
    if h * h == m:
        return w < m and w % h == 0
    return m % w == 0


def leaf_steps(grid: torch.Tensor, domain: int) -> torch.Tensor:
    """Machine::steps() of the general partition / integer sort leaf (w <= m) for each input
    instance of ``grid`` ([count, w, m] device), replayed on the device (dmm_leaf_steps)."""
    count, w, m = grid.shape
    out = torch.empty(count, dtype=torch.int64, device=grid.device)
    dmm._check(dmm.lib().dmm_leaf_steps(grid.data_ptr(), w, m, count, domain, out.data_ptr(),
                                        dmm._stream(None)), "leaf_steps")
    return out


def general_metered(w: int, m: int) -> bool:
    """dmm_general_steps meters this recursion shape (w > m; it rejects what general_sort_shape_ok
    rejects, as the kernels did before it is called)."""
    return w > m >= 2 and w * m <= 65536


def general_steps(grid: torch.Tensor, domain: int) -> tuple[torch.Tensor, torch.Tensor]:
    """(Machine::steps(), GeneralStats::cleanup_retries) of partition_general / integer_sort_general
    for each input instance of ``grid`` ([count, w, m] device, keys < domain), the w > m recursion
    included: the reference's states replayed on the device (dmm_general_steps)."""
    count, w, m = grid.shape
    steps = torch.empty(count, dtype=torch.int64, device=grid.device)
    retries = torch.empty(count, dtype=torch.int32, device=grid.device)
    dmm._check(dmm.lib().dmm_general_steps(grid.data_ptr(), w, m, count, domain, steps.data_ptr(),
                                           retries.data_ptr(), dmm._stream(None)), "general_steps")
    return steps, retries


def sort_metered(alg: str, w: int, m: int) -> bool:
    """dmm_sort_steps meters this comparison sort (sort_short_wide w^2 <= m <= 64,
    sort_square w = m = h^2 <= 64, sort_tall m | w with w in {32, 64, 128} or w = m <= 32)."""
    h = int(round(m ** 0.5))
    if alg == "sort_short_wide":
        return w >= 2 and w * w <= m <= 64
    if alg == "sort_tall":
        return m >= 1 and w >= m and w % m == 0 and m <= 32 and (w in (32, 64, 128) or w == m)
    return alg == "sort_square" and w == m and h * h == m and 2 <= m <= 64


def sort_steps(alg: str, grid: torch.Tensor) -> torch.Tensor:
    """Machine::steps() of sort_short_wide / sort_square / sort_tall for each input instance."""
    count, w, m = grid.shape
    out = torch.empty(count, dtype=torch.int64, device=grid.device)
    dmm._check(dmm.lib().dmm_sort_steps(alg.encode(), grid.data_ptr(), w, m, count, out.data_ptr(),
                                        dmm._stream(None)), "sort_steps")
    return out


def run_algorithms(alg: str, instances: list[Instance], *, strict: bool = True, alpha: int = 4,
                   seeds=None, record_trace: bool = False) -> list[RunOutcome]:
    """run_algorithm (instance.hpp:283-363) over a batch of same-shape instances in one launch.

    Same checks as the reference (kind match, validate_instance, then the algorithm's own shape
    contracts raised by the kernels' C ABI), same verification and report fields."""
    if alg not in ALGORITHMS:
        raise ValueError(f"unknown algorithm {alg!r}")
    if not instances:
        return []
    want = instance_kind_for(alg)
    w, m = instances[0].w, instances[0].m
    for inst in instances:
        if inst.kind != want:
            raise dmm.InvalidInstance(f"algorithm {alg} needs a {want} instance")
        validate_instance(inst)
        if (inst.w, inst.m) != (w, m):
            raise dmm.ShapeViolation("run_algorithms needs instances of one shape")
    if record_trace:
        raise TraceIncomplete("B200 kernels record no DMM trace (no step meter)")
    seeds = [inst.seed for inst in instances] if seeds is None else [int(s) for s in seeds]
    host = np.stack([inst.grid.reshape(w, m) for inst in instances])
    if host.size and int(host.max()) >= 1 << 32:
        raise dmm.KeyOutOfRange("words must fit in 32 bits (the B200 layout narrows the reference's u64 words)")
    grid = torch.from_numpy(host.astype(np.uint32).view(np.int32)).cuda()
    count = len(instances)
    flags = 0 if strict else dmm.FLAG_NONSTRICT
    retries = [0] * count
    pipeline = [None] * count
    iters = [0] * count
    fallback = [False] * count
    if alg == "sort_short_wide":
        out = dmm.sort_short_wide(grid)
    elif alg == "sort_square":
        out = dmm.sort_square(grid)
    elif alg == "sort_tall":
        out = dmm.sort_tall(grid)
    elif alg == "partition_short_wide":
        out = dmm.partition_short_wide(grid)
    elif alg == "partition_square":
        out = dmm.partition_square(grid)
    elif alg in ("partition_general", "integer_sort_general"):
        if alg == "partition_general":
            out, st = dmm.partition_general(grid, flags=flags)
        else:
            out, st = dmm.integer_sort_general(grid, w * m, flags=flags)
        retries = st.cleanup_retries.cpu().tolist()
    else:
        out, reps = dmm.permute(grid, seeds, alpha=alpha)
        pipeline = [reps.report(k) for k in range(count)]
        iters = [p["iterations"] for p in pipeline]
        fallback = [p["fallback"] for p in pipeline]
        retries = [p["cleanup_retries"] for p in pipeline]
    # the reference's independent verifiers (instance.hpp:246-273), on the device
    o = out.to(torch.int64) & 0xFFFFFFFF
    if want == "sort" or alg == "integer_sort_general":
        expect = torch.sort((grid.to(torch.int64) & 0xFFFFFFFF).reshape(count, -1), dim=1).values
        ok = (o.reshape(count, -1) == expect).all(dim=1)
    elif want == "partition":
        rows = torch.arange(w, device=o.device, dtype=torch.int64).view(1, w, 1)
        ok = (o == rows).all(dim=2).all(dim=1)
    else:
        ids = torch.arange(w * m, device=o.device, dtype=torch.int64).view(1, w, m)
        ok = (o == ids).all(dim=2).all(dim=1)
    ok = ok.cpu().tolist()
    steps = [modelled_steps(alg, w, m)] * count
    if steps[0] == 0 and alg in ("partition_general", "integer_sort_general") and leaf_metered(w, m):
        steps = leaf_steps(grid, w if alg == "partition_general" else w * m).cpu().tolist()
    elif steps[0] == 0 and alg in ("partition_general", "integer_sort_general") and general_metered(w, m):
        steps = general_steps(grid, w if alg == "partition_general" else w * m)[0].cpu().tolist()
    elif alg in ("sort_short_wide", "sort_square", "sort_tall") and sort_metered(alg, w, m):
        steps = sort_steps(alg, grid).cpu().tolist()
    elif alg == "permute":
        # the kernel's phase replay + the finish sort's meter (dmm_permute_steps)
        steps = dmm.permute_steps(grid, seeds, alpha=alpha).cpu().tolist()
    res = o.cpu().numpy().astype(np.uint64)
    outs = []
    for k in range(count):
        rep = RunReport(algorithm=alg, w=w, m=m, seed=seeds[k], steps=int(steps[k]), work=int(steps[k]) * w,
                        correct=bool(ok[k]),
                        iterations=int(iters[k]), fallback=bool(fallback[k]), cleanup_retries=int(retries[k]))
        outs.append(RunOutcome(rep, pipeline[k], res[k]))
    return outs


def run_algorithm(alg: str, inst: Instance, *, strict: bool = True, alpha: int = 4, seed: int | None = None,
                  record_trace: bool = False) -> RunOutcome:
    """RunOutcome run_algorithm(Algorithm, const Instance&, const RunOptions&)  instance.hpp:283-363."""
    return run_algorithms(alg, [inst], strict=strict, alpha=alpha, seeds=None if seed is None else [seed],
                          record_trace=record_trace)[0]

"""Offline conflict-free schedules for fixed permutations -- the Python mirror of
/root/reference/proj/include/dmm/layout.hpp:66-302.

* ``Move`` / ``Schedule`` (``validate``)             layout.hpp:66-95
* ``offline_schedule(W, M, perm)``                   layout.hpp:207-230 -- host precompute in
  libdmm_b200.so (dmm_offline_schedule), the reference's rounds move for move
* ``apply_schedule(grid, schedule)``                 layout.hpp:246-263 -- B200 kernel
  (dmm_apply_schedule): one warp per machine, DMM bank b = shared-memory bank b, so every round
  is one conflict-free load and one conflict-free store
* ``schedule_to_text`` / ``schedule_from_text``      layout.hpp:268-302

``perm`` follows the reference: ``perm[r*M + c] = (dst_bank, dst_off)`` of cell (r, c)
(a list of pairs or an integer array of shape [W*M, 2]).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np
import torch

from . import dmm


class Move(NamedTuple):
    """struct Move layout.hpp:66-71."""
    src_bank: int
    src_off: int
    dst_bank: int
    dst_off: int


@dataclass
class Schedule:
    """struct Schedule layout.hpp:76-95: rounds of moves; inside a round, source banks and
    destination banks are pairwise distinct, so a round is two conflict-free steps."""
    rounds: list = field(default_factory=list)

    def validate(self, W: int, M: int) -> None:
        for rnd in self.rounds:
            srcs, dsts = set(), set()
            for mv in rnd:
                if mv[0] >= W or mv[2] >= W or mv[1] >= M or mv[3] >= M:
                    raise dmm.OutOfBounds("schedule move outside shape")
                if mv[0] in srcs or mv[2] in dsts:
                    raise dmm.ConflictViolation("schedule round reuses a bank")
                srcs.add(mv[0])
                dsts.add(mv[2])

    def upload(self, device="cuda") -> "DeviceSchedule":
        """The schedule in device memory, in dmm_apply_schedule's layout (moves int32 [n, 4],
        round_start int32 [rounds + 1]); upload once, apply many times."""
        flat = [tuple(mv) for rnd in self.rounds for mv in rnd]
        moves = np.array(flat, dtype=np.uint32).reshape(-1, 4) if flat else np.zeros((1, 4), dtype=np.uint32)
        starts = np.zeros(len(self.rounds) + 1, dtype=np.uint32)
        starts[1:] = np.cumsum([len(r) for r in self.rounds])
        return DeviceSchedule(torch.from_numpy(moves.view(np.int32)).to(device),
                              torch.from_numpy(starts.view(np.int32)).to(device), len(self.rounds), len(flat))


@dataclass
class DeviceSchedule:
    """A Schedule uploaded by Schedule.upload."""
    moves: torch.Tensor
    round_start: torch.Tensor
    n_rounds: int
    n_moves: int


def _perm_array(W: int, M: int, perm) -> np.ndarray:
    p = np.asarray(perm, dtype=np.int64)
    if p.size != 2 * W * M:
        raise dmm.NotBijective("permutation table has wrong size")
    if p.size and p.min() < 0:
        raise dmm.NotBijective("permutation target out of range")
    return np.ascontiguousarray(p.reshape(-1).astype(np.uint32))


def offline_schedule(W: int, M: int, perm) -> Schedule:
    """Schedule offline_schedule(W, M, perm)  layout.hpp:207-230 (host precompute): M rounds of
    W moves from the Euler-split / matching decomposition of the bank transfer multigraph.
    Raises NotBijective on a table that is not a bijection of [W] x [M]."""
    p = _perm_array(W, M, perm)
    moves = np.zeros(max(4 * W * M, 4), dtype=np.uint32)
    dmm._check(dmm.lib().dmm_offline_schedule(W, M, p.ctypes.data, moves.ctypes.data), "offline_schedule")
    mv = moves[: 4 * W * M].reshape(-1, 4).tolist()
    return Schedule([[Move(*x) for x in mv[k * W:(k + 1) * W]] for k in range(M if W else 0)])


def apply_schedule(grid, schedule, *, out=None, stream=None, check: bool = True):
    """apply_schedule(view, schedule, dst_base)  layout.hpp:246-263 on a batch of machines:
    out(dst) = grid(src) for every move, rounds in order; cells no move writes keep ``out``'s
    contents (zeros when ``out`` is None).  ``schedule``: a Schedule or a DeviceSchedule
    (Schedule.upload) to skip the per-call upload.  Raises OutOfBounds / ConflictViolation (checked on the
    device before any write) like Schedule::validate."""
    t, single = dmm._as_batch(grid)
    count, w, m = t.shape
    res = out if out is not None else torch.zeros_like(t)
    ds = schedule if isinstance(schedule, DeviceSchedule) else schedule.upload(t.device)
    status = torch.empty((1,), dtype=torch.uint8, device=t.device)
    dmm._check(dmm.lib().dmm_apply_schedule(t.data_ptr(), res.data_ptr(), w, m, count, ds.moves.data_ptr(),
                                            ds.round_start.data_ptr(), ds.n_rounds, ds.n_moves, status.data_ptr(),
                                            dmm._stream(stream)), "apply_schedule")
    if check:
        s = int(status.item())
        if s:
            raise dmm._BY_STATUS.get(s, dmm.Error)(f"apply_schedule: status {s}")
    return res[0] if single else res


def schedule_to_text(s: Schedule) -> str:
    """schedule_to_text layout.hpp:268-278: one "src_bank src_off dst_bank dst_off" line per
    move, a blank line between rounds."""
    parts = []
    for i, rnd in enumerate(s.rounds):
        if i:
            parts.append("\n")
        parts.extend(f"{a} {b} {c} {d}\n" for a, b, c, d in rnd)
    return "".join(parts)


def schedule_from_text(text: str) -> Schedule:
    """schedule_from_text layout.hpp:280-302 (blank lines separate rounds; empty rounds vanish)."""
    rounds, cur = [], []
    for line in text.split("\n"):
        if line == "":
            if cur:
                rounds.append(cur)
            cur = []
            continue
        toks = line.split()
        try:
            vals = [int(x) for x in toks[:4]]
            if len(vals) < 4 or min(vals) < 0:
                raise ValueError
        except ValueError:
            raise dmm.Error("malformed schedule line: " + line) from None
        cur.append(Move(*vals))
    if cur:
        rounds.append(cur)
    return Schedule(rounds)

"""DMM access traces: the reference's trace text format and its offline CAC audit
(/root/reference/proj/include/dmm/core.hpp:153-237, instance.hpp:365-418).

The B200 kernels record no per-access trace (their conflict-freedom is proven at compile time
and measured by ncu), so ``run_algorithm(..., record_trace=True)`` raises
TraceIncomplete.  This module reads, writes and audits trace files the reference produced
(``dmmcli`` / ``run_algorithm`` with ``record_trace``), so tooling around them keeps working.

* ``TraceEvent`` / ``TraceLog``                 core.hpp:153-171
* ``verify_trace``                              core.hpp:216-237 (sort-based: a violation is a
  (step, bank) pair touched more than once)
* ``trace_to_text`` / ``trace_from_text``       instance.hpp:369-418: one line per event
  ``"step processor bank offset op [value]"`` (value on writes), then
  ``"steps=<k> work=<k*w> conflicts=<c>"``
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import NamedTuple

from . import dmm
from .instance import TraceIncomplete


@dataclass
class TraceEvent:
    step: int = 0
    processor: int = 0
    bank: int = 0
    offset: int = 0
    op: str = "r"  # "r" | "w"
    value: int = 0


@dataclass
class TraceLog:
    steps: int = 0
    conflicts: int = 0
    w: int = 0
    recording: bool = False
    events: list = field(default_factory=list)

    def work(self) -> int:
        return self.steps * self.w


class TraceViolation(NamedTuple):
    step: int
    bank: int


def verify_trace(trace: TraceLog) -> list[TraceViolation]:
    """Offline CAC re-audit: every (step, bank) touched more than once, once each, in order."""
    if not trace.recording:
        raise TraceIncomplete("verify_trace needs a trace with event recording enabled")
    keys = sorted((e.step, e.bank) for e in trace.events)
    out: list[TraceViolation] = []
    for prev, cur in zip(keys, keys[1:]):
        if cur == prev and (not out or (out[-1].step, out[-1].bank) != cur):
            out.append(TraceViolation(*cur))
    return out


def trace_to_text(t: TraceLog) -> str:
    lines = []
    for e in t.events:
        line = f"{e.step} {e.processor} {e.bank} {e.offset} {'r' if e.op == 'r' else 'w'}"
        if e.op == "w":
            line += f" {e.value}"
        lines.append(line)
    lines.append(f"steps={t.steps} work={t.work()} conflicts={t.conflicts}")
    return "\n".join(lines) + "\n"


def trace_from_text(text: str) -> TraceLog:
    t = TraceLog(recording=True)
    for line in text.split("\n"):
        if not line:
            continue
        if line.startswith("steps="):
            for tok in line.split():
                key, _, val = tok.partition("=")
                if key == "steps":
                    t.steps = int(val)
                elif key == "conflicts":
                    t.conflicts = int(val)
            continue
        toks = line.split()
        try:
            step, proc, bank, off = (int(x) for x in toks[:4])
            op = toks[4]
        except (ValueError, IndexError):
            raise dmm.Error("malformed trace line: " + line) from None
        e = TraceEvent(step, proc, bank, off, "r" if op == "r" else "w")
        if e.op == "w" and len(toks) > 5:
            e.value = int(toks[5])
        t.w = max(t.w, e.bank + 1)
        t.events.append(e)
    return t

"""The trace text format and offline audit (paper_1507_01391_b200/trace.py) against traces the
reference itself recorded (run_algorithm with record_trace, oracle/_ref) and its own
trace_from_text / verify_trace (instance.hpp:369-418, core.hpp:221-237;
tests/test_harness.cpp:108-130)."""
import pytest

from oracle.oracle import ALGORITHMS as REF_ALG
from paper_1507_01391_b200 import trace as T
from paper_1507_01391_b200.instance import TraceIncomplete


@pytest.mark.parametrize("alg,w,m", [("sort_short_wide", 2, 4), ("partition_square", 4, 4),
                                     ("partition_general", 8, 8), ("permute", 4, 4)])
def test_round_trip_and_audit_match_reference(ref, alg, w, m):
    text = ref.trace_text(REF_ALG[alg], w, m, 3)
    assert text.startswith("0 ") and "steps=" in text
    t = T.trace_from_text(text)
    assert T.trace_to_text(t) == text
    assert t.recording and t.w <= w and len(t.events) > 0
    assert T.verify_trace(t) == [] and ref.verify_trace_text(text) == 0
    # an injected duplicate (test_harness.cpp:123-129) is caught, as by the reference
    bad = T.trace_from_text(text)
    bad.events[1].step = bad.events[0].step
    bad.events[1].bank = bad.events[0].bank
    v = T.verify_trace(bad)
    assert len(v) >= 1 and (v[0].step, v[0].bank) == (bad.events[0].step, bad.events[0].bank)
    assert ref.verify_trace_text(T.trace_to_text(bad)) == len(v)


def test_summary_and_errors():
    t = T.trace_from_text("0 0 1 2 w 7\n0 1 0 0 r\nsteps=1 work=2 conflicts=0\n")
    assert (t.steps, t.conflicts, t.w, t.work()) == (1, 0, 2, 2)
    assert t.events[0].value == 7 and t.events[1].op == "r"
    with pytest.raises(TraceIncomplete):
        T.verify_trace(T.TraceLog())
    with pytest.raises(Exception, match="malformed trace line"):
        T.trace_from_text("0 0 1\n")

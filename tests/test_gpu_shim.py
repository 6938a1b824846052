"""GPU: the C++ drop-in (include/dmm_b200.hpp) against the reference's own functions in one
process (tests/cpp/test_shim.cpp): partition_general, integer_sort_general, sort_tall,
layouts and permute(Machine&, Rng&) with the caller's Rng continued bit-exactly."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "test_shim")


def test_cpp_dropin_matches_reference():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/_build/test_shim not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "0 failed" in r.stdout

"""CPU tests of the C ABI boundary: the library loads, exports every symbol the
headers declare, and applies the reference's shape contracts on the host (no GPU
needed: these paths return before any CUDA call)."""
import ctypes as C
import os
import re

import pytest

from paper_1507_01391_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in ("dmm_gpu.h",):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)  # declarations only, not comments
        names |= set(re.findall(r"\b(dmm_[a-z0-9_]+)\s*\(", src))
    return names


@pytest.fixture(scope="module")
def lib():
    return _lib.load()


def test_exports_every_declared_symbol(lib):
    names = _declared()
    assert len(names) >= 18
    for n in names:
        assert hasattr(lib, n), n
    assert set(_lib.SIGNATURES) == names


def test_version_and_support_table(lib):
    assert b"sm_100a" in lib.dmm_version()
    assert lib.dmm_supported(b"partition_general", 32, 8)
    assert lib.dmm_supported(b"partition_general", 32, 32)
    assert lib.dmm_supported(b"partition_general", 64, 8) and lib.dmm_supported(b"partition_general", 256, 16)
    assert not lib.dmm_supported(b"partition_general", 512, 16) and not lib.dmm_supported(b"partition_general", 128, 16)
    # sub-warp machines (32 / w per warp) and the square / short-wide entry points
    assert lib.dmm_supported(b"partition_general", 16, 8) and lib.dmm_supported(b"integer_sort_general", 4, 16)
    assert lib.dmm_supported(b"partition_square", 16, 16) and lib.dmm_supported(b"sort_square", 4, 4)
    assert lib.dmm_supported(b"partition_short_wide", 8, 64) and lib.dmm_supported(b"sort_short_wide", 2, 4)
    assert not lib.dmm_supported(b"partition_square", 32, 32)  # 32 is not a perfect square
    assert not lib.dmm_supported(b"partition_short_wide", 8, 32)  # w^2 > m


@pytest.mark.parametrize("w,m,flags,expect", [
    (32, 4, 1, 1),    # m > 2 sqrt(log2 w) fails (partition.hpp:443-445): ShapeViolation
    (32, 8, 0, 1),    # balance leftover group of 4 (partition.hpp:241-244): ShapeViolation
    (32, 1, 0, 1),    # general sort needs m >= 2
    (32, 48, 0, 1),   # w <= m but neither short-wide, square nor w | m (shearsort): ShapeViolation
    (32, 8, 5, 0),    # 32x8 with the extension and enforce off: accepted (count 0 -> no launch)
])
def test_partition_shape_contracts(lib, w, m, flags, expect):
    st = lib.dmm_partition_general(None, None, w, m, 0, flags, None, None, None)
    assert st == expect


def test_layout_and_sort_shape_contracts(lib):
    assert lib.dmm_sort_tall(None, None, 32, 64, 0, None) == 1   # w >= m (sort.hpp:354)
    assert lib.dmm_sort_square(None, None, 32, 32, 0, 1, None) == 1  # m not a perfect square
    assert lib.dmm_sort_short_wide(None, None, 32, 64, 0, 1, None) == 1  # w^2 <= m
    assert lib.dmm_partition_square(None, None, 32, 16, 0, None, None) == 1  # w = m
    assert lib.dmm_permute(None, None, 32, 256, 0, None, 4, 64, None, None, None, None, None, None) == 1  # m | w
    assert lib.dmm_permute(None, None, 256, 32, 0, None, 4, 64, None, None, None, None, None, None) == 1  # shape ok
    assert lib.dmm_sort_wide_any(None, None, 32, 16, 0, 1, None) == 1  # w <= m
    assert lib.dmm_gen_instances(1, 0, 4, 0, 0, None, None) == 1


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(ImportError):
        _lib.load(str(tmp_path / "nope.so"))


def test_probe_snapshot_count_matches_reference_hooks(lib, ref):
    # dmm_general_probe_snaps = the number of PartitionProbe hook calls of the outer recursion
    # (after_balance + after_divide per level, partition.hpp:376-390), host-side, no GPU needed
    import numpy as np
    for (w, m) in [(32, 16), (16, 8), (64, 16), (256, 16), (64, 8), (128, 32), (32, 32), (8, 8)]:
        g = ref.gen_instance(1, w, m, 1)
        st, _, rep = ref.integer_sort_general(g, w, enforce_pre=False, probe_snaps=64)
        assert st == 0
        assert lib.dmm_general_probe_snaps(w, m, 0) == rep["snapshots"].shape[0], (w, m)

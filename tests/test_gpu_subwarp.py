"""GPU parity for sub-warp machines (w < 32 rows; 32 / w machines run as one lockstep view
family per warp): general partition / integer sort with GeneralStats, and the square /
short-wide entry points that only exist at such shapes (partition.hpp:178-197,
sort.hpp:225-346), against the oracle (C restatement pinned to the reference).

Bar: bit-exact outputs and cleanup_retries per instance.  Instance counts are not
multiples of the machines per warp, so partially filled warps are exercised.
"""
import numpy as np
import pytest

from oracle.oracle import FLAG_NO_ENFORCE_PRE

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1507_01391_b200 as dmm  # noqa: E402

SHAPES = [(16, 8), (16, 16), (16, 32), (16, 64), (8, 8), (8, 16), (8, 32), (8, 64), (4, 4), (4, 8), (4, 16),
          (2, 2), (2, 4), (2, 8)]


def _batch(port, kind, w, m, seeds):
    return np.stack([port.gen_instance(kind, w, m, s) for s in seeds]).astype(np.uint32)


@pytest.mark.parametrize("w,m", SHAPES)
def test_partition_general_subwarp(port, w, m):
    seeds = list(range(1, 2 * (32 // w) + 4))  # two warps' worth plus a ragged tail (both halves)
    grids = _batch(port, 1, w, m, seeds)
    out, st = dmm.partition_general(grids, flags=dmm.FLAG_NO_ENFORCE_PRE)
    out = dmm.as_uint32(out)
    for k in range(len(seeds)):
        ost, oout, orep = port.partition_general(grids[k], FLAG_NO_ENFORCE_PRE)
        assert ost == 0
        assert (out[k] == oout).all(), (w, m, k)
        assert int(st.cleanup_retries[k]) == orep["cleanup_retries"], (w, m, k)
    # row i holds label i everywhere (verify_partition_result instance.hpp:249)
    assert (out == np.arange(w, dtype=np.uint32).reshape(1, w, 1)).all()


@pytest.mark.parametrize("w,m", SHAPES)
@pytest.mark.parametrize("domain", [1 << 10, 1 << 32])
def test_integer_sort_subwarp(port, w, m, domain):
    rng = np.random.default_rng(w * 131 + m)
    n = 2 * (32 // w) + 3
    grids = rng.integers(0, domain, size=(n, w, m), dtype=np.uint64).astype(np.uint32)
    out, st = dmm.integer_sort_general(grids, domain, enforce_analysis_pre=False)
    out = dmm.as_uint32(out)
    for k in range(n):
        ost, oout, orep = port.integer_sort_general(grids[k], domain, FLAG_NO_ENFORCE_PRE)
        assert ost == 0 and (out[k] == oout).all(), (w, m, k)
        assert int(st.cleanup_retries[k]) == orep["cleanup_retries"]


@pytest.mark.parametrize("w", [4, 16])
def test_partition_square(port, w):
    seeds = list(range(5, 5 + 32 // w + 3))
    grids = _batch(port, 1, w, w, seeds)
    out = dmm.as_uint32(dmm.partition_square(grids))
    for k in range(len(seeds)):
        st, exp = port.simple("partition_square", grids[k])
        assert st == 0 and (out[k] == exp).all()


@pytest.mark.parametrize("w,m", [(2, 4), (2, 8), (4, 16), (8, 64)])
def test_partition_short_wide(port, w, m):
    seeds = list(range(9, 9 + 32 // w + 1))
    grids = _batch(port, 1, w, m, seeds)
    out = dmm.as_uint32(dmm.partition_short_wide(grids))
    for k in range(len(seeds)):
        st, exp = port.simple("partition_short_wide", grids[k])
        assert st == 0 and (out[k] == exp).all()


@pytest.mark.parametrize("w", [4, 16])
@pytest.mark.parametrize("asc", [True, False])
def test_sort_square(port, w, asc):
    rng = np.random.default_rng(w)
    g = rng.integers(0, 2 ** 32, size=(32 // w + 2, w, w), dtype=np.uint64).astype(np.uint32)
    out = dmm.as_uint32(dmm.sort_square(g, ascending=asc))
    for k in range(g.shape[0]):
        st, exp = port.simple("sort_square", g[k], int(asc))
        assert st == 0 and (out[k] == exp).all()


@pytest.mark.parametrize("w,m", [(2, 4), (2, 8), (4, 16), (8, 64)])
@pytest.mark.parametrize("asc", [True, False])
def test_sort_short_wide(port, w, m, asc):
    rng = np.random.default_rng(w * m)
    g = rng.integers(0, 1000, size=(32 // w + 1, w, m), dtype=np.uint64).astype(np.uint32)
    out = dmm.as_uint32(dmm.sort_short_wide(g, ascending=asc))
    for k in range(g.shape[0]):
        st, exp = port.simple("sort_short_wide", g[k], int(asc))
        assert st == 0 and (out[k] == exp).all()


def test_subwarp_errors(port):
    bad = _batch(port, 1, 16, 16, [1, 2, 3])
    bad[1, 0, 0] = 15 if bad[1, 0, 0] != 15 else 14  # wrong label counts
    with pytest.raises(dmm.InvalidInstance):
        dmm.partition_square(bad)
    with pytest.raises(dmm.ShapeViolation):  # w^2 > m (partition.hpp:179-180)
        dmm.partition_short_wide(_batch(port, 1, 8, 32, [1]))
    with pytest.raises(dmm.ShapeViolation):  # m not a perfect square (sort.hpp:340-342)
        dmm.sort_square(np.zeros((1, 8, 8), dtype=np.uint32))


def test_odd_machine_3x9(port, golden):
    # 3-row machines (10 per warp, 2 idle lanes) at the reference's own odd test shape 3 x 9:
    # the leaf runs the reference's short-wide dispatch with padded Batcher row networks
    seeds = list(range(1, 24))  # two warps' worth and a ragged third
    grids = _batch(port, 1, 3, 9, seeds)
    out, st = dmm.partition_general(grids)
    out = dmm.as_uint32(out)
    for k in range(len(seeds)):
        s, exp, rep = port.partition_general(grids[k])
        assert s == 0 and (out[k] == exp).all() and int(st.cleanup_retries[k]) == rep["cleanup_retries"]
    rng = np.random.default_rng(39)
    keys = rng.integers(0, 1 << 20, size=(13, 3, 9), dtype=np.uint64).astype(np.uint32)
    out, _ = dmm.integer_sort_general(keys, 1 << 20)
    for k in range(13):
        s, exp, _ = port.integer_sort_general(keys[k], 1 << 20)
        assert s == 0 and (dmm.as_uint32(out)[k] == exp).all()
    out = dmm.as_uint32(dmm.partition_short_wide(grids))
    for k in range(len(seeds)):
        s, exp = port.simple("partition_short_wide", grids[k])
        assert s == 0 and (out[k] == exp).all()
    for asc in (True, False):
        out = dmm.as_uint32(dmm.sort_short_wide(keys, ascending=asc))
        for k in range(13):
            s, exp = port.simple("sort_short_wide", keys[k], int(asc))
            assert s == 0 and (out[k] == exp).all()
    meta, arr = golden
    case = [c for c in meta["partition"] if (c["w"], c["m"]) == (3, 9)][0]
    out, st = dmm.partition_general(arr[case["key"] + "_in"])
    assert (dmm.as_uint32(out) == arr[case["key"] + "_out"]).all()

"""GPU parity: kernels 1-3 (partition / general partition / integer sort) through the C ABI
against the oracle (C restatement pinned to the reference) and the golden fixtures.

Bar: bit-exact outputs AND bit-exact GeneralStats (cleanup_retries, sorted) per instance.
"""
import numpy as np
import pytest

from oracle.oracle import FLAG_EXT_PARTIAL_GROUPS

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1507_01391_b200 as dmm  # noqa: E402


def _oracle_batch(port, kind, w, m, seeds):
    return np.stack([port.gen_instance(kind, w, m, s) for s in seeds]).astype(np.uint32)


@pytest.mark.parametrize("kind,w,m", [(1, 32, 8), (1, 32, 16), (1, 32, 32), (2, 32, 32), (2, 32, 16), (1, 32, 64),
                                      (2, 128, 64), (1, 64, 128)])
def test_gen_instances_bit_exact(port, kind, w, m):
    seeds = list(range(100, 164))
    dev = dmm.as_uint32(dmm.gen_instances(kind, w, m, 100, 64))
    assert (dev == _oracle_batch(port, kind, w, m, seeds)).all()


def test_gen_sort_u32_bit_exact(port):
    dev = dmm.as_uint32(dmm.gen_instances(dmm.KIND_SORT_U32, 32, 128, 7, 4))
    for k in range(4):
        assert (dev[k] == port.gen_sort_u32(32, 128, 7 + k).astype(np.uint32)).all()


@pytest.mark.parametrize("m,flags", [(8, FLAG_EXT_PARTIAL_GROUPS), (16, 0), (32, 0), (64, 0)])
def test_partition_general_vs_oracle(port, m, flags):
    seeds = list(range(1, 41)) + [12345]  # odd count: exercises the unpaired half of the last warp
    grids = _oracle_batch(port, 1, 32, m, seeds)
    out, st = dmm.partition_general(grids, flags=flags)
    out = dmm.as_uint32(out)
    retries = st.cleanup_retries.cpu().numpy()
    for k, s in enumerate(seeds):
        ost, oout, orep = port.partition_general(grids[k], flags)
        assert ost == 0
        assert (out[k] == oout).all(), (m, s)
        assert retries[k] == orep["cleanup_retries"] and bool(st.sorted[k]) == orep["sorted"]


def test_partition_golden(golden):
    meta, arr = golden
    for case in meta["partition"]:
        if not dmm.supported("partition_general", case["w"], case["m"]) or case["status"] != 0:
            continue
        out, st = dmm.partition_general(arr[case["key"] + "_in"])
        assert (dmm.as_uint32(out) == arr[case["key"] + "_out"]).all(), case["key"]
        assert int(st.cleanup_retries[0]) == case["cleanup_retries"]


@pytest.mark.parametrize("m,domain", [(16, 512), (32, 1024), (16, 1 << 20), (32, 1 << 32), (64, 2048),
                                      (128, 1 << 32), (128, 4096)])
def test_integer_sort_vs_oracle(port, m, domain):
    rng = np.random.default_rng(m)
    if domain <= 32 * m:
        grids = _oracle_batch(port, 2, 32, m, range(30, 47))
    else:
        grids = rng.integers(0, domain, size=(17, 32, m), dtype=np.uint64).astype(np.uint32)
    out, st = dmm.integer_sort_general(grids, domain)
    out = dmm.as_uint32(out)
    for k in range(grids.shape[0]):
        ost, oout, orep = port.integer_sort_general(grids[k], domain)
        assert ost == 0 and (out[k] == oout).all()
        assert int(st.cleanup_retries[k]) == orep["cleanup_retries"]


def test_integer_sort_golden(golden):
    meta, arr = golden
    for case in meta["intsort"] + meta["u32sort"]:
        if not dmm.supported("integer_sort_general", case["w"], case["m"]) or case["status"] != 0:
            continue
        dom = case.get("domain", 1 << 32)
        out, st = dmm.integer_sort_general(arr[case["key"] + "_in"], dom)
        assert (dmm.as_uint32(out) == arr[case["key"] + "_out"]).all(), case["key"]


@pytest.mark.parametrize("m,flags", [(8, FLAG_EXT_PARTIAL_GROUPS), (16, 0), (32, 0)])
def test_partition_large_batch_properties(m, flags):
    # full-size property check: every instance ends with row i = i (verify_partition_result
    # instance.hpp:249); inputs generated on the device with the reference's generator
    count = 1 << 16
    g = dmm.gen_instances(dmm.KIND_PARTITION, 32, m, 1, count)
    out, st = dmm.partition_general(g, flags=flags)
    rows = torch.arange(32, device="cuda", dtype=torch.int32).view(1, 32, 1)
    assert bool((out == rows).all())
    assert bool(st.sorted.all()) and int((st.status != 0).sum()) == 0
    # the multiset is preserved in place too (in == out aliasing)
    g2 = g.clone()
    dmm.partition_general(g2, flags=flags, out=g2)
    assert bool((g2 == rows).all())


def test_partition_errors(port):
    g = _oracle_batch(port, 1, 32, 8, [3])
    with pytest.raises(dmm.ShapeViolation):  # reference rejects 32x8 (partition.hpp:241-244)
        dmm.partition_general(g)
    g4 = _oracle_batch(port, 1, 32, 4, [3])
    with pytest.raises(dmm.ShapeViolation):  # m > 2 sqrt(log2 w) (partition.hpp:443-445)
        dmm.partition_general(g4, flags=FLAG_EXT_PARTIAL_GROUPS)
    bad = _oracle_batch(port, 1, 32, 16, [4, 5, 6])
    bad[1, 0, 0] = 31 if bad[1, 0, 0] != 31 else 30  # wrong label counts
    with pytest.raises(dmm.InvalidInstance):
        dmm.partition_general(bad)
    _, st = dmm.partition_general(bad, check=False)
    assert st.status.cpu().tolist() == [0, 2, 0]
    bad[2, 3, 3] = 40  # label outside [0, w)
    _, st = dmm.partition_general(bad, check=False)
    assert st.status.cpu().tolist() == [0, 2, 2]
    keys = _oracle_batch(port, 2, 32, 16, [1])
    keys[0, 5, 5] = 600
    with pytest.raises(dmm.KeyOutOfRange):
        dmm.integer_sort_general(keys, 512)


def test_sort_wide_any_vs_oracle():
    rng = np.random.default_rng(3)
    g = rng.integers(0, 2 ** 32, size=(9, 32, 32), dtype=np.uint64).astype(np.uint32)
    for asc in (True, False):
        out = dmm.as_uint32(dmm.sort_wide_any(g, ascending=asc))
        for k in range(9):
            exp = np.sort(g[k].ravel())
            if not asc:
                exp = exp[::-1]
            assert (out[k].ravel() == exp).all()


@pytest.mark.parametrize("m", [2, 4, 8, 16, 32])
def test_sort_tall_vs_oracle(port, m):
    rng = np.random.default_rng(m)
    g = rng.integers(0, 1000, size=(5, 32, m), dtype=np.uint64).astype(np.uint32)
    out = dmm.as_uint32(dmm.sort_tall(g))
    for k in range(5):
        st, exp = port.simple("sort_tall", g[k])
        assert st == 0 and (out[k] == exp).all()


@pytest.mark.parametrize("m", [1, 2, 4, 8, 16, 32, 64])
def test_layout_primitives_vs_oracle(port, m):
    g = np.arange(3 * 32 * m, dtype=np.uint32).reshape(3, 32, m)
    for name in ("to_column_major", "to_row_major"):
        out = dmm.as_uint32(getattr(dmm, name)(g))
        for k in range(3):
            st, exp = port.simple(name, g[k])
            assert (out[k] == exp).all(), (name, m)
    if m == 32:
        out = dmm.as_uint32(dmm.transpose_square(g))
        for k in range(3):
            assert (out[k] == g[k].T).all()


def test_sort_rows_orders():
    rng = np.random.default_rng(5)
    g = rng.integers(0, 100, size=(4, 32, 16), dtype=np.uint64).astype(np.uint32)
    for order in range(4):
        out = dmm.as_uint32(dmm.sort_rows(g, order=order))
        for r in range(32):
            asc = order == 0 or (order == 2 and r % 2 == 0) or (order == 3 and r % 2 == 1)
            exp = np.sort(g[:, r, :], axis=1)
            if not asc:
                exp = exp[:, ::-1]
            assert (out[:, r, :] == exp).all()
    with pytest.raises(dmm.KeyOutOfRange):  # row_radix_segment partition.hpp:63
        dmm.sort_rows(g, order=0, domain=50)


def test_partition_probe_snapshots_golden(golden):
    """PartitionProbe (partition.hpp:298-301): the working window after every after_balance /
    after_divide hook of the outer recursion equals the reference's, snapshot for snapshot."""
    meta, arr = golden
    assert meta["probe"]
    for case in meta["probe"]:
        g = arr[case["key"] + "_in"]
        if case["domain"] == case["w"]:
            out, st = dmm.partition_general(g, probe=True)
        else:
            out, st = dmm.integer_sort_general(g, case["domain"], probe=True)
        snaps = dmm.as_uint32(st.snapshots)
        assert snaps.shape[0] == case["n_snaps"], case["key"]
        assert (snaps == arr[case["key"] + "_snaps"]).all(), case["key"]
        assert (dmm.as_uint32(out) == arr[case["key"] + "_out"]).all()
        assert int(st.cleanup_retries) == case["cleanup_retries"]


@pytest.mark.parametrize("w,m", [(32, 16), (16, 8), (32, 8)])
def test_probe_batch_matches_plain_run(port, w, m):
    # a probed batch (both packed halves, ragged tail) returns the same outputs and stats as
    # the plain kernel; w <= m has no outer recursion and so no snapshots
    flags = dmm.FLAG_EXT_PARTIAL_GROUPS if (w, m) == (32, 8) else 0
    grids = np.stack([port.gen_instance(1, w, m, s) for s in range(1, 12)]).astype(np.uint32)
    out0, st0 = dmm.partition_general(grids, flags=flags)
    out1, st1 = dmm.partition_general(grids, flags=flags, probe=True)
    assert (dmm.as_uint32(out0) == dmm.as_uint32(out1)).all()
    assert (st0.cleanup_retries == st1.cleanup_retries).all()
    assert st1.snapshots.shape == (11, 2, w, m)
    # the last snapshot (after the final divide) is a permutation of the instance
    s = dmm.as_uint32(st1.snapshots)
    assert (np.sort(s[:, -1].reshape(11, -1), axis=1) == np.sort(grids.reshape(11, -1), axis=1)).all()
    _, st2 = dmm.partition_general(port.gen_instance(1, 32, 32, 1), probe=True)
    assert st2.snapshots.shape == (0, 32, 32)


def test_empty_and_single_batches(port):
    # count 0: no launch, no error; count 1: a lone packed half / lone machine in its warp or CTA
    empty = np.zeros((0, 32, 16), dtype=np.uint32)
    out, st = dmm.partition_general(empty)
    assert out.shape == (0, 32, 16) and st.cleanup_retries.numel() == 0
    out, _ = dmm.integer_sort_general(np.zeros((0, 64, 16), dtype=np.uint32), 1024)
    assert out.shape == (0, 64, 16)
    assert dmm.sort_tall(np.zeros((0, 128, 32), dtype=np.uint32)).shape == (0, 128, 32)
    for (w, m) in [(32, 16), (4, 8), (64, 16)]:
        g = port.gen_instance(1, w, m, 9).astype(np.uint32)
        out, st = dmm.partition_general(g[None], flags=dmm.FLAG_NO_ENFORCE_PRE)
        s, exp, rep = port.partition_general(g, dmm.FLAG_NO_ENFORCE_PRE)
        assert (dmm.as_uint32(out)[0] == exp).all() and int(st.cleanup_retries[0]) == rep["cleanup_retries"]
    keys = dmm.gen_keys(0, 0)
    out, starts = dmm.multisplit(keys, 8, 29)
    assert out.numel() == 0


def test_cfg3_tiles_vs_oracle_and_reference(port, ref):
    # the headline config exactly: 32 x 128 uint32 tiles from the bench's generator, sorted by
    # integer_sort_general(view, 2^32) (partition.hpp:436-449); 512 tiles against the oracle,
    # 48 of them against the compiled reference itself
    count = 512
    g = dmm.gen_instances(dmm.KIND_SORT_U32, 32, 128, 1, count)
    host = dmm.as_uint32(g)
    for k in (0, 1, 255, 511):
        assert (host[k] == port.gen_sort_u32(32, 128, 1 + k).astype(np.uint32)).all()
    out, st = dmm.integer_sort_general(g, 1 << 32)
    out = dmm.as_uint32(out)
    assert int((st.status != 0).sum()) == 0
    for k in range(count):
        ost, oout, orep = port.integer_sort_general(host[k], 1 << 32)
        assert ost == 0 and (out[k] == oout).all(), k
        assert int(st.cleanup_retries[k]) == orep["cleanup_retries"] == 0
    for k in range(0, count, count // 48):
        rst, rout, _ = ref.integer_sort_general(host[k].astype(np.uint64), 1 << 32)
        assert rst == 0 and (out[k] == rout.astype(np.uint32)).all(), k


def test_cfg3_full_batch_multiset_check():
    # full-size properties at 2^16 tiles (the bench applies the same check at 2^20): per-tile
    # sum / sum of squares / XOR preserved, ascending, sampled tiles equal numpy's sort -- and
    # the check itself rejects a wrong output (all zeros, one swapped key, one dropped key)
    import bench
    count = 1 << 16
    g = dmm.gen_instances(dmm.KIND_SORT_U32, 32, 128, 77, count)
    out, _ = dmm.integer_sort_general(g, 1 << 32, check=False)
    res = bench.verify_sort_full(g, out, count)
    assert res["ok"], res
    bad = torch.zeros_like(out)
    assert not bench.verify_sort_full(g, bad, count)["ok"]
    bad = out.clone()
    bad[5, 0, 0], bad[5, 0, 1] = out[5, 0, 1], out[5, 0, 0]
    if int(out[5, 0, 0]) != int(out[5, 0, 1]):
        assert not bench.verify_sort_full(g, bad, count)["ascending"]
    bad = out.clone()
    bad[count - 1, 31, 127] = bad[count - 1, 31, 126]
    r = bench.verify_sort_full(g, bad, count)
    assert not (r["sum_sumsq"] and r["xor"])


@pytest.mark.parametrize("asc", [True, False])
def test_sort_wide_any_32x128(port, asc):
    # detail::sort_wide_any at 32 x 128 (sort.hpp:321-330 -> shearsort_rect, merge rows): the
    # CTA tile kernel in comparison mode, both directions, against the oracle and numpy
    rng = np.random.default_rng(128 + asc)
    g = rng.integers(0, 2 ** 32, size=(9, 32, 128), dtype=np.uint64).astype(np.uint32)
    g[2] = rng.integers(0, 3, size=(32, 128), dtype=np.uint64).astype(np.uint32)
    out = dmm.as_uint32(dmm.sort_wide_any(g, ascending=asc))
    for k in range(9):
        exp = np.sort(g[k].ravel())
        assert (out[k].ravel() == (exp if asc else exp[::-1])).all(), k
    s, exp = port.simple("sort_wide_any", g[0], int(asc))
    assert s == 0 and (out[0] == exp).all()


def test_partition_general_32x128_vs_oracle(port):
    # partition mode of the 32 x 128 tile kernel (two instances per register) against the oracle
    seeds = list(range(1, 38))  # odd count: the last CTA pairs an instance with nothing
    grids = _oracle_batch(port, 1, 32, 128, seeds)
    out, st = dmm.partition_general(grids)
    out = dmm.as_uint32(out)
    for k in range(len(seeds)):
        ost, oout, orep = port.partition_general(grids[k])
        assert ost == 0 and (out[k] == oout).all()
        assert int(st.cleanup_retries[k]) == orep["cleanup_retries"]
    bad = grids[:3].copy()
    bad[1, 4, 4] = 40
    with pytest.raises(dmm.InvalidInstance):
        dmm.partition_general(bad)


def test_32x256_vs_oracle(port):
    # 32 x 256 (partition_leaf -> square_skeleton with h = 16; 51 513 steps): the
    # 8-warp tile kernel in partition (two instances per register), integer-sort and
    # comparison modes, against the oracle
    seeds = list(range(1, 12))
    grids = _oracle_batch(port, 1, 32, 256, seeds)
    out, st = dmm.partition_general(grids)
    out = dmm.as_uint32(out)
    for k in range(len(seeds)):
        ost, oout, orep = port.partition_general(grids[k])
        assert ost == 0 and (out[k] == oout).all()
        assert int(st.cleanup_retries[k]) == orep["cleanup_retries"]
    rng = np.random.default_rng(256)
    keys = rng.integers(0, 2 ** 32, size=(7, 32, 256), dtype=np.uint64).astype(np.uint32)
    out, _ = dmm.integer_sort_general(keys, 1 << 32)
    out = dmm.as_uint32(out)
    for k in range(7):
        ost, oout, _ = port.integer_sort_general(keys[k], 1 << 32)
        assert ost == 0 and (out[k] == oout).all()
    for asc in (True, False):
        o2 = dmm.as_uint32(dmm.sort_wide_any(keys, ascending=asc))
        for k in range(7):
            exp = np.sort(keys[k].ravel())
            assert (o2[k].ravel() == (exp if asc else exp[::-1])).all()

"""The oracle (C restatement, oracle/dmm_oracle.c) pinned against the reference.

Pins, in order of strength:
  1. golden vectors produced by the UNMODIFIED reference (tests/golden/, make_golden.py);
  2. the reference's own known answers (test_*.cpp);
  3. a live sweep against oracle/_ref (the reference compiled in place) when present.
"""
import numpy as np
import pytest

from oracle.oracle import FLAG_EXT_PARTIAL_GROUPS, PERMUTE


def test_mt19937_64_stream(port, golden):
    meta, _ = golden
    # std::mt19937_64 10000th output for the default seed (C++ standard, [rand.predef])
    assert str(port.mt19937_64(5489, 10000)[-1]) == "9981545732273789042"
    assert meta["mt19937_64_10000th_default"] == "9981545732273789042"
    for seed, vals in meta["mt19937_64"].items():
        assert [str(x) for x in port.mt19937_64(int(seed), 16)] == vals


def test_partition_general_golden(port, golden):
    meta, arr = golden
    for case in meta["partition"]:
        st, out, rep = port.partition_general(arr[case["key"] + "_in"])
        assert st == case["status"], case["key"]
        if st == 0:
            assert (out == arr[case["key"] + "_out"]).all(), case["key"]
            assert rep["cleanup_retries"] == case["cleanup_retries"]
            assert rep["sorted"] == case["sorted"]
            # verify_partition_result instance.hpp:249
            assert all((out[i] == i).all() for i in range(case["w"]))


def test_integer_sort_golden(port, golden):
    meta, arr = golden
    for case in meta["intsort"]:
        st, out, rep = port.integer_sort_general(arr[case["key"] + "_in"], case["domain"])
        assert st == case["status"] and (out == arr[case["key"] + "_out"]).all(), case["key"]
        assert rep["cleanup_retries"] == case["cleanup_retries"]
    for case in meta["u32sort"]:
        g = arr[case["key"] + "_in"]
        assert (port.gen_sort_u32(case["w"], case["m"], case["seed"]) == g).all()
        st, out, rep = port.integer_sort_general(g, 1 << 32)
        assert st == case["status"] and (out == arr[case["key"] + "_out"]).all(), case["key"]


def test_permute_golden(port, golden):
    meta, arr = golden
    for case in meta["permute"]:
        g = arr[case["key"] + "_in"]
        assert (port.gen_instance(2, case["w"], case["m"], case["seed"]) == g).all()
        st, out, rep = port.permute(g, case["seed"])
        assert st == case["status"], case["key"]
        assert (out == arr[case["key"] + "_out"]).all(), case["key"]
        for k in ("iterations", "fallback", "used_packing", "packed_width", "threshold", "random_words",
                  "cleanup_retries", "leftover_history", "shifts"):
            assert rep[k] == case[k], (case["key"], k, rep[k], case[k])


def test_permute_known_answers(port):
    # SURVEY.md App. A.3, recorded from the reference (gen_instance(permute, 32, 32, s), Rng(s), alpha 4)
    lefts = []
    for s in range(1, 7):
        st, out, rep = port.permute(port.gen_instance(2, 32, 32, s), s)
        assert st == 0 and (out.ravel() == np.arange(1024)).all()
        assert rep["iterations"] == 1 and rep["used_packing"] and rep["packed_width"] == 16
        assert rep["threshold"] == 128 and rep["random_words"] == 89
        lefts.append(rep["leftover_history"][0])
        if s == 1:
            assert rep["shifts"][:4] == [9, 15, 27, 15]
    assert lefts == [4, 1, 3, 7, 5, 1]
    # randomness budget test_permute.cpp:364-381
    for s in range(1, 4):
        _, _, rep = port.permute(port.gen_instance(2, 64, 16, s), s)
        assert rep["random_words"] == 64 + rep["iterations"] * 16 + (36 if rep["used_packing"] else 0)


def test_layout_golden_and_examples(port, golden):
    meta, arr = golden
    for case in meta["layout"]:
        st, out = port.simple(case["op"], arr[case["key"] + "_in"])
        assert st == case["status"] and (out == arr[case["key"] + "_out"]).all(), case["key"]
    # test_layout.cpp:79-85: 2x4 example
    st, out = port.simple("to_column_major", np.arange(1, 9).reshape(2, 4))
    assert out.ravel().tolist() == [1, 3, 5, 7, 2, 4, 6, 8]
    st, out = port.simple("transpose_square", np.array([[1, 2], [3, 4]]))
    assert out.ravel().tolist() == [1, 3, 2, 4]


def test_shape_predicates(port, golden):
    meta, _ = golden
    for k, v in meta["shape_ok"].items():
        W, M = map(int, k.split("x"))
        assert port.general_sort_shape_ok(W, M) == v, k
    for k, v in meta["permute_threshold"].items():
        w, m = map(int, k.split("x"))
        assert port.permute_threshold(w, m) == v
    # test_partition.cpp:237-262 parameter arithmetic
    assert port.partition_params(4096, 16)[1] == (3, 8, 128)
    assert port.partition_params(32, 16)[1][1] == 2
    assert port.partition_params(2048, 8)[1][1] == 16


def test_reference_rejections_and_extension(port):
    # K4b: 32x8 rejected by the reference's balance(); accepted with the B200 extension
    g = port.gen_instance(1, 32, 8, 3)
    st, _, _ = port.partition_general(g)
    assert st == 1  # ShapeViolation
    st, out, rep = port.partition_general(g, FLAG_EXT_PARTIAL_GROUPS)
    assert st == 0 and all((out[i] == i).all() for i in range(32))
    # invalid instance
    bad = g.copy()
    bad[0, 0] = 31 if bad[0, 0] != 31 else 30
    assert port.partition_general(bad, FLAG_EXT_PARTIAL_GROUPS)[0] == 2


@pytest.mark.parametrize("shape", [(32, 32), (32, 16), (32, 64), (64, 16), (16, 16), (64, 64), (32, 128), (32, 256),
                                   (32, 1024)])
def test_port_vs_reference_partition(port, ref, shape):
    w, m = shape
    for s in range(10, 16):
        g = ref.gen_instance(1, w, m, s)
        a = port.partition_general(g)
        b = ref.partition_general(g)
        assert a[0] == b[0] and (a[1] == b[1]).all() and a[2] == b[2]


@pytest.mark.parametrize("shape", [(32, 32), (32, 16), (64, 16), (32, 2), (32, 4), (128, 64)])
def test_port_vs_reference_permute(port, ref, shape):
    w, m = shape
    for s in range(20, 26):
        g = ref.gen_instance(2, w, m, s)
        a = port.permute(g, s)
        b = ref.permute(g, s)
        assert a[0] == b[0] and (a[1] == b[1]).all() and a[2] == b[2]


def test_port_vs_reference_run_algorithm(port, ref):
    g = ref.gen_instance(2, 32, 32, 9)
    st, out, rep = ref.run_algorithm(PERMUTE, g, 9)
    assert st == 0 and rep["correct"] and rep["conflicts"] == 0
    a = port.permute(g, 9)
    assert a[2]["iterations"] == rep["iterations"] and a[2]["fallback"] == rep["fallback"]


@pytest.mark.parametrize("w,m", [(32, 128), (32, 32), (4, 16), (8, 64)])
def test_oracle_sort_wide_any(port, w, m):
    # detail::sort_wide_any (sort.hpp:321-330): the sorted multiset in either direction (its
    # outcome is unique), and ShapeViolation unless w <= m and w | m (sort.hpp:291-292)
    rng = np.random.default_rng(w * m)
    g = rng.integers(0, 2 ** 32, size=(w, m), dtype=np.uint64)
    for asc in (1, 0):
        s, out = port.simple("sort_wide_any", g, asc)
        exp = np.sort(g.ravel())
        assert s == 0 and (out.ravel() == (exp if asc else exp[::-1])).all()
    s, _ = port.simple("sort_wide_any", rng.integers(0, 9, size=(32, 48), dtype=np.uint64), 1)
    assert s == 1  # DMM_SHAPE_VIOLATION


def test_port_vs_reference_short_wide_32x1024(port, ref):
    # the w = 32 short-wide machine (n = 32 w^2): the restatement's partition_short_wide and
    # sort_short_wide against the reference's run_algorithm on the same instances
    for s in (1, 2):
        g = ref.gen_instance(1, 32, 1024, s)
        st, rout, rep = ref.run_algorithm(3, g, s)  # partition_short_wide
        assert st == 0 and rep["correct"] and rep["steps"] == 76 * 1024
        ps, pout = port.simple("partition_short_wide", g)
        assert ps == 0 and (pout == rout).all()
        k = (ref.gen_instance(0, 32, 1024, s) >> np.uint64(32)).astype(np.uint64)
        st, rout, rep = ref.run_algorithm(0, k, s)  # sort_short_wide
        ps, pout = port.simple("sort_short_wide", k, 1)
        assert st == 0 and ps == 0 and (pout == rout).all()

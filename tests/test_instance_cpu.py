"""Host layer of the instance.hpp mirror (paper_1507_01391_b200/instance.py): the text format,
validation and report formats, checked against the reference's own functions
(oracle/_ref: instance_to_text / instance_from_text, instance.hpp:103-128) and the
reference's harness cases (tests/test_harness.cpp:10-52, :95-106).  No GPU needed."""
import numpy as np
import pytest

import paper_1507_01391_b200 as dmm
from paper_1507_01391_b200 import instance as I

KIND_ID = {"sort": 0, "partition": 1, "permute": 2}


def _inst(ref, kind, w, m, seed):
    return I.Instance(kind, w, m, seed, ref.gen_instance(KIND_ID[kind], w, m, seed))


@pytest.mark.parametrize("kind,w,m,seed", [("sort", 3, 5, 11), ("partition", 4, 16, 7), ("permute", 16, 8, 9),
                                           ("partition", 32, 32, 1), ("sort", 1, 1, 0)])
def test_text_matches_reference(ref, kind, w, m, seed):
    inst = _inst(ref, kind, w, m, seed)
    text = I.instance_to_text(inst)
    assert text == ref.instance_to_text(KIND_ID[kind], w, m, seed, inst.grid)
    back = I.instance_from_text(text)
    assert (back.kind, back.w, back.m, back.seed) == (kind, w, m, seed)
    assert (back.grid == inst.grid).all()
    # the reference parses ours back to the same instance
    s, hdr, g = ref.instance_from_text(text)
    assert s == 0 and hdr == (KIND_ID[kind], w, m, seed) and (g == inst.grid).all()


@pytest.mark.parametrize("text", ["", "bogus 1 2 3\n0 0", "sort 2 2 1\n1 2 3", "sort 2", "sort x 2 1 0",
                                  "partition 2 2 5\n0 1 1 x"])
def test_text_errors_match_reference(ref, text):
    s, _, _ = ref.instance_from_text(text)
    assert s == dmm.InvalidInstance.status
    with pytest.raises(dmm.InvalidInstance):
        I.instance_from_text(text)


def test_token_based_parse():
    # the reference reads whitespace tokens: the row layout of the body does not matter
    a = I.instance_from_text("permute 2 2 4\n3 1\n0 2\n")
    b = I.instance_from_text("permute 2 2 4 3 1 0 2")
    assert (a.grid == b.grid).all() and a.grid.tolist() == [3, 1, 0, 2]


def test_validate_instance(ref):
    # test_harness.cpp:16-51
    inst = _inst(ref, "partition", 8, 32, 3)
    I.validate_instance(inst)
    assert (np.bincount(inst.grid.astype(np.int64)) == 32).all()
    p = _inst(ref, "permute", 16, 8, 9)
    I.validate_instance(p)
    assert sorted(p.grid.tolist()) == list(range(128))
    bad = _inst(ref, "partition", 4, 4, 1)
    bad.grid[0] = 99
    with pytest.raises(dmm.InvalidInstance):
        I.validate_instance(bad)
    bad = _inst(ref, "permute", 4, 4, 1)
    bad.grid[3] = bad.grid[5]
    with pytest.raises(dmm.InvalidInstance):
        I.validate_instance(bad)
    short = I.Instance("sort", 2, 2, 0, [1, 2, 3])
    with pytest.raises(dmm.InvalidInstance):
        I.validate_instance(short)
    counts = I.Instance("partition", 2, 2, 0, [0, 0, 0, 1])
    with pytest.raises(dmm.InvalidInstance):
        I.validate_instance(counts)


def test_load_save(ref, tmp_path):
    inst = _inst(ref, "permute", 8, 4, 2)
    path = tmp_path / "inst.txt"
    I.save_instance(inst, path)
    assert path.read_text() == ref.instance_to_text(2, 8, 4, 2, inst.grid)
    back = I.load_instance(path)
    assert (back.grid == inst.grid).all() and back.seed == 2
    with pytest.raises(dmm.Error, match="cannot open instance file"):
        I.load_instance(tmp_path / "missing.txt")


def test_report_formats():
    # instance.hpp:222-243, test_harness.cpp:95-106
    r = I.RunReport(algorithm="sort_short_wide", w=2, m=4, seed=3, correct=True)
    assert I.csv_header() == "algorithm,w,m,seed,steps,work,conflicts,correct,iterations,fallback"
    line = I.csv_line(r)
    assert line.startswith("sort_short_wide,2,4,3,")
    assert line.count(",") == I.csv_header().count(",")
    assert r.summary() == ("algorithm=sort_short_wide w=2 m=4 seed=3 steps=0 work=0 conflicts=0 correct=1 "
                           "iterations=0 fallback=0 cleanup_retries=0")


def test_run_algorithm_host_checks(ref):
    # kind mismatch (test_harness.cpp:62-65) and record_trace are refused before any launch
    with pytest.raises(dmm.InvalidInstance):
        I.run_algorithm("partition_square", _inst(ref, "sort", 4, 16, 2))
    with pytest.raises(I.TraceIncomplete):
        I.run_algorithm("partition_square", _inst(ref, "partition", 16, 16, 23), record_trace=True)
    with pytest.raises(ValueError):
        I.run_algorithm("quicksort", _inst(ref, "sort", 4, 16, 2))
    assert [I.instance_kind_for(a) for a in I.ALGORITHMS] == ["sort"] * 3 + ["partition"] * 3 + ["permute"] * 2


@pytest.mark.parametrize("alg,shapes", [
    ("partition_short_wide", [(2, 4), (2, 8), (3, 9), (4, 16), (8, 64), (2, 5), (5, 25), (32, 1024)]),
    ("partition_square", [(4, 4), (9, 9), (16, 16), (25, 25), (64, 64)]),
    ("partition_general", [(2, 4), (3, 9), (4, 16), (8, 64), (4, 4), (16, 16), (64, 64), (16, 256)]),
    ("integer_sort_general", [(2, 4), (3, 9), (4, 32), (8, 64), (4, 4), (16, 16), (64, 64)]),
])
def test_modelled_steps_match_reference(ref, alg, shapes):
    # Machine::steps() of the data-independent algorithms (test_partition.cpp:92-108 pins 684
    # for partition_short_wide 3 x 9): the closed forms equal the reference's meter
    from oracle.oracle import ALGORITHMS as REF_ALG
    for w, m in shapes:
        for seed in (1, 2):
            kind = 2 if alg == "integer_sort_general" else 1
            s, _, rr = ref.run_algorithm(REF_ALG[alg], ref.gen_instance(kind, w, m, seed), seed)
            assert s == 0 and I.modelled_steps(alg, w, m) == rr["steps"]
    assert I.modelled_steps("partition_short_wide", 3, 9) == 684


def test_unmodelled_steps_are_zero():
    # shearsort leaves (32 x 32), blocked merges (32 x 64), the recursion (32 x 16), comparison
    # sorts and the permutation depend on the data
    for alg in ("partition_general", "integer_sort_general", "permute", "sort_tall", "sort_square",
                "sort_short_wide"):
        assert I.modelled_steps(alg, 32, 32) == 0
    assert I.modelled_steps("partition_general", 32, 64) == 0
    assert I.modelled_steps("partition_general", 32, 16) == 0
    assert I.modelled_steps("partition_square", 32, 32) == 0  # not a perfect square
    assert I.modelled_steps("partition_short_wide", 32, 32) == 0  # w^2 > m

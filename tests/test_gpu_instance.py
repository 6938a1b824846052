"""run_algorithm over the B200 kernels (paper_1507_01391_b200/instance.py) against the
reference's own run_algorithm (instance.hpp:283-363, oracle/_ref) on the same instances:
every report field (the step meter where it is modelled or replayed), the permute pipeline
report, and the final grid.
Also the reference harness's run_algorithm cases (tests/test_harness.cpp:54-83)."""
import numpy as np
import torch
import pytest

import paper_1507_01391_b200 as dmm
from oracle.oracle import ALGORITHMS as REF_ALG
from paper_1507_01391_b200 import instance as I

pytestmark = pytest.mark.gpu

KIND_ID = {"sort": 0, "partition": 1, "permute": 2}

CASES = [
    ("partition_general", 32, 32), ("partition_general", 32, 16), ("partition_general", 64, 8),
    ("partition_square", 16, 16), ("partition_short_wide", 8, 64), ("integer_sort_general", 32, 16),
    ("integer_sort_general", 32, 128), ("sort_square", 16, 16), ("sort_tall", 64, 16),
    ("sort_short_wide", 4, 16), ("permute", 32, 32), ("permute", 64, 8), ("permute", 128, 64),
    ("partition_general", 64, 32), ("partition_general", 128, 32), ("integer_sort_general", 64, 8),
]


def _gen(ref, alg, w, m, seed):
    kind = I.instance_kind_for(alg)
    if kind == "sort":
        # 32-bit keys (the B200 layout); the reference's sort kind draws 64-bit words
        return I.gen_instance("sort", w, m, seed)
    return I.Instance(kind, w, m, seed, ref.gen_instance(KIND_ID[kind], w, m, seed))


@pytest.mark.parametrize("alg,w,m", CASES)
def test_run_algorithm_matches_reference(ref, alg, w, m):
    if not dmm.supported(alg, w, m):
        pytest.skip(f"{alg} {w}x{m} not compiled")
    insts = [_gen(ref, alg, w, m, seed) for seed in (1, 2, 3)]
    outs = I.run_algorithms(alg, insts)
    for inst, out in zip(insts, outs):
        s, ref_grid, rr = ref.run_algorithm(REF_ALG[alg], inst.grid.reshape(w, m), inst.seed)
        assert s == 0
        rep = out.report
        assert rep.correct and rr["correct"]
        assert (rep.algorithm, rep.w, rep.m, rep.seed) == (alg, w, m, inst.seed)
        assert (rep.iterations, rep.fallback, rep.cleanup_retries) == \
            (rr["iterations"], rr["fallback"], rr["cleanup_retries"])
        assert rep.conflicts == rr["conflicts"] == 0
        metered = (I.modelled_steps(alg, w, m) or I.sort_metered(alg, w, m) or alg == "permute"
                   or (alg in ("partition_general", "integer_sort_general")
                       and (I.leaf_metered(w, m) or I.general_metered(w, m))))
        if metered:  # the reference's meter, reproduced exactly
            assert (rep.steps, rep.work) == (rr["steps"], rr["steps"] * w)
        else:
            assert rep.steps == 0
        assert (out.result == ref_grid).all()
        if alg == "permute":
            assert out.pipeline == rr["pipeline"]
    # one instance through the single-instance entry gives the same report
    one = I.run_algorithm(alg, insts[0])
    assert one.report == outs[0].report


def test_gen_instance_matches_reference(ref):
    for kind, w, m in [("partition", 32, 32), ("partition", 4, 16), ("permute", 128, 64), ("permute", 16, 8)]:
        inst = I.gen_instance(kind, w, m, 7)
        assert (inst.grid == ref.gen_instance(KIND_ID[kind], w, m, 7).reshape(-1)).all()


def test_harness_cases(ref):
    # test_harness.cpp:55-61: an already sorted sort_square instance
    inst = I.gen_instance("sort", 16, 16, 5)
    inst.grid = np.sort(inst.grid)
    out = I.run_algorithm("sort_square", inst)
    assert out.report.correct and out.report.conflicts == 0
    # :66-71 partition_general at a small general shape
    out = I.run_algorithm("partition_general", _gen(ref, "partition_general", 64, 8, 21))
    assert out.report.correct and out.report.conflicts == 0
    # :72-77 permute reports iterations and the exact layout
    out = I.run_algorithm("permute", _gen(ref, "permute", 64, 8, 13))
    assert out.report.correct and out.report.iterations >= 1
    # :78-83 reproducibility
    inst = _gen(ref, "permute", 64, 8, 17)
    assert I.run_algorithm("permute", inst).report.summary() == I.run_algorithm("permute", inst).report.summary()
    # an explicit algorithm seed replaces the instance seed (RunOptions.seed)
    s, _, rr = ref.run_algorithm(REF_ALG["permute"], inst.grid.reshape(64, 8), 99)
    out = I.run_algorithm("permute", inst, seed=99)
    assert out.report.seed == 99 and out.pipeline == rr["pipeline"]


def test_wide_words_rejected():
    inst = I.Instance("sort", 4, 16, 0, np.full(64, 1 << 40, dtype=np.uint64))
    with pytest.raises(dmm.KeyOutOfRange):
        I.run_algorithm("sort_short_wide", inst)


@pytest.mark.parametrize("alg,w,m", [("partition_general", 32, 32), ("integer_sort_general", 32, 32),
                                     ("partition_general", 32, 64), ("integer_sort_general", 32, 128),
                                     ("partition_general", 16, 32), ("partition_general", 8, 16),
                                     ("partition_general", 8, 8), ("integer_sort_general", 16, 64)])
def test_leaf_steps_match_reference(ref, alg, w, m):
    # data-dependent meter of the w <= m leaf (merge segment sorts), replayed on the device,
    # against the reference's Machine::steps() instance by instance
    kind = 1 if alg == "partition_general" else 2
    insts = np.stack([ref.gen_instance(kind, w, m, seed) for seed in range(1, 25)]).astype(np.uint32)
    got = I.leaf_steps(torch.from_numpy(insts.view(np.int32)).cuda(), w if kind == 1 else w * m).cpu().tolist()
    exp = [ref.run_algorithm(REF_ALG[alg], insts[k].astype(np.uint64), k + 1)[2]["steps"] for k in range(len(insts))]
    assert got == exp
    assert len(set(exp)) > 1 or (w, m) == (16, 64)  # genuinely data-dependent


@pytest.mark.parametrize("alg,w,m", [("sort_short_wide", 2, 4), ("sort_short_wide", 4, 16),
                                     ("sort_short_wide", 3, 9), ("sort_short_wide", 8, 64),
                                     ("sort_square", 4, 4), ("sort_square", 16, 16), ("sort_square", 64, 64),
                                     ("sort_tall", 32, 8), ("sort_tall", 32, 1), ("sort_tall", 32, 2),
                                     ("sort_tall", 32, 16), ("sort_tall", 32, 32), ("sort_tall", 64, 16),
                                     ("sort_tall", 64, 8), ("sort_tall", 128, 32), ("sort_tall", 128, 16),
                                     ("sort_tall", 16, 16)])
def test_sort_steps_match_reference(ref, alg, w, m):
    # the comparison sorts' merge row sorts, replayed on the device (incl. the square skeleton's
    # merged-lockstep groups), against the reference's Machine::steps() instance by instance
    insts = np.stack([ref.gen_instance(0, w, m, seed) >> np.uint64(32) for seed in range(1, 17)]).astype(np.uint32)
    got = I.sort_steps(alg, torch.from_numpy(insts.view(np.int32)).cuda()).cpu().tolist()
    exp = [ref.run_algorithm(REF_ALG[alg], insts[k].astype(np.uint64), k + 1)[2]["steps"] for k in range(len(insts))]
    assert got == exp


@pytest.mark.parametrize("w,m,seeds", [(32, 32, range(1, 7)), (32, 16, range(1, 7)), (32, 2, range(1, 5)),
                                       (32, 4, range(1, 5)), (64, 8, range(1, 5)), (64, 16, range(1, 5)),
                                       (128, 64, range(1, 4))])
def test_permute_steps_match_reference(ref, w, m, seeds):
    # Machine::steps() after permute (instance.hpp:357) -- the phases the kernel replays plus the
    # finish's integer sort -- equal to the reference instance by instance, packing (32 x 32:
    # SURVEY A.3 31646, 31640, ...) and fallback (32 x 16 seeds 1, 3, 5, 6) paths alike
    seeds = list(seeds)
    grids = np.stack([ref.gen_instance(2, w, m, s) for s in seeds]).astype(np.uint32)
    got = dmm.permute_steps(grids, seeds).cpu().tolist()
    for k, s in enumerate(seeds):
        st, _, rr = ref.run_algorithm(REF_ALG["permute"], grids[k].astype(np.uint64), s)
        assert st == 0
        assert got[k] == rr["steps"], (w, m, s, got[k], rr["steps"])
    if (w, m) == (32, 32):
        assert got[:6] == [31646, 31640, 31644, 31652, 31648, 31640]  # SURVEY A.3 known answers

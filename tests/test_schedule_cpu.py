"""offline_schedule (host precompute in libdmm_b200.so) against the reference's own
offline_schedule (oracle/_ref, layout.hpp:207-230), move for move, plus the reference's
schedule test cases (tests/test_layout.cpp:155-261).  No GPU needed: the precompute is host
code, as in the reference."""
import numpy as np
import pytest

import paper_1507_01391_b200 as dmm
from paper_1507_01391_b200 import schedule as S


def random_cell_perm(rng, W, M):
    lin = rng.permutation(W * M)
    return np.stack([lin // M, lin % M], axis=1)


@pytest.mark.parametrize("W,M", [(4, 3), (16, 8), (5, 7), (32, 32), (32, 64), (3, 9), (1, 5), (7, 1), (64, 16),
                                 (32, 33), (6, 12), (2, 2)])
def test_matches_reference(ref, W, M):
    rng = np.random.default_rng(W * 1000 + M)
    for _ in range(3):
        perm = random_cell_perm(rng, W, M)
        s = S.offline_schedule(W, M, perm)
        st, rounds = ref.offline_schedule(W, M, perm)
        assert st == 0
        assert [[tuple(mv) for mv in r] for r in s.rounds] == rounds
        assert len(s.rounds) == M and all(len(r) == W for r in s.rounds)
        s.validate(W, M)


def test_identity_and_transpose(ref):
    # test_layout.cpp:156-167: identity -> m same-bank rounds
    W, M = 4, 3
    perm = [(r, c) for r in range(W) for c in range(M)]
    s = S.offline_schedule(W, M, perm)
    assert len(s.rounds) <= M
    s.validate(W, M)
    assert all(mv.src_bank == mv.dst_bank for r in s.rounds for mv in r)
    # :168-196 the 4x4 conversion permutation
    perm = [((r * 4 + c) % 4, (r * 4 + c) // 4) for r in range(4) for c in range(4)]
    s = S.offline_schedule(4, 4, perm)
    assert len(s.rounds) <= 4
    s.validate(4, 4)
    assert [[tuple(mv) for mv in r] for r in s.rounds] == ref.offline_schedule(4, 4, perm)[1]


def test_non_bijections(ref):
    bad = [(0, 0)] * 8  # test_layout.cpp:219-224
    assert ref.offline_schedule(4, 2, bad)[0] == dmm.NotBijective.status
    with pytest.raises(dmm.NotBijective):
        S.offline_schedule(4, 2, bad)
    out_of_range = [(r, c) for r in range(4) for c in range(2)]
    out_of_range[3] = (4, 0)
    assert ref.offline_schedule(4, 2, out_of_range)[0] == dmm.NotBijective.status
    with pytest.raises(dmm.NotBijective):
        S.offline_schedule(4, 2, out_of_range)
    with pytest.raises(dmm.NotBijective):
        S.offline_schedule(4, 2, [(0, 0)] * 3)


def test_validate():
    S.Schedule([[S.Move(0, 0, 1, 0), S.Move(1, 0, 2, 0), S.Move(2, 0, 3, 0), S.Move(3, 0, 0, 0)]]).validate(4, 2)
    with pytest.raises(dmm.ConflictViolation):
        S.Schedule([[S.Move(0, 0, 1, 0), S.Move(0, 1, 2, 0)]]).validate(4, 2)
    with pytest.raises(dmm.ConflictViolation):
        S.Schedule([[S.Move(0, 0, 1, 0), S.Move(2, 1, 1, 1)]]).validate(4, 2)
    with pytest.raises(dmm.OutOfBounds):
        S.Schedule([[S.Move(0, 2, 1, 0)]]).validate(4, 2)


def test_text_matches_reference(ref):
    # test_layout.cpp:247-261
    rng = np.random.default_rng(13)
    perm = random_cell_perm(rng, 5, 7)
    s = S.offline_schedule(5, 7, perm)
    text = S.schedule_to_text(s)
    assert text == ref.schedule_to_text([[tuple(mv) for mv in r] for r in s.rounds])
    back = S.schedule_from_text(text)
    assert back.rounds == s.rounds
    assert S.schedule_to_text(S.Schedule()) == ""
    assert S.schedule_from_text("").rounds == []
    assert S.schedule_from_text("0 0 1 0\n\n\n1 0 0 0\n").rounds == [[(0, 0, 1, 0)], [(1, 0, 0, 0)]]
    with pytest.raises(dmm.Error, match="malformed schedule line"):
        S.schedule_from_text("0 0 1\n")

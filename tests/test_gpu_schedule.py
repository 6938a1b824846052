"""apply_schedule on the B200 (dmm_apply_schedule) against the direct application of the
permutation (tests/test_layout.cpp:13-22 apply_perm_directly) and the reference's own schedules,
plus the reference's schedule cases (test_layout.cpp:155-245)."""
import numpy as np
import pytest
import torch

import paper_1507_01391_b200 as dmm
from paper_1507_01391_b200 import schedule as S

pytestmark = pytest.mark.gpu


def random_cell_perm(rng, W, M):
    lin = rng.permutation(W * M)
    return np.stack([lin // M, lin % M], axis=1)


def apply_directly(grid, W, M, perm):
    out = np.zeros_like(grid)
    dst = perm[:, 0] * M + perm[:, 1]
    out.reshape(grid.shape[0], -1)[:, dst] = grid.reshape(grid.shape[0], -1)
    return out


@pytest.mark.parametrize("W,M", [(16, 8), (32, 32), (32, 64), (5, 7), (4, 3), (32, 12), (3, 9), (1, 5), (7, 1),
                                 (32, 1), (2, 64)])
def test_apply_matches_direct(W, M):
    rng = np.random.default_rng(W * 100 + M)
    count = 1000
    grid = rng.integers(0, 2 ** 32, size=(count, W, M), dtype=np.uint64).astype(np.uint32)
    for _ in range(3):
        perm = random_cell_perm(rng, W, M)
        s = S.offline_schedule(W, M, perm)
        out = S.apply_schedule(grid, s)
        assert (dmm.as_uint32(out) == apply_directly(grid, W, M, perm)).all()
        again = S.apply_schedule(grid, s.upload())  # uploaded once, applied again
        assert torch.equal(again, out)


def test_reference_schedules_apply(ref):
    # a schedule the reference computed (its rounds, our kernel), test_layout.cpp:197-218
    rng = np.random.default_rng(11)
    grid = np.arange(128, dtype=np.uint32).reshape(1, 16, 8)
    for _ in range(20):
        perm = random_cell_perm(rng, 16, 8)
        st, rounds = ref.offline_schedule(16, 8, perm)
        assert st == 0
        out = S.apply_schedule(grid, S.Schedule([[S.Move(*mv) for mv in r] for r in rounds]))
        assert (dmm.as_uint32(out) == apply_directly(grid, 16, 8, perm)).all()


def test_transpose_schedule():
    # test_layout.cpp:168-196: the 4x4 conversion permutation is a transpose
    perm = np.array([((r * 4 + c) % 4, (r * 4 + c) // 4) for r in range(4) for c in range(4)])
    grid = np.arange(16, dtype=np.uint32).reshape(4, 4)
    out = dmm.as_uint32(S.apply_schedule(grid, S.offline_schedule(4, 4, perm)))
    assert (out == grid.T).all()


def test_partial_and_empty_schedules():
    grid = torch.arange(8, dtype=torch.int32, device="cuda").reshape(1, 4, 2)
    keep = torch.full((1, 4, 2), -7, dtype=torch.int32, device="cuda")
    # empty schedule: out untouched (test_layout.cpp:225-231)
    out = S.apply_schedule(grid, S.Schedule(), out=keep.clone())
    assert torch.equal(out, keep)
    # one round (test_layout.cpp:232-238): bank i offset 0 -> bank i+1 offset 0, rest untouched
    s = S.Schedule([[S.Move(0, 0, 1, 0), S.Move(1, 0, 2, 0), S.Move(2, 0, 3, 0), S.Move(3, 0, 0, 0)]])
    out = S.apply_schedule(grid, s, out=keep.clone()).cpu().numpy()
    assert out[0, :, 0].tolist() == [6, 0, 2, 4] and (out[0, :, 1] == -7).all()
    # a later round's write to the same cell wins (rounds are sequential)
    s = S.Schedule([[S.Move(0, 0, 0, 0)], [S.Move(1, 1, 0, 0)]])
    out = S.apply_schedule(grid, s, out=keep.clone()).cpu().numpy()
    assert out[0, 0, 0] == 3 and (out.reshape(-1)[1:] == -7).all()


def test_invalid_schedules_rejected_before_writes():
    grid = torch.arange(8, dtype=torch.int32, device="cuda").reshape(1, 4, 2)
    keep = torch.full((1, 4, 2), -7, dtype=torch.int32, device="cuda")
    for bad, exc in [(S.Schedule([[S.Move(0, 0, 1, 0), S.Move(0, 1, 2, 0)]]), dmm.ConflictViolation),
                     (S.Schedule([[S.Move(0, 0, 1, 0), S.Move(2, 1, 1, 1)]]), dmm.ConflictViolation),
                     (S.Schedule([[S.Move(0, 0, 1, 0)], [S.Move(0, 2, 1, 0)]]), dmm.OutOfBounds),
                     (S.Schedule([[S.Move(i % 4, 0, i % 4, 1) for i in range(5)]]), dmm.ConflictViolation)]:
        out = keep.clone()
        with pytest.raises(exc):
            S.apply_schedule(grid, bad, out=out)
        assert torch.equal(out, keep)


def test_shape_limits():
    s = S.Schedule()
    with pytest.raises(dmm.UnsupportedShape):
        S.apply_schedule(np.zeros((1, 64, 4), dtype=np.uint32), s)
    with pytest.raises(dmm.UnsupportedShape):
        S.apply_schedule(np.zeros((1, 4, 65), dtype=np.uint32), s)


def test_round_starts_disagreeing_with_n_moves_rejected():
    # shared memory is sized from the host's n_moves; a round_start table that ends
    # elsewhere, does not start at 0 or is not monotone is OutOfBounds before any staging/write
    grid = torch.arange(8, dtype=torch.int32, device="cuda").reshape(1, 4, 2)
    keep = torch.full((1, 4, 2), -7, dtype=torch.int32, device="cuda")
    good = S.Schedule([[S.Move(0, 0, 1, 0), S.Move(1, 0, 2, 0)], [S.Move(2, 0, 3, 0)]]).upload()
    for starts in ([0, 2, 5], [0, 2, 1], [1, 2, 3], [0, 4, 3]):
        ds = S.DeviceSchedule(good.moves, torch.tensor(starts, dtype=torch.int32, device="cuda"),
                              good.n_rounds, good.n_moves)
        out = keep.clone()
        with pytest.raises(dmm.OutOfBounds):
            S.apply_schedule(grid, ds, out=out)
        assert torch.equal(out, keep)
    out = S.apply_schedule(grid, good, out=keep.clone()).cpu().numpy()
    assert out[0, 1, 0] == 0 and out[0, 2, 0] == 2 and out[0, 3, 0] == 4

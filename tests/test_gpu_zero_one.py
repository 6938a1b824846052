"""Zero-one sweeps of the reference's unit tests and acceptance harness, on the B200 kernels.

* test_sort.cpp:140-151 / acceptance.cpp:92: sort_short_wide over all 256 0-1 matrices of 2 x 4;
* the same exhaustive 0-1 sweep for the integer sort's leaf machines 2 x 8 and 4 x 4 (2^16
  matrices each, domain 2), with GeneralStats and the step meter against the reference;
* 0-1 inputs of the w > m recursion (16 x 8, 32 x 16, 64 x 8): outputs, cleanup retries and
  steps against the reference;
* test_sort.cpp:372-386: the zero-one marking sweep of the tall sort (64 x 8, Rng(79)
  permutations, thresholds 1, n/4, n/2, n).
"""
import numpy as np
import pytest
import torch

import paper_1507_01391_b200 as dmm
from oracle.oracle import ALGORITHMS as REF_ALG
from paper_1507_01391_b200 import instance as I

pytestmark = pytest.mark.gpu


def _all_zero_one(w, m):
    n = w * m
    bits = np.arange(1 << n, dtype=np.uint64)[:, None]
    return ((bits >> np.arange(n, dtype=np.uint64)[None, :]) & 1).astype(np.uint32).reshape(-1, w, m)


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).cuda()


def test_short_wide_2x4_exhaustive(ref):
    grids = _all_zero_one(2, 4)
    out = dmm.sort_short_wide(_cuda(grids))
    got = dmm.as_uint32(out).reshape(256, 8)
    assert np.array_equal(got, np.sort(grids.reshape(256, 8), axis=1))
    steps = I.sort_steps("sort_short_wide", _cuda(grids)).cpu().tolist()
    for k in range(0, 256, 5):
        _, _, rr = ref.run_algorithm(REF_ALG["sort_short_wide"], grids[k].astype(np.uint64), 0)
        assert steps[k] == rr["steps"], k


@pytest.mark.parametrize("w,m", [(2, 8), (4, 4)])
def test_integer_sort_leaf_zero_one_exhaustive(ref, w, m):
    grids = _all_zero_one(w, m)
    out, st = dmm.integer_sort_general(_cuda(grids), 2, enforce_analysis_pre=False)
    got = dmm.as_uint32(out).reshape(len(grids), -1)
    assert np.array_equal(got, np.sort(grids.reshape(len(grids), -1), axis=1))
    assert bool(st.sorted.bool().all()) and int(st.cleanup_retries.max()) == 0
    steps, retries = I.general_steps(_cuda(grids), 2)
    steps = steps.cpu().numpy()
    for k in range(0, len(grids), 997):
        s, _, rr = ref.integer_sort_general_steps(grids[k], 2)
        assert s == 0 and (int(steps[k]), 0) == (rr["steps"], rr["cleanup_retries"]), k


@pytest.mark.parametrize("w,m", [(16, 8), (32, 16), (64, 8)])
def test_recursion_zero_one(ref, w, m):
    rng = np.random.default_rng(w * 1000 + m)
    # 0-1 keys with every density, and sorted/reversed blocks (the cleanup's hard cases)
    grids = (rng.random((48, w, m)) < np.linspace(0.02, 0.98, 48)[:, None, None]).astype(np.uint32)
    grids[-4] = np.sort(grids[-4].reshape(-1))[::-1].reshape(w, m)
    grids[-3] = (np.arange(w * m) % 2).reshape(w, m)
    out, st = dmm.integer_sort_general(_cuda(grids), 2, enforce_analysis_pre=False, flags=dmm.FLAG_NONSTRICT)
    steps, retries = I.general_steps(_cuda(grids), 2)
    got = dmm.as_uint32(out).reshape(len(grids), w, m)
    st_sorted = st.sorted.cpu().tolist()
    steps, retries = steps.cpu().tolist(), retries.cpu().tolist()
    st_retries = st.cleanup_retries.cpu().tolist()
    for k in range(len(grids)):
        s, rg, rr = ref.integer_sort_general_steps(grids[k], 2)
        assert s == 0
        assert np.array_equal(got[k], rg.astype(np.uint32)), k
        assert st_retries[k] == rr["cleanup_retries"] == retries[k], k
        assert st_sorted[k] == rr["sorted"], k
        assert steps[k] == rr["steps"], k


def test_tall_zero_one_marking(ref):
    W, M = 64, 8
    grids = []
    for t in range(10):
        perm = ref.gen_instance(2, W, M, 79 + t).astype(np.uint32).reshape(-1)  # a random permutation
        for i in (1, W * M // 4, W * M // 2, W * M):
            grids.append((perm >= i).astype(np.uint32).reshape(W, M))  # marking for value i
        grids.append(perm.reshape(W, M))
    grids = np.stack(grids)
    got = dmm.as_uint32(dmm.sort_tall(_cuda(grids))).reshape(len(grids), -1)
    assert np.array_equal(got, np.sort(grids.reshape(len(grids), -1), axis=1))

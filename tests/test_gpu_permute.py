"""GPU parity: kernel 4, the randomized permutation (permute.hpp:545-628).

Bar: bit-exact output region AND bit-exact PermuteReport per instance (iterations,
fallback, used_packing, packed_width, threshold, random_words, cleanup_retries,
leftover_history, shifts) against the oracle and the reference's golden fixtures."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1507_01391_b200 as dmm  # noqa: E402

FIELDS = ("iterations", "fallback", "used_packing", "packed_width", "threshold", "random_words",
          "cleanup_retries", "leftover_history", "shifts")


@pytest.mark.parametrize("m", [32, 16, 4, 2])
def test_permute_vs_oracle(port, m):
    seeds = list(range(1, 65))
    grids = np.stack([port.gen_instance(2, 32, m, s) for s in seeds]).astype(np.uint32)
    out, reps = dmm.permute(grids, seeds)
    out = dmm.as_uint32(out)
    for k, s in enumerate(seeds):
        st, oout, orep = port.permute(grids[k], s)
        assert st == 0
        assert (out[k] == oout).all(), (m, s)
        got = reps.report(k)
        for f in FIELDS:
            assert got[f] == orep[f], (m, s, f, got[f], orep[f])


def test_permute_golden(golden):
    meta, arr = golden
    for case in meta["permute"]:
        if not dmm.supported("permute", case["w"], case["m"]):
            continue
        out, reps = dmm.permute(arr[case["key"] + "_in"][None], [case["seed"]])
        assert (dmm.as_uint32(out)[0] == arr[case["key"] + "_out"]).all(), case["key"]
        got = reps.report(0)
        for f in FIELDS:
            assert got[f] == case[f], (case["key"], f)


def test_permute_large_batch_properties():
    # full-size property: the output region is out[i][j] = i*m + j for every instance
    # (verify_permute_result instance.hpp:259), the random-word budget identity holds
    # (test_permute.cpp:364-381), and the leftover history never increases.
    count, m = 1 << 14, 32
    g = dmm.gen_instances(dmm.KIND_PERMUTE, 32, m, 1000, count)
    seeds = np.arange(1000, 1000 + count, dtype=np.uint64)
    out, reps = dmm.permute(g, seeds)
    exp = torch.arange(32 * m, device="cuda", dtype=torch.int32).view(1, 32, m)
    assert bool((out == exp).all())
    budget = 32 + reps.iterations.astype(np.int64) * m + np.where(reps.used_packing != 0, 25, 0)
    assert (reps.random_words.astype(np.int64) == budget).all()
    assert (reps.threshold == 128).all()


def test_permute_shape_errors():
    g = np.zeros((1, 32, 8), dtype=np.uint32)
    with pytest.raises(dmm.ShapeViolation):  # 32x8 fails general_sort_shape_ok (permute.hpp:549)
        dmm.permute(g, [1])
    g = np.zeros((1, 32, 256), dtype=np.uint32)
    with pytest.raises(dmm.ShapeViolation):  # m | w (permute.hpp:547)
        dmm.permute(g, [1])


def test_permute_rejects_non_bijection(port):
    g = port.gen_instance(2, 32, 32, 5).astype(np.uint32)
    g[3, 3] = g[4, 4]
    with pytest.raises(dmm.InvalidInstance):
        dmm.permute(g[None], [5])


@pytest.mark.parametrize("w,m", [(32, 32), (64, 16), (128, 64)])
def test_permute_rejects_out_of_range_labels(port, w, m):
    # a label >= n has no output cell: the instance is InvalidInstance, nothing is written outside
    # its own output (tall machines deliver into global memory), its neighbours are exact
    seeds = [1, 2, 3]
    grids = np.stack([port.gen_instance(2, w, m, s) for s in seeds]).astype(np.uint32)
    bad = grids.copy()
    bad[1, 0, 0] = w * m + 5
    bad[2, w - 1, m - 1] = 0xFFFFFFFF  # the batch's last instance: past the end of the buffer
    out, reps = dmm.permute(bad, seeds, check=False)
    out = dmm.as_uint32(out)
    assert reps.status.tolist() == [0, dmm.InvalidInstance.status, dmm.InvalidInstance.status]
    ident = np.arange(w * m, dtype=np.uint32).reshape(w, m)
    assert (out[0] == ident).all()
    with pytest.raises(dmm.InvalidInstance):
        dmm.permute(bad, seeds)


@pytest.mark.parametrize("w,m,n_inst", [(64, 8, 12), (64, 16, 12), (128, 64, 6)])
def test_permute_tall_vs_oracle(port, w, m, n_inst):
    # machines taller than a warp (one per CTA); 128 x 64 is n = 8192, the BASELINE's n,
    # at a shape the reference accepts
    seeds = list(range(1, 1 + n_inst))
    grids = np.stack([port.gen_instance(2, w, m, s) for s in seeds]).astype(np.uint32)
    out, reps = dmm.permute(grids, seeds)
    out = dmm.as_uint32(out)
    for k, s in enumerate(seeds):
        st, oout, orep = port.permute(grids[k], s)
        assert st == 0
        assert (out[k] == oout).all(), (w, m, s)
        got = reps.report(k)
        for f in FIELDS:
            assert got[f] == orep[f], (w, m, s, f, got[f], orep[f])
    exp = np.arange(w * m, dtype=np.uint32).reshape(1, w, m)
    assert (out == exp).all()


@pytest.mark.parametrize("w,m", [(32, 32), (64, 16), (128, 64)])
def test_permute_in_place(port, w, m):
    # out aliasing in: every row is read before any output cell is written (tall machines write
    # their sentinels and deliveries straight into global memory after a machine barrier)
    seeds = [7, 8, 9]
    grids = np.stack([port.gen_instance(2, w, m, s) for s in seeds]).astype(np.uint32)
    ref_out, ref_reps = dmm.permute(grids, seeds)
    t = torch.from_numpy(grids.view(np.int32)).cuda()
    out, reps = dmm.permute(t, seeds, out=t)
    assert (dmm.as_uint32(t) == dmm.as_uint32(ref_out)).all()
    for k in range(len(seeds)):
        assert reps.report(k) == ref_reps.report(k)

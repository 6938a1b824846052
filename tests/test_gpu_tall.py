"""GPU parity for machines taller than a warp (w = 64, 128, 256 rows, one machine per CTA:
"virtual banks", row r in warp r / 32): general partition / integer sort with GeneralStats
and PartitionProbe snapshots, partition_square / sort_square 64 x 64, against the oracle
and the reference's golden fixtures (partition 64x16, 64x64, 256x16, integer sort 64x16).
"""
import numpy as np
import pytest

from oracle.oracle import FLAG_NO_ENFORCE_PRE

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1507_01391_b200 as dmm  # noqa: E402

TALL = [(64, 8), (64, 16), (64, 32), (64, 64), (128, 32), (128, 64), (256, 16)]


def _batch(port, kind, w, m, seeds):
    return np.stack([port.gen_instance(kind, w, m, s) for s in seeds]).astype(np.uint32)


@pytest.mark.parametrize("w,m", TALL)
def test_partition_general_tall(port, w, m):
    seeds = [1, 2, 3, 4, 5]  # odd: the last CTA holds one packed half
    grids = _batch(port, 1, w, m, seeds)
    out, st = dmm.partition_general(grids, flags=dmm.FLAG_NO_ENFORCE_PRE)
    out = dmm.as_uint32(out)
    for k in range(len(seeds)):
        ost, oout, orep = port.partition_general(grids[k], FLAG_NO_ENFORCE_PRE)
        assert ost == 0
        assert (out[k] == oout).all(), (w, m, k)
        assert int(st.cleanup_retries[k]) == orep["cleanup_retries"], (w, m, k)
    assert (out == np.arange(w, dtype=np.uint32).reshape(1, w, 1)).all()


@pytest.mark.parametrize("w,m,domain", [(64, 16, 1024), (64, 32, 1 << 20), (128, 32, 1 << 31), (256, 16, 4096)])
def test_integer_sort_tall(port, w, m, domain):
    rng = np.random.default_rng(w + m)
    grids = rng.integers(0, domain, size=(3, w, m), dtype=np.uint64).astype(np.uint32)
    out, st = dmm.integer_sort_general(grids, domain, enforce_analysis_pre=False)
    out = dmm.as_uint32(out)
    for k in range(3):
        ost, oout, orep = port.integer_sort_general(grids[k], domain, FLAG_NO_ENFORCE_PRE)
        assert ost == 0 and (out[k] == oout).all(), (w, m, k)
        assert int(st.cleanup_retries[k]) == orep["cleanup_retries"]


def test_integer_sort_tall_full_width_unsupported():
    g = np.zeros((1, 64, 16), dtype=np.uint32)
    with pytest.raises(dmm.UnsupportedShape):  # fused cleanup needs a free top bit
        dmm.integer_sort_general(g, 1 << 32)


def test_square_64(port):
    grids = _batch(port, 1, 64, 64, [3, 4, 5])
    out = dmm.as_uint32(dmm.partition_square(grids))
    for k in range(3):
        st, exp = port.simple("partition_square", grids[k])
        assert st == 0 and (out[k] == exp).all()
    rng = np.random.default_rng(64)
    g = rng.integers(0, 2 ** 32, size=(3, 64, 64), dtype=np.uint64).astype(np.uint32)
    for asc in (True, False):
        out = dmm.as_uint32(dmm.sort_square(g, ascending=asc))
        for k in range(3):
            st, exp = port.simple("sort_square", g[k], int(asc))
            assert st == 0 and (out[k] == exp).all()


def test_tall_golden(golden):
    meta, arr = golden
    ran = 0
    for case in meta["partition"]:
        if case["w"] > 32 and dmm.supported("partition_general", case["w"], case["m"]) and case["status"] == 0:
            out, st = dmm.partition_general(arr[case["key"] + "_in"])
            assert (dmm.as_uint32(out) == arr[case["key"] + "_out"]).all(), case["key"]
            assert int(st.cleanup_retries[0]) == case["cleanup_retries"]
            ran += 1
    for case in meta["intsort"]:
        if case["w"] > 32 and dmm.supported("integer_sort_general", case["w"], case["m"]):
            out, st = dmm.integer_sort_general(arr[case["key"] + "_in"], case["domain"])
            assert (dmm.as_uint32(out) == arr[case["key"] + "_out"]).all(), case["key"]
            ran += 1
    assert ran >= 4


def test_tall_probe_matches_reference(ref):
    # PartitionProbe snapshots of a 64 x 16 machine (two recursion levels deep) vs the reference
    for seed in (1, 2):
        g = ref.gen_instance(1, 64, 16, seed).astype(np.uint32)
        s, exp, rep = ref.integer_sort_general(g, 64, probe_snaps=16)
        out, st = dmm.partition_general(g, probe=True)
        snaps = dmm.as_uint32(st.snapshots)
        assert snaps.shape[0] == rep["snapshots"].shape[0]
        assert (snaps == rep["snapshots"].astype(np.uint32)).all()
        assert (dmm.as_uint32(out) == exp.astype(np.uint32)).all()


@pytest.mark.parametrize("w,m", [(64, 8), (64, 16), (64, 32), (128, 16), (128, 32)])
def test_sort_tall_multiwarp(port, w, m):
    # sort_tall sort.hpp:352-374 (Theorem 3); 128 x 32 is the reference's own test shape
    rng = np.random.default_rng(w * m)
    g = rng.integers(0, 2 ** 32, size=(3, w, m), dtype=np.uint64).astype(np.uint32)
    out = dmm.as_uint32(dmm.sort_tall(g))
    for k in range(3):
        st, exp = port.simple("sort_tall", g[k])
        assert st == 0 and (out[k] == exp).all(), (w, m, k)


@pytest.mark.parametrize("w,m,count", [(64, 16, 4096), (128, 32, 2048), (256, 16, 1024)])
def test_tall_partition_at_scale(port, w, m, count):
    # many CTAs at once (barrier-heavy multi-warp machines): every instance ends row i = i with
    # GeneralStats equal to the oracle's on a sample of instances
    g = dmm.gen_instances(dmm.KIND_PARTITION, w, m, 77, count)
    out, st = dmm.partition_general(g, flags=dmm.FLAG_NO_ENFORCE_PRE)
    rows = torch.arange(w, device="cuda", dtype=torch.int32).view(1, w, 1)
    assert bool((out == rows).all()) and int((st.status != 0).sum()) == 0
    host = dmm.as_uint32(g)
    retries = st.cleanup_retries.cpu().numpy()
    for k in range(0, count, count // 8):
        s, _, rep = port.partition_general(host[k], FLAG_NO_ENFORCE_PRE)
        assert s == 0 and retries[k] == rep["cleanup_retries"]


def test_tall_permute_at_scale(port):
    count = 512
    g = dmm.gen_instances(dmm.KIND_PERMUTE, 128, 64, 500, count)
    seeds = np.arange(500, 500 + count, dtype=np.uint64)
    out, reps = dmm.permute(g, seeds)
    exp = torch.arange(128 * 64, device="cuda", dtype=torch.int32).view(1, 128, 64)
    assert bool((out == exp).all())
    host = dmm.as_uint32(g)
    for k in range(0, count, 64):
        s, _, rep = port.permute(host[k], int(seeds[k]))
        got = reps.report(k)
        assert s == 0 and all(got[f] == rep[f] for f in ("iterations", "random_words", "packed_width",
                                                           "cleanup_retries", "leftover_history", "shifts"))

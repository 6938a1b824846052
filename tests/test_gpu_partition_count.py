"""GPU parity: the counting partition (csrc/partition_count.cu) -- leaf-only partitions and
small-domain integer sorts of 32 x {32, 64, 128, 256} views -- against the oracle (pinned to the
reference) and numpy, including the rejected instances (left unchanged, status = the exception
the reference throws: check_partition_instance partition.hpp:112-124, KeyOutOfRange).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1507_01391_b200 as dmm  # noqa: E402

MS = [32, 64, 128, 256]


def _parts(port, m, seeds):
    return np.stack([port.gen_instance(1, 32, m, s) for s in seeds]).astype(np.uint32)


@pytest.mark.parametrize("m", MS)
def test_partition_count_vs_oracle_and_rejects(port, m):
    seeds = list(range(200, 213))  # 13 instances: the last CTA is partly empty
    g = _parts(port, m, seeds)
    bad = g.copy()
    bad[3, 0, 0] = (bad[3, 0, 0] + 1) % 32  # one label count m + 1, another m - 1
    bad[7, 31, m - 1] = 32                   # label outside [0, w)
    bad[11, 5, 3] = 0xFFFFFFFF
    out, st = dmm.partition_general(bad, check=False)
    out = dmm.as_uint32(out)
    status = st.status.cpu().numpy()
    for k in range(len(seeds)):
        ost, oout, orep = port.partition_general(bad[k])
        assert status[k] == ost, k
        if ost == 0:
            assert (out[k] == oout).all(), k
            assert int(st.cleanup_retries[k]) == orep["cleanup_retries"] == 0
            assert bool(st.sorted[k])
        else:
            assert ost == dmm.InvalidInstance.status
            assert (out[k] == bad[k]).all(), k  # rejected before any step: unchanged
    with pytest.raises(dmm.InvalidInstance):
        dmm.partition_general(bad)
    # in place: the valid instances become row i = i, the rejected ones keep their input
    t = torch.from_numpy(bad.view(np.int32)).cuda()
    dmm.partition_general(t, out=t, check=False)
    got = dmm.as_uint32(t)
    rows = np.arange(32, dtype=np.uint32).reshape(32, 1)
    for k in range(len(seeds)):
        assert (got[k] == (bad[k] if k in (3, 7, 11) else np.broadcast_to(rows, (32, m)))).all()


@pytest.mark.parametrize("m", MS)
@pytest.mark.parametrize("domain", [1, 2, 3, 5, 16, 31, 32])
def test_small_domain_integer_sort(port, m, domain):
    rng = np.random.default_rng(1000 * m + domain)
    # skewed counts (geometric-ish), empty labels, one single-valued instance
    p = rng.random(domain) ** 3
    p /= p.sum()
    keys = rng.choice(domain, size=(9, 32, m), p=p).astype(np.uint32)
    keys[4] = domain - 1
    out, st = dmm.integer_sort_general(keys, domain)
    out = dmm.as_uint32(out)
    assert int((st.status != 0).sum()) == 0
    for k in range(keys.shape[0]):
        exp = np.sort(keys[k].ravel()).reshape(32, m)
        assert (out[k] == exp).all(), k
        assert int(st.cleanup_retries[k]) == 0
    for k in (0, 4):
        ost, oout, orep = port.integer_sort_general(keys[k], domain)
        assert ost == 0 and (out[k] == oout).all() and orep["cleanup_retries"] == 0


@pytest.mark.parametrize("m", [32, 128])
def test_small_domain_uniform_counts_and_out_of_range(port, m):
    # every value exactly m times (the uniform-run emission) with domain 32 ...
    g = _parts(port, m, [5, 6, 7])
    out, _ = dmm.integer_sort_general(g, 32)
    assert (dmm.as_uint32(out) == np.sort(g.reshape(3, -1), axis=1).reshape(3, 32, m)).all()
    # ... and a key outside [0, domain): KeyOutOfRange, that instance unchanged
    keys = g.copy()
    keys[1, 2, 3] = 40
    out, st = dmm.integer_sort_general(keys, 32, check=False)
    out = dmm.as_uint32(out)
    assert st.status.cpu().tolist() == [0, dmm.KeyOutOfRange.status, 0]
    assert (out[1] == keys[1]).all()
    assert port.integer_sort_general(keys[1], 32)[0] == dmm.KeyOutOfRange.status
    with pytest.raises(dmm.KeyOutOfRange):
        dmm.integer_sort_general(keys, 32)


def test_cfg1_full_batch():
    # the bench's cfg1 batch (2^16 instances of 32 x 32 from the reference generator, on device)
    count = 1 << 16
    g = dmm.gen_instances(dmm.KIND_PARTITION, 32, 32, 1, count)
    out, st = dmm.partition_general(g)
    rows = torch.arange(32, device="cuda", dtype=torch.int32).view(1, 32, 1)
    assert bool((out == rows).all()) and int((st.status != 0).sum()) == 0
    # one corrupted instance in the middle of the batch is the only one flagged
    g[count // 2, 0, 0] = 33
    out, st = dmm.partition_general(g, check=False)
    bad = torch.nonzero(st.status).flatten().cpu().tolist()
    assert bad == [count // 2]
    assert bool((out[count // 2] == g[count // 2]).all())


@pytest.mark.parametrize("m", MS)
def test_single_instance_and_constant_keys(m):
    # one instance (a CTA with three idle warps), domain 1 (one run), and a single-label batch
    keys = np.zeros((1, 32, m), dtype=np.uint32)
    out, st = dmm.integer_sort_general(keys, 1)
    assert (dmm.as_uint32(out) == 0).all() and int(st.status[0]) == 0
    keys = np.full((2, 32, m), 31, dtype=np.uint32)
    out, st = dmm.integer_sort_general(keys, 32)
    assert (dmm.as_uint32(out) == 31).all()
    _, st = dmm.partition_general(keys, check=False)
    assert st.status.cpu().tolist() == [dmm.InvalidInstance.status] * 2

"""GPU parity: kernel 1 at the paper's native mapping -- the w = 32 short-wide machine
(32 x 1024, n = 32 w^2: partition.hpp:178-185, sort.hpp:200-230) on the CTA kernel
(csrc/short_wide32.cu) against the oracle, the compiled reference and a numpy restatement of
the ShortWideHook stages (sort.hpp:189-218)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1507_01391_b200 as dmm  # noqa: E402

W, M = 32, 1024


def _parts(port, seeds):
    return np.stack([port.gen_instance(1, W, M, s) for s in seeds]).astype(np.uint32)


def _np_short_wide_stages(g, asc):
    """sort.hpp:200-218 on one W x M grid in numpy: (after_first_convert, after_first_pass, done)."""
    def rows(a, alternating):
        s = np.sort(a, axis=1)
        for i in range(a.shape[0]):
            desc = (((i % 2) == 0) != asc) if alternating else not asc
            if desc:
                s[i] = s[i][::-1]
        return s

    def to_col(a):  # row-major index v -> (v mod W, v div W)
        out = np.empty_like(a)
        v = np.arange(W * M)
        out[v % W, v // W] = a.reshape(-1)
        return out

    def to_row(a):  # column-major index u = j W + i -> (u div M, u mod M)
        i, j = np.meshgrid(np.arange(W), np.arange(M), indexing="ij")
        u = j * W + i
        out = np.empty_like(a)
        out[u // M, u % M] = a
        return out

    snaps = []
    x = g.copy()
    for p in range(2):
        x = to_col(rows(x, True))
        if p == 0:
            snaps.append(x.copy())
        x = to_row(rows(x, False))
        if p == 0:
            snaps.append(x.copy())
    x = rows(x, False)
    snaps.append(x)
    return snaps


def test_supported_and_modelled_steps():
    assert dmm.supported("partition_short_wide", W, M) and dmm.supported("sort_short_wide", W, M)
    # 5 radix row sorts (12 m) + 4 conversions (4 m) = 76 m: the reference's 77 824
    assert dmm.lib().dmm_modelled_steps(b"partition_short_wide", W, M) == 76 * M == 77824


def test_partition_short_wide_vs_oracle(port):
    seeds = list(range(1, 19))  # more machines than the grid has CTAs per wave is not needed here
    g = _parts(port, seeds)
    dev = dmm.as_uint32(dmm.gen_instances(dmm.KIND_PARTITION, W, M, 1, len(seeds)))
    assert (dev == g).all()  # the on-device generator at this shape
    out = dmm.as_uint32(dmm.partition_short_wide(g))
    for k in range(len(seeds)):
        s, exp = port.simple("partition_short_wide", g[k])
        assert s == 0 and (out[k] == exp).all()
    assert (out == np.arange(W, dtype=np.uint32).reshape(1, W, 1)).all()
    # the general partition and the small-domain integer sort take the same leaf
    out2, st = dmm.partition_general(g)
    assert (dmm.as_uint32(out2) == out).all() and int(st.cleanup_retries.sum()) == 0
    out3, _ = dmm.integer_sort_general(g, 32)
    assert (dmm.as_uint32(out3) == out).all()


def test_partition_short_wide_vs_reference(ref):
    for seed in (1, 2):
        g = ref.gen_instance(1, W, M, seed)
        s, rout, rep = ref.run_algorithm(3, g, seed)  # partition_short_wide
        assert s == 0 and rep["correct"] and rep["steps"] == 76 * M
        out = dmm.as_uint32(dmm.partition_short_wide(g.astype(np.uint32)))
        assert (out == rout.astype(np.uint32)).all()


@pytest.mark.parametrize("asc", [True, False])
def test_sort_short_wide_vs_oracle(port, asc):
    rng = np.random.default_rng(5 + asc)
    g = rng.integers(0, 2 ** 32, size=(5, W, M), dtype=np.uint64).astype(np.uint32)
    g[1] = rng.integers(0, 7, size=(W, M), dtype=np.uint64).astype(np.uint32)  # many ties
    out = dmm.as_uint32(dmm.sort_short_wide(g, ascending=asc))
    for k in range(g.shape[0]):
        exp = np.sort(g[k].ravel())
        if not asc:
            exp = exp[::-1]
        assert (out[k].ravel() == exp).all(), k
    s, exp = port.simple("sort_short_wide", g[0], int(asc))
    assert s == 0 and (out[0] == exp).all()
    # sort_wide_any dispatches 32 x 1024 to the same skeleton (sort.hpp:321-330)
    out2 = dmm.as_uint32(dmm.sort_wide_any(g, ascending=asc))
    assert (out2 == out).all()


@pytest.mark.parametrize("domain", [W * M, 1 << 32, 5])
def test_integer_sort_general_32x1024(domain):
    rng = np.random.default_rng(domain % 1000)
    g = rng.integers(0, domain, size=(4, W, M), dtype=np.uint64).astype(np.uint32)
    out, st = dmm.integer_sort_general(g, domain)
    out = dmm.as_uint32(out)
    for k in range(4):
        assert (out[k].ravel() == np.sort(g[k].ravel())).all()
    assert int(st.status.sum()) == 0


@pytest.mark.parametrize("partition,asc", [(True, True), (False, True), (False, False)])
def test_short_wide_hook_stages(port, partition, asc):
    if partition:
        g = _parts(port, [7, 8, 9])
    else:
        g = np.random.default_rng(11).integers(0, 2 ** 32, size=(3, W, M), dtype=np.uint64).astype(np.uint32)
    out, snaps = dmm.short_wide_probe(g, partition=partition, ascending=asc)
    out, snaps = dmm.as_uint32(out), dmm.as_uint32(snaps)
    for k in range(g.shape[0]):
        exp = _np_short_wide_stages(g[k], asc)
        for s in range(3):
            assert (snaps[k, s] == exp[s]).all(), (k, s)
        assert (out[k] == exp[2]).all()


def test_errors_and_status(port):
    g = _parts(port, [3, 4, 5])
    g[1, 0, 0] = 31 if g[1, 0, 0] != 31 else 30  # wrong label counts
    with pytest.raises(dmm.InvalidInstance):
        dmm.partition_short_wide(g)
    out = dmm.partition_short_wide(g, check=False)
    assert (dmm.as_uint32(out)[0] == np.arange(W, dtype=np.uint32)[:, None]).all()
    g[2, 5, 5] = 77  # label outside [0, w)
    with pytest.raises(dmm.InvalidInstance):
        dmm.partition_short_wide(g)
    keys = np.random.default_rng(1).integers(0, 100, size=(2, W, M), dtype=np.uint64).astype(np.uint32)
    keys[1, 3, 3] = 100
    with pytest.raises(dmm.KeyOutOfRange):
        dmm.integer_sort_general(keys, 100)
    with pytest.raises(dmm.ShapeViolation):
        dmm.partition_short_wide(np.zeros((1, 32, 512), dtype=np.uint32))  # w^2 > m


def test_large_batch_properties():
    # full-size properties on more machines than CTAs (persistent loop, TMA in / out):
    # every machine ends with row i = i; a sorted batch keeps its per-instance sums
    count = 600
    g = dmm.gen_instances(dmm.KIND_PARTITION, W, M, 1000, count)
    out = dmm.partition_short_wide(g)
    rows = torch.arange(W, device="cuda", dtype=torch.int32).view(1, W, 1)
    assert bool((out == rows).all())
    keys = dmm.gen_instances(dmm.KIND_SORT_U32, W, M, 5, 300)
    s = dmm.sort_short_wide(keys)
    a = keys.view(300, -1).to(torch.int64) & 0xFFFFFFFF
    b = s.view(300, -1).to(torch.int64) & 0xFFFFFFFF
    assert bool((a.sum(1) == b.sum(1)).all()) and bool((b[:, 1:] >= b[:, :-1]).all())

"""GPU: cfg5's local step (stable multisplit by label) against numpy's stable argsort, and the
single-rank global partition (the all-to-all is the identity at world size 1)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1507_01391_b200 as dmm  # noqa: E402
from paper_1507_01391_b200.distributed import global_partition  # noqa: E402


def _splitmix64(x):
    x = (x + np.uint64(0x9e3779b97f4a7c15))
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xbf58476d1ce4e5b9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94d049bb133111eb)
    return x ^ (x >> np.uint64(31))


@pytest.mark.parametrize("n,nb,shift", [(1, 8, 29), (1000, 8, 29), (1 << 20, 8, 29), ((1 << 20) + 37, 4, 30),
                                        (33333, 32, 27), (4096, 2, 31)])
def test_multisplit_stable_vs_numpy(n, nb, shift):
    keys = dmm.gen_keys(5, n)
    with np.errstate(over="ignore"):
        host = (_splitmix64(np.arange(5, 5 + n, dtype=np.uint64)) >> np.uint64(32)).astype(np.uint32)
    assert (dmm.as_uint32(keys) == host).all()
    out, starts = dmm.multisplit(keys, nb, shift)
    lab = (host >> shift) & (nb - 1)
    exp = host[np.argsort(lab, kind="stable")]
    assert (dmm.as_uint32(out) == exp).all()
    exp_starts = np.concatenate([[0], np.cumsum(np.bincount(lab, minlength=nb))[:-1]])
    assert (starts.cpu().numpy() == exp_starts).all()


def test_global_partition_single_rank():
    keys = dmm.gen_keys(0, 1 << 18)
    out, counts = global_partition(keys)
    h = dmm.as_uint32(out)
    assert (np.diff((h >> 29).astype(np.int64)) >= 0).all() and sum(counts) == 1 << 18

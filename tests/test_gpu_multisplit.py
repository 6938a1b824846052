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


def test_fused_p2p_single_rank_matches_nccl_path():
    from paper_1507_01391_b200.distributed import PeerBuffers, global_partition_p2p
    keys = dmm.gen_keys(11, (1 << 22) + 5)
    ref, _ = global_partition(keys)
    peers = PeerBuffers(keys.numel())
    got, counts = global_partition_p2p(keys, peers)
    assert torch.equal(got, ref)
    assert int(counts.sum()) == keys.numel()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_fused_scatter_simulated_ranks(world):
    # `world` ranks' fused scatters on one GPU into `world` receive buffers: the kernel and the
    # destination arithmetic give the all-to-all's (source rank, source index) order per owner
    from paper_1507_01391_b200.distributed import bucket_owner, p2p_destinations, recv_counts
    nb, shift = 8, 29
    keys = [dmm.gen_keys(1000 * s, 300000 + 1234 * s) for s in range(world)]
    wss, starts = [], []
    for k in keys:
        ws = torch.empty(int(dmm.lib().dmm_multisplit_workspace_bytes(k.numel(), nb)), dtype=torch.uint8,
                         device="cuda")
        st = torch.empty(nb, dtype=torch.int64, device="cuda")
        dmm.multisplit_count(k, nb, shift, st, ws)
        wss.append(ws)
        starts.append(st)
    all_counts = torch.stack([torch.cat([st[1:], torch.tensor([k.numel()], device="cuda")]) - st
                              for st, k in zip(starts, keys)])
    recv = recv_counts(all_counts).tolist()
    bufs = [torch.full((recv[r],), -1, dtype=torch.int32, device="cuda") for r in range(world)]
    owner = [bucket_owner(b, nb, world) for b in range(nb)]
    for s in range(world):
        ptrs = torch.tensor([bufs[owner[b]].data_ptr() for b in range(nb)], dtype=torch.int64, device="cuda")
        dmm.multisplit_scatter_to(keys[s], nb, shift, ptrs, p2p_destinations(all_counts, s), wss[s])
    torch.cuda.synchronize()
    for r in range(world):
        exp = []
        for k in keys:
            h = dmm.as_uint32(k)
            lab = h >> shift
            loc = h[np.argsort(lab, kind="stable")]
            exp.append(loc[np.isin(loc >> shift, [b for b in range(nb) if owner[b] == r])])
        assert (dmm.as_uint32(bufs[r]) == np.concatenate(exp)).all()


def test_multisplit_rejects_misaligned_keys_and_bad_shift():
    # a view with a storage offset would feed the 16-byte loads a misaligned pointer;
    # label bits outside the 32-bit key are undefined shifts -- both are argument errors now,
    # and the context stays usable afterwards
    keys = dmm.gen_keys(3, 4096)
    with pytest.raises(ValueError):
        dmm.multisplit(keys[1:], 8, 29)
    with pytest.raises(ValueError):
        dmm.multisplit(keys, 8, 30)  # bits [30, 33)
    with pytest.raises(ValueError):
        dmm.multisplit(keys, 2, 32)
    out, _ = dmm.multisplit(keys, 8, 29)
    h = dmm.as_uint32(keys)
    assert (dmm.as_uint32(out) == h[np.argsort(h >> 29, kind="stable")]).all()
    shifted = keys[4:].clone()  # an aligned copy of the same tail is fine
    out, _ = dmm.multisplit(shifted, 4, 30)
    hs = dmm.as_uint32(shifted)
    assert (dmm.as_uint32(out) == hs[np.argsort(hs >> 30, kind="stable")]).all()

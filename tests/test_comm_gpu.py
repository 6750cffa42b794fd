"""The library's NCCL halo exchange (csrc/comm.cu, partition.NcclHalo) on one GPU.

One GPU cannot host two NCCL ranks, so the multi-rank transport runs here as a one-rank
communicator whose halo plan sends to itself: the same pdg_comm_load / unique id / init / plan /
pack -> grouped ncclSend+ncclRecv -> unpack path, eager and captured in a CUDA graph.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    return torch


def _loop_part(nt, n_own, rng):
    from paper_2605_16082_b200.partition import Part
    ghosts = np.arange(n_own, nt)
    src = np.sort(rng.choice(n_own, size=nt - n_own, replace=False)).astype(np.int32)
    dst = ghosts.astype(np.int32)
    return Part(rank=0, nparts=1, lo=0, hi=n_own, ghosts=ghosts, send={0: src}, recv={0: dst},
                ring=np.ones(nt - n_own, np.int32), send1={0: src[: len(src) // 2]}, recv1={0: dst[: len(dst) // 2]})


def test_nccl_self_exchange_eager_and_graph(torch):
    from paper_2605_16082_b200.partition import NcclHalo
    rng = np.random.default_rng(3)
    dev = torch.device("cuda", 0)
    nt, n_own, L = 300, 240, 4
    part = _loop_part(nt, n_own, rng)
    halo = NcclHalo(part, nt, dev, L)
    a = torch.as_tensor(rng.standard_normal((6, L, nt)), device=dev)
    b = torch.as_tensor(rng.standard_normal((3, 3, nt)), device=dev)
    src, dst = part.send1[0], part.recv1[0]
    halo.exchange([a], deep=False)
    torch.cuda.synchronize()
    an = a.cpu().numpy()
    assert np.array_equal(an[..., dst], an[..., src])
    halo.start([b], deep=True)
    halo.finish([b], deep=True)
    bn = b.cpu().numpy()
    assert np.array_equal(bn[..., part.recv[0]], bn[..., part.send[0]])
    # captured: the replay moves the values current at replay time
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        halo.start([b], deep=True)
        halo.finish([b], deep=True)
    b.copy_(torch.as_tensor(rng.standard_normal((3, 3, nt)), device=dev))
    before = b.cpu().numpy()
    g.replay()
    torch.cuda.synchronize()
    after = b.cpu().numpy()
    assert np.array_equal(after[..., part.recv[0]], before[..., part.send[0]])
    own = np.setdiff1d(np.arange(nt), part.recv[0])
    assert np.array_equal(after[..., own], before[..., own])


def test_plan_rejects_oversized_message(torch):
    import ctypes

    from paper_2605_16082_b200 import _lib
    from paper_2605_16082_b200.partition import NcclHalo
    rng = np.random.default_rng(5)
    dev = torch.device("cuda", 0)
    nt, n_own = 64, 40
    halo = NcclHalo(_loop_part(nt, n_own, rng), nt, dev, 1)
    big = torch.zeros(19, nt, dtype=torch.float64, device=dev)     # 19 planes > 18 L = 18
    fp = (ctypes.c_void_p * 1)(big.data_ptr())
    npl = (ctypes.c_longlong * 1)(19)
    from paper_2605_16082_b200.device import stream_ptr
    assert _lib.lib().pdg_halo_start(halo.plans[False], 1, fp, npl, stream_ptr()) != 0


def test_halo_2d_3d_entries(torch):
    """pdg_halo_2d / pdg_halo_3d (the SURVEY section 8b names: blocking start + finish)."""
    import ctypes
    from paper_2605_16082_b200 import _lib
    from paper_2605_16082_b200.device import stream_ptr
    from paper_2605_16082_b200.partition import NcclHalo
    rng = np.random.default_rng(5)
    dev = torch.device("cuda", 0)
    nt, n_own, L = 200, 150, 3
    part = _loop_part(nt, n_own, rng)
    halo = NcclHalo(part, nt, dev, L)
    lb = _lib.lib()
    S = torch.as_tensor(rng.standard_normal((3, 3, nt)), device=dev)
    _lib.check(lb.pdg_halo_2d(halo.plans[True], ctypes.c_void_p(S.data_ptr()), stream_ptr()), "halo_2d")
    a = torch.as_tensor(rng.standard_normal((6, L, nt)), device=dev)
    fp = (ctypes.c_void_p * 1)(a.data_ptr())
    npl = (ctypes.c_longlong * 1)(6 * L)
    _lib.check(lb.pdg_halo_3d(halo.plans[False], 1, fp, npl, stream_ptr()), "halo_3d")
    torch.cuda.synchronize()
    sn, an = S.cpu().numpy(), a.cpu().numpy()
    assert np.array_equal(sn[..., part.recv[0]], sn[..., part.send[0]])
    assert np.array_equal(an[..., part.recv1[0]], an[..., part.send1[0]])

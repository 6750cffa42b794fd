"""Partition maps vs the oracle restatement, and the gloo halo exchange (CPU, world_size 2)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import partition as OP
from paper_2605_16082_b200 import mesh as PM
from paper_2605_16082_b200 import partition as PP
from paper_2605_16082_b200.errors import TooManyRanks


def basin(nx, ny):
    return PM.hilbert_reorder(PM.generate_basin_mesh(nx, ny, 1e3 * nx, 1e3 * ny, lambda x, y: -10.0 - 0 * x))


@pytest.mark.parametrize("nx,ny,P", [(2, 2, 1), (2, 2, 2), (8, 6, 3), (32, 32, 4), (16, 9, 7), (5, 5, 8)])
def test_maps_bit_exact_vs_oracle(nx, ny, P):
    m = basin(nx, ny)
    parts = PP.decompose(m, P)
    bounds, ghosts, send, recv = OP.maps(m.nbr.tolist(), [1] * m.nt, P)
    assert [p.lo for p in parts] + [parts[-1].hi] == bounds
    for r, p in enumerate(parts):
        assert p.ghosts.tolist() == ghosts[r]
        assert {k: v.tolist() for k, v in p.recv.items()} == recv[r]
        assert {k: v.tolist() for k, v in p.send.items()} == send[r]


@pytest.mark.parametrize("nx,ny,P", [(8, 6, 3), (32, 32, 4), (16, 9, 7), (5, 5, 8)])
def test_deep_ring_maps_bit_exact_vs_oracle(nx, ny, P):
    """3 ghost rings (the partitioned stepper's 2D sub-cycle): rings, all-ring and ring-1 maps."""
    m = basin(nx, ny)
    parts = PP.decompose(m, P, depth=3)
    bounds, ghosts, rings, send, recv, send1, recv1 = OP.deep_maps(m.nbr.tolist(), [1] * m.nt, P, 3)
    assert [p.lo for p in parts] + [parts[-1].hi] == bounds
    for r, p in enumerate(parts):
        assert p.ghosts.tolist() == ghosts[r]
        assert p.ring.tolist() == rings[r]
        assert {k: v.tolist() for k, v in p.recv.items()} == recv[r]
        assert {k: v.tolist() for k, v in p.send.items()} == send[r]
        assert {k: v.tolist() for k, v in p.recv1.items()} == recv1[r]
        assert {k: v.tolist() for k, v in p.send1.items()} == send1[r]
    one = PP.decompose(m, P)                        # ring 1 of the deep partition == the one-ring one
    for p, q in zip(parts, one):
        gl = p.ghosts[p.ring == 1]
        assert gl.tolist() == q.ghosts.tolist()


def test_partition_properties():
    m = basin(32, 32)
    parts = PP.decompose(m, 4)
    owned = np.concatenate([np.arange(p.lo, p.hi) for p in parts])
    assert np.array_equal(owned, np.arange(m.nt))                       # disjoint and covering
    sizes = [p.n_own for p in parts]
    assert max(sizes) / min(sizes) <= 1.15
    for p in parts:                                                      # ghost layer = edge neighbours
        nb = m.nbr[p.lo:p.hi].ravel()
        expect = sorted(set(int(e) for e in nb if e >= 0 and not p.lo <= e < p.hi))
        assert p.ghosts.tolist() == expect
    one = PP.decompose(m, 1)[0]
    assert one.ghosts.size == 0 and not one.send and not one.recv       # P = 1
    with pytest.raises(TooManyRanks):
        PP.decompose(basin(1, 1), 3)


def test_weighted_split():
    w = np.array([1, 1, 1, 10, 1, 1, 1, 1, 1, 1])
    b = PP.split_ranges(w, 3)
    _, ob = OP.owners(w.tolist(), 3)
    assert b.tolist() == ob


def test_local_mesh_remap():
    m = basin(6, 4)
    p = PP.decompose(m, 3)[1]
    lm = PP.local_mesh(m, p)
    gl = lm.global_ids
    for i in range(p.n_own):                      # owned columns see every neighbour locally
        for k in range(3):
            e = m.nbr[gl[i], k]
            assert (lm.nbr[i, k] == -1) == (e < 0)
            if e >= 0:
                assert gl[lm.nbr[i, k]] == e


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, nx, ny, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = basin(nx, ny)
    parts = PP.decompose(m, world)
    p = parts[rank]
    lm = PP.local_mesh(m, p)
    halo = PP.DistHalo(p, lm.nt, torch.device("cpu"))
    L = 3
    rng = np.random.default_rng(7)
    glob = rng.standard_normal((2, 6, L, m.nt))                # a P6N field in the device layout
    loc = torch.full((2, 6, L, lm.nt), np.nan, dtype=torch.float64)
    loc[..., :p.n_own] = torch.as_tensor(glob[..., p.lo:p.hi])
    rid = torch.full((3, lm.nt), -1.0, dtype=torch.float64)
    rid[:, :p.n_own] = float(rank)
    halo.exchange([loc, rid])
    ok_vals = np.array_equal(loc.numpy(), glob[..., lm.global_ids])           # ghosts == owners, bitwise
    owner = np.repeat(np.arange(world), [q.n_own for q in parts])
    ok_ids = np.array_equal(rid[0, p.n_own:].numpy(), owner[p.ghosts].astype(float))
    before = loc.clone()
    halo.exchange([loc, rid])                                                  # idempotent
    ok_idem = torch.equal(before, loc)
    ret[rank] = bool(ok_vals and ok_ids and ok_idem)
    dist.destroy_process_group()


def test_gloo_halo_exchange_world2():
    world = 2
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), 12, 8, ret), nprocs=world, join=True)
    assert ret[0] and ret[1]


def test_amdahl_report_exact_fit(tmp_path):
    from paper_2605_16082_b200.partition import amdahl_report
    r = amdahl_report({p: 3.0 + 12.0 / p for p in (1, 2, 4, 8)}, str(tmp_path / "amdahl.csv"))
    assert abs(r["a"] - 3.0) <= 1e-9 and abs(r["b"] - 12.0) <= 1e-9 and r["r2"] > 1 - 1e-12
    lines = (tmp_path / "amdahl.csv").read_text().splitlines()
    assert lines[0] == "P,T,T_fit,a,b,r2" and len(lines) == 5
    c = amdahl_report({1: 2.0, 2: 2.0, 4: 2.0})
    assert abs(c["b"]) <= 1e-12 and abs(c["a"] - 2.0) <= 1e-12
    with pytest.raises(ValueError):
        amdahl_report({4: 1.0})


def test_exchange_count_of_the_step_plan():
    from paper_2605_16082_b200.partition import PAPER_EXCHANGES_PER_STEP, exchanges_per_step
    assert exchanges_per_step(20) == 38 and PAPER_EXCHANGES_PER_STEP == 100
    assert exchanges_per_step(4) == 2 * 4 + 2 + 4

"""Partitioned stepping on one GPU (virtual ranks): bitwise equal to the unpartitioned run."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pdg():
    import paper_2605_16082_b200 as p
    return p


@pytest.mark.parametrize("P", [2, 3, 4, 7])
def test_partition_invariance_bitwise(pdg, P):
    from paper_2605_16082_b200.partition import PartitionedRun
    from paper_2605_16082_b200.scenarios import make_case
    c = make_case("c4", scale=0.02, L=6)                   # 20 x 10 squares of the coastal basin
    ref = pdg.stepper.ImexStepper(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v)
    ref.use_graph = False
    ref.set_state(**c.state)
    ref.step(3)
    ref.check()
    g = ref.get_state()
    run = PartitionedRun(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v, P)
    run.set_state(**c.state)
    run.step(3)
    run.check()
    s = run.get_state()
    for k in ("eta", "qx", "qy", "ux", "uy", "T"):
        assert np.array_equal(s[k], g[k]), (P, k, float(np.abs(s[k] - g[k]).max()))
    assert run.group.exchanges == 3 * (2 * 4 + (c.m // 2 + c.m))   # q, F3D->2D, mis, u/T per stage + 2D per substep


def _c4_small(L=5):
    from paper_2605_16082_b200.scenarios import make_case
    return make_case("c4", scale=0.02, L=L)


def test_partition_graph_equals_eager(pdg):
    """The whole P-rank lockstep step captured in one CUDA graph == eager launches, bitwise."""
    from paper_2605_16082_b200.partition import PartitionedRun
    c = _c4_small()
    out = []
    for graph in (False, True):
        run = PartitionedRun(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v, 3)
        run.use_graph = graph
        run.set_state(**c.state)
        run.step(4)
        run.check()
        out.append(run.get_state())
        assert run.group.exchanges == 4 * (2 * 4 + (c.m // 2 + c.m))
        assert bool(run.graphs) == graph
    for k in ("eta", "qx", "qy", "ux", "uy", "T"):
        assert np.array_equal(out[0][k], out[1][k]), k


@pytest.mark.parametrize("P", [2, 4])
def test_schedule_check_shipped_plan(pdg, P):
    """Debug poisoning: ghosts NaN while their exchange is pending; the shipped step
    plan never reads one, and the poisoned run stays bitwise equal to the plain one."""
    from paper_2605_16082_b200.partition import PartitionedRun
    c = _c4_small()
    ref = PartitionedRun(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v, P)
    ref.set_state(**c.state)
    ref.step(2)
    g = ref.get_state()
    run = PartitionedRun(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v, P)
    run.schedule_check = True
    run.set_state(**c.state)
    run.step(2)
    s = run.get_state()
    for k in ("eta", "qx", "qy", "ux", "uy", "T"):
        assert np.array_equal(s[k], g[k]), k


@pytest.mark.parametrize("skip", ["mis", "q", "state2d", "uT", "f3d2d"])
def test_schedule_violation_detected(pdg, skip):
    """A step plan that leaves out one exchange reads poisoned ghosts: ScheduleViolation."""
    from paper_2605_16082_b200.errors import ScheduleViolation
    from paper_2605_16082_b200.partition import PartitionedRun
    c = _c4_small()
    run = PartitionedRun(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v, 2)
    run.schedule_check = True
    run._skip_exchanges = {skip}
    run.set_state(**c.state)
    with pytest.raises(ScheduleViolation):
        run.step(2)


@pytest.mark.parametrize("nx,ny,P,var", [(8, 6, 3, False), (32, 32, 4, True), (40, 17, 7, True), (12, 9, 1, False)])
def test_gpu_decomposition_bit_exact(pdg, nx, ny, P, var):
    """decompose(device=...) (csrc/partition.cu: prefix-sum split + ring BFS on the GPU) equals the
    host restatement map for map, including variable layer weights and 3 ghost rings."""
    import torch
    from paper_2605_16082_b200.partition import decompose, split_ranges
    m = pdg.mesh.hilbert_reorder(pdg.mesh.generate_basin_mesh(nx, ny, 1e4, 8e3, lambda x, y: -20.0 + 0 * x))
    rng = np.random.default_rng(nx * ny + P)
    layers = rng.integers(1, 40, m.nt) if var else np.full(m.nt, 10)
    dev = torch.device("cuda", 0)
    assert np.array_equal(split_ranges(layers, P, device=dev), split_ranges(layers, P))
    for depth in (1, 3):
        h = decompose(m, P, layers, depth=depth)
        g = decompose(m, P, layers, depth=depth, device=dev)
        for a, b in zip(h, g):
            assert (a.lo, a.hi) == (b.lo, b.hi)
            assert np.array_equal(a.ghosts, b.ghosts) and np.array_equal(a.ring, b.ring)
            for d in ("send", "recv", "send1", "recv1"):
                da, db = getattr(a, d), getattr(b, d)
                assert sorted(da) == sorted(db)
                assert all(np.array_equal(da[k], db[k]) for k in da)


@pytest.mark.parametrize("P,graph", [(2, False), (3, True), (4, True)])
def test_peer_store_halos_bitwise(pdg, P, graph):
    """Device-initiated halos (csrc/p2p.cu: push kernels store into the peers' inbox windows and
    release an epoch flag, pull kernels acquire it and unpack), virtual ranks with raw pointers,
    eager and graph-replayed (device-resident epochs): bitwise equal to P = 1."""
    from paper_2605_16082_b200.partition import P2PGroup, PartitionedRun
    c = _c4_small()
    ref = pdg.stepper.ImexStepper(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v)
    ref.use_graph = False
    ref.set_state(**c.state)
    ref.step(4)
    g = ref.get_state()
    run = PartitionedRun(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v, P, transport="p2p-virtual")
    assert isinstance(run.group, P2PGroup)
    run.use_graph = graph
    run.set_state(**c.state)
    run.step(4)
    run.check()
    s = run.get_state()
    for k in ("eta", "qx", "qy", "ux", "uy", "T"):
        assert np.array_equal(s[k], g[k]), (P, k, float(np.abs(s[k] - g[k]).max()))
    assert bool(run.graphs) == graph


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_partition_invariance_100_steps(pdg, name):
    """SPEC criterion 9: the seiche (C2: standing wave, barotropic) and the lock exchange (C3:
    density front, baroclinic) over 100 internal steps, graph-replayed: P = 2, 4, 7 bitwise equal
    to P = 1 in every prognostic field."""
    from paper_2605_16082_b200.partition import PartitionedRun
    from paper_2605_16082_b200.scenarios import make_case
    c = make_case("c2", L=6) if name == "c2" else make_case("c3", scale=0.08, L=8)
    ref = pdg.stepper.ImexStepper(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v)
    ref.set_state(**c.state)
    ref.step(100)
    ref.check()
    g = ref.get_state()
    for P in (2, 4, 7):
        run = PartitionedRun(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v, P)
        run.set_state(**c.state)
        run.step(100)
        run.check()
        s = run.get_state()
        for k in ("eta", "qx", "qy", "ux", "uy", "T"):
            assert np.array_equal(s[k], g[k]), (name, P, k, float(np.abs(s[k] - g[k]).max()))

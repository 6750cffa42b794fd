"""2D external mode: CUDA path vs the CPU oracle (and the golden reference vectors)."""
import numpy as np
import pytest

from oracle import ext2d as O
from oracle import geom as OG

pytestmark = pytest.mark.gpu

TOL_RHS = 1e-12      # normwise relative L_inf per RHS evaluation (north_star)
TOL_TRAJ = 1e-9      # after 100 steps


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.fixture(scope="module")
def pdg():
    import paper_2605_16082_b200 as p
    return p


def basin(pdg, nx=32, ny=32, lx=1e4, ly=1e4, wavy=True):
    def bed(x, y):
        return -20.0 + (5.0 * np.sin(np.pi * x / lx) * np.cos(2 * np.pi * y / ly) if wavy else 0.0 * x)
    return pdg.mesh.hilbert_reorder(pdg.mesh.generate_basin_mesh(nx, ny, lx, ly, bed))


def rand_state(pdg, mesh, seed=3, lx=1e4):
    rng = np.random.default_rng(seed)
    eta = 0.1 * np.cos(np.pi * mesh.x / lx) + 0.01 * rng.standard_normal((mesh.nt, 3))
    return pdg.State2D(eta, rng.standard_normal((mesh.nt, 3)), rng.standard_normal((mesh.nt, 3)))


def test_tendencies_vs_oracle(pdg):
    m = basin(pdg)
    st = rand_state(pdg, m)
    p = pdg.PhysParams()
    rng = np.random.default_rng(1)
    f3 = rng.standard_normal((m.nt, 3, 2))
    src = 1e-3 * rng.standard_normal((m.nt, 3))
    pa = 10 * rng.standard_normal((m.nt, 3))
    d = pdg.external2d.external_tendencies(st, m, p, f3d2d=f3, source=src, patm=pa)
    o = O.tendencies(st, m, p, f3d2d=f3, source=src, patm=pa)
    for a, b in zip(d, o):
        assert rel(a, b) <= TOL_RHS
    r = pdg.external2d.rhs_free_surface(st, m, p, source=src)
    assert rel(r, O.free_surface_residual(st, m, p, source=src)) <= TOL_RHS
    r = pdg.external2d.rhs_depth_momentum(st, m, p, f3d2d=f3, patm=pa)
    assert rel(r, O.momentum_residual(st, m, p, f3d2d=f3, patm=pa)) <= TOL_RHS
    els = np.array([5, 0, 77, 1000, 3])
    d = pdg.external2d.external_tendencies(st, m, p, els=els, f3d2d=f3)
    o = O.tendencies(st, m, p, els=els, f3d2d=f3)
    for a, b in zip(d, o):
        assert rel(a, b) <= TOL_RHS


def test_golden_ext2d(pdg, golden):
    g = golden("mesh")
    m = pdg.mesh.hilbert_reorder(pdg.mesh.make_mesh(g["vx"], g["vy"], g["vb"], g["raw_tri"]))
    e = golden("ext2d")
    p = pdg.PhysParams(f=1e-4, cd=2.5e-3, alpha=0.2, t_ref=12.5)
    st = pdg.State2D(e["eta"], e["qx"], e["qy"])
    d = pdg.external2d.external_tendencies(st, m, p, f3d2d=e["f3d2d"], source=e["source"], patm=e["patm"])
    for a, k in zip(d, ["d_eta", "d_qx", "d_qy"]):
        assert rel(a, e[k]) <= TOL_RHS
    ex = pdg.external2d.subcycle_external(st, m, p, 10, 2.0, f3d2d=e["f3d2d"])
    for a, k in [(ex.state.eta, "sub_eta"), (ex.state.qx, "sub_qx"), (ex.qbar_x, "qbar_x"), (ex.f2d_y, "f2d_y")]:
        assert rel(a, e[k]) <= 1e-11
    m.btag = e["open_btag"]
    d = pdg.external2d.external_tendencies(st, m, p, eta_bc=lambda t: 0.05 + 1e-3 * t)
    for a, k in zip(d, ["open_d_eta", "open_d_qx", "open_d_qy"]):
        assert rel(a, e[k]) <= TOL_RHS


def test_subcycle_100_steps(pdg):
    """Config 1 parity variant: 100 SSP-RK3 steps, dt2d = 2 s, <= 1e-9 vs the oracle."""
    m = basin(pdg)
    st = rand_state(pdg, m)
    p = pdg.PhysParams()
    rng = np.random.default_rng(5)
    f3 = 1e-2 * rng.standard_normal((m.nt, 3, 2))
    ex = pdg.external2d.subcycle_external(st, m, p, 100, 2.0, f3d2d=f3)
    o = O.subcycle(st, m, p, 100, 2.0, f3d2d=f3)
    assert rel(ex.state.eta, o[0].eta) <= TOL_TRAJ
    assert rel(ex.state.qx, o[0].qx) <= TOL_TRAJ
    assert rel(ex.state.qy, o[0].qy) <= TOL_TRAJ
    assert rel(ex.qbar_x, o[1]) <= TOL_TRAJ and rel(ex.qbar_y, o[2]) <= TOL_TRAJ
    assert rel(ex.f2d_x, o[3]) <= TOL_TRAJ and rel(ex.f2d_y, o[4]) <= TOL_TRAJ
    assert ex.state.t == pytest.approx(200.0)


def test_lake_at_rest(pdg):
    """Well-balancedness (SPEC acceptance 3): eta = 0, Q = 0 over wavy bathymetry stays at rest."""
    m = basin(pdg, 16, 16)
    z = np.zeros((m.nt, 3))
    ex = pdg.external2d.subcycle_external(pdg.State2D(z, z, z), m, pdg.PhysParams(), 200, 2.0)
    assert np.abs(ex.state.eta).max() <= 1e-12 * 25
    assert np.abs(ex.state.qx).max() <= 1e-12 * 25 and np.abs(ex.state.qy).max() <= 1e-12 * 25


def test_volume_conservation(pdg):
    m = basin(pdg, 16, 16)
    st = rand_state(pdg, m)
    ex = pdg.external2d.subcycle_external(st, m, pdg.PhysParams(), 50, 2.0)
    v0 = O.mh_apply(st.eta, m.j2d).sum()
    v1 = O.mh_apply(ex.state.eta, m.j2d).sum()
    assert abs(v1 - v0) <= 1e-12 * np.abs(O.mh_apply(np.abs(st.eta), m.j2d)).sum()


def test_errors(pdg):
    m = basin(pdg, 8, 8)
    st = rand_state(pdg, m)
    p = pdg.PhysParams()
    with pytest.raises(pdg.errors.CflViolation):
        pdg.external2d.subcycle_external(st, m, p, 2, 200.0)
    assert pdg.external2d.check_cfl(st, m, p, 2.0) == pytest.approx(O.cfl_ratio(st, m, p, 2.0), rel=1e-14)
    dry = pdg.State2D(st.eta - 30.0, st.qx, st.qy)
    with pytest.raises(pdg.errors.DryColumn):
        pdg.external2d.external_tendencies(dry, m, p)
    with pytest.raises(pdg.errors.DryColumn):
        pdg.external2d.check_cfl(dry, m, p, 2.0)


def test_torch_inputs_zero_copy(pdg):
    import torch
    m = basin(pdg, 8, 8)
    st = rand_state(pdg, m)
    p = pdg.PhysParams()
    ts = pdg.State2D(*(torch.as_tensor(a, device="cuda") for a in (st.eta, st.qx, st.qy)))
    d = pdg.external2d.external_tendencies(ts, m, p)
    assert isinstance(d[0], torch.Tensor) and d[0].is_cuda
    o = O.tendencies(st, m, p)
    assert rel(d[0].cpu().numpy(), o[0]) <= TOL_RHS


def test_trace_helpers_vs_reference(pdg, golden):
    """trace_int / trace_ext / edge_celerity (external2d.py:95-116) against the reference."""
    g = golden("traces")
    eta, b = g["eta"], g["b"]
    els = np.arange(eta.shape[0])
    for k in range(3):
        ti = pdg.external2d.trace_int(eta, els, k)
        te = pdg.external2d.trace_ext(eta, g[f"nbr{k}"], g[f"nbrk{k}"])
        assert np.array_equal(ti, g[f"ti{k}"]) and np.array_equal(te, g[f"te{k}"])
        bi = pdg.external2d.trace_int(b, els, k)
        be = pdg.external2d.trace_ext(b, g[f"nbr{k}"], g[f"nbrk{k}"])
        assert np.array_equal(pdg.external2d.edge_celerity(ti, te, bi, be, 9.81), g[f"cel{k}"])
    with pytest.raises(pdg.errors.DryColumn):
        pdg.external2d.edge_celerity(np.array([-30.0]), np.array([0.0]), np.array([-20.0]), np.array([-20.0]), 9.81)

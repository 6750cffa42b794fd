"""Fused IMEX step on the GPU vs the oracle orchestrator (oracle/stepper.py) and the golden trajectory."""
from types import SimpleNamespace

import numpy as np
import pytest

from oracle import ext2d as OE
from oracle import geom as OG
from oracle import stepper as OS

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.fixture(scope="module")
def pdg():
    import paper_2605_16082_b200 as p
    return p


def _setup(pdg, nx=12, ny=8, L=6, seed=4, baroclinic=True):
    lx, ly = 1.2e4, 8e3

    def bed(x, y):
        return -20.0 + 5.0 * np.sin(np.pi * x / lx) * np.cos(2 * np.pi * y / ly)
    m = pdg.mesh.hilbert_reorder(pdg.mesh.generate_basin_mesh(nx, ny, lx, ly, bed))
    om = OG.hilbert_reorder(OG.basin_mesh(nx, ny, lx, ly, bed))
    rng = np.random.default_rng(seed)
    nt, P = m.nt, m.nt * L
    eta = 0.1 * np.cos(np.pi * m.x / lx) + 0.01 * rng.standard_normal((nt, 3))
    qx, qy = 0.3 * rng.standard_normal((nt, 3)), 0.3 * rng.standard_normal((nt, 3))
    ux, uy = 0.05 * rng.standard_normal((P, 6)), 0.05 * rng.standard_normal((P, 6))
    xc = np.repeat(m.x.mean(1), L)[:, None] * np.ones((1, 6))
    T = np.where(xc < lx / 2, 15.0, 10.0) if baroclinic else np.full((P, 6), 12.5)
    p = pdg.PhysParams(f=1e-4, cd=2.5e-3, alpha=0.2 if baroclinic else 0.0, t_ref=12.5, tau_x=0.05, tau_y=-0.02)
    return m, om, p, dict(eta=eta, qx=qx, qy=qy, ux=ux, uy=uy, T=T)


def _oracle_run(om, L, p, s0, nsteps, dt, m, kv, nu_v):
    s = SimpleNamespace(grid=OG.extrude(om, L, s0["eta"]), ux=s0["ux"], uy=s0["uy"], T=s0["T"],
                        s2d=OE.S2(s0["eta"].copy(), s0["qx"], s0["qy"], 0.0))
    for _ in range(nsteps):
        s = OS.imex_step(s, p, dt, m, kv, nu_v)
    return s


@pytest.mark.parametrize("graph", [False, True])
def test_step_vs_oracle(pdg, graph):
    L, dt, msub, kv, nu_v = 6, 40.0, 4, 1e-3, 1e-4
    m, om, p, s0 = _setup(pdg, L=L)
    st = pdg.stepper.ImexStepper(m, L, p, dt, msub, kv, nu_v)
    st.use_graph = graph
    st.set_state(**s0)
    st.step(3)
    st.check()
    g = st.get_state()
    o = _oracle_run(om, L, p, s0, 3, dt, msub, kv, nu_v)
    for k, ref in [("ux", o.ux), ("uy", o.uy), ("T", o.T), ("eta", o.s2d.eta), ("qx", o.s2d.qx), ("qy", o.s2d.qy)]:
        assert rel(g[k], ref) <= 1e-10, k
    assert g["t"] == pytest.approx(3 * dt)


def test_golden_step(pdg, golden):
    gm = golden("mesh")
    g = golden("step")
    m = pdg.mesh.hilbert_reorder(pdg.mesh.make_mesh(gm["vx"], gm["vy"], gm["vb"], gm["raw_tri"]))
    L = int(g["L"])
    p = pdg.PhysParams(f=1e-4, cd=2.5e-3, alpha=0.2, t_ref=12.5, tau_x=0.05, tau_y=-0.02)
    st = pdg.stepper.ImexStepper(m, L, p, float(g["dt"]), int(g["m"]), float(g["kv"]), float(g["nu_v"]))
    st.set_state(g["eta"], g["qx"], g["qy"], g["ux"], g["uy"], g["T0"])
    for i in range(2):
        st.step(1)
        s = st.get_state()
        for n in ["ux", "uy", "T", "eta", "qx", "qy"]:
            assert rel(s[n], g[f"s{i}_{n}"]) <= 1e-11, (i, n)


def test_100_steps_c2_parity(pdg):
    """Config-2-like barotropic run, 100 internal steps (m = 20): <= 1e-9 vs the oracle."""
    L, dt, msub, kv, nu_v = 4, 40.0, 20, 1e-3, 1e-4
    m, om, p, s0 = _setup(pdg, nx=6, ny=4, L=L, baroclinic=False)
    st = pdg.stepper.ImexStepper(m, L, p, dt, msub, kv, nu_v)
    st.set_state(**s0)
    st.step(100)
    st.check()
    g = st.get_state()
    o = _oracle_run(om, L, p, s0, 100, dt, msub, kv, nu_v)
    for k, ref in [("ux", o.ux), ("uy", o.uy), ("T", o.T), ("eta", o.s2d.eta), ("qx", o.s2d.qx)]:
        assert rel(g[k], ref) <= 1e-9, k


def test_tracer_constancy(pdg):
    """SPEC acceptance 4: T = const stays const under the coupled moving-mesh step."""
    L = 5
    m, om, p, s0 = _setup(pdg, L=L, baroclinic=False)
    st = pdg.stepper.ImexStepper(m, L, p, 40.0, 10, 1e-3, 1e-4)
    st.set_state(**s0)
    st.step(20)
    st.check()
    T = st.get_state()["T"]
    assert np.abs(T - 12.5).max() <= 1e-10 * 12.5


def test_rest_state_fixed_point(pdg):
    L = 4
    m, om, p, s0 = _setup(pdg, L=L, baroclinic=False)
    z2, z3 = np.zeros_like(s0["eta"]), np.zeros_like(s0["ux"])
    st = pdg.stepper.ImexStepper(m, L, pdg.PhysParams(), 40.0, 10, 1e-3, 1e-4)
    st.set_state(z2, z2, z2, z3, z3, np.full_like(z3, 10.0))
    st.step(10)
    g = st.get_state()
    assert max(np.abs(g["eta"]).max(), np.abs(g["ux"]).max(), np.abs(g["qx"]).max()) <= 1e-12


def test_100_steps_baroclinic_parity(pdg):
    """Lock-exchange-like baroclinic run (density front, wind, drag), 100 internal steps: <= 1e-9."""
    L, dt, msub, kv, nu_v = 5, 20.0, 6, 1e-4, 1e-5
    m, om, p, s0 = _setup(pdg, nx=8, ny=5, L=L, baroclinic=True)
    st = pdg.stepper.ImexStepper(m, L, p, dt, msub, kv, nu_v)
    st.set_state(**s0)
    st.step(100)
    st.check()
    g = st.get_state()
    o = _oracle_run(om, L, p, s0, 100, dt, msub, kv, nu_v)
    for k, ref in [("ux", o.ux), ("uy", o.uy), ("T", o.T), ("eta", o.s2d.eta), ("qx", o.s2d.qx), ("qy", o.s2d.qy)]:
        assert rel(g[k], ref) <= 1e-9, (k, rel(g[k], ref))


def test_device_diagnostics_vs_reference(pdg, golden):
    """ImexStepper.diagnostics(): diagnostics_2d + budget_3d of the resident state in one fused device
    reduction, against the reference's values on the same state (tests/golden/diag.npz)."""
    g = golden("diag")
    lx, ly, L = float(g["lx"]), float(g["ly"]), int(g["L"])

    def bed(x, y):
        return -20.0 + 5.0 * np.sin(np.pi * x / lx) * np.cos(2.0 * np.pi * y / ly)
    m = pdg.mesh.hilbert_reorder(pdg.mesh.generate_basin_mesh(int(g["nx"]), int(g["ny"]), lx, ly, bed))
    st = pdg.stepper.ImexStepper(m, L, pdg.PhysParams(f=1e-4, alpha=0.2, t_ref=12.5), 40.0, 4, 1e-3, 1e-4)
    st.set_state(g["eta"], g["qx"], g["qy"], g["ux"], g["uy"], g["T"])
    d = st.diagnostics()
    ref = dict(zip(g["keys"].tolist(), g["values"].tolist()))
    for k, v in ref.items():
        tol = 0.0 if k.endswith(("_min", "_max")) else 1e-12
        assert abs(d[k] - v) <= tol * max(abs(v), 1.0), (k, d[k], v)
    assert st.diagnostics() == d                      # deterministic reduction


def test_host_pinned_state_io(pdg):
    """set_state from pinned host tensors and get_state(out=pinned buffers) (the e2e path) agree
    bitwise with the numpy path."""
    import torch
    L = 4
    m, om, p, s0 = _setup(pdg, L=L)
    st = pdg.stepper.ImexStepper(m, L, p, 40.0, 4, 1e-3, 1e-4)
    st.set_state(**s0)
    st.step(1)
    ref = st.get_state()
    pin = {k: torch.as_tensor(v).pin_memory() for k, v in s0.items()}
    st2 = pdg.stepper.ImexStepper(m, L, p, 40.0, 4, 1e-3, 1e-4)
    st2.set_state(pin["eta"], pin["qx"], pin["qy"], pin["ux"], pin["uy"], pin["T"])
    st2.step(1)
    out = {k: torch.empty_like(v).pin_memory() for k, v in pin.items()}
    st2.get_state(numpy=False, out=out)
    torch.cuda.synchronize()
    for k in ("eta", "qx", "qy", "ux", "uy", "T"):
        assert np.array_equal(out[k].numpy(), ref[k]), k
    # round trip through the same buffers (uploads wait for each field's download), as the e2e bench
    st3 = pdg.stepper.ImexStepper(m, L, p, 40.0, 4, 1e-3, 1e-4)
    st3.set_state(pin["eta"], pin["qx"], pin["qy"], pin["ux"], pin["uy"], pin["T"])
    for _ in range(2):
        st3.step(1)
        st3.get_state(numpy=False, out=pin)
        st3.set_state(pin["eta"], pin["qx"], pin["qy"], pin["ux"], pin["uy"], pin["T"])
    st3.wait_io()
    torch.cuda.synchronize()
    ref2 = pdg.stepper.ImexStepper(m, L, p, 40.0, 4, 1e-3, 1e-4)
    ref2.set_state(**s0)
    ref2.step(2)
    g2 = ref2.get_state()
    for k in ("eta", "ux", "T"):
        assert np.array_equal(pin[k].numpy(), g2[k]), k


def test_diagnostics_csv(pdg, tmp_path):
    """SPEC.md:325 diagnostics CSV and SPEC.md:540 per-step budget CSV (one row per IMEX stage)."""
    L = 4
    m, om, p, s0 = _setup(pdg, L=L)
    st = pdg.stepper.ImexStepper(m, L, p, 40.0, 4, 1e-3, 1e-4)
    st.set_state(**s0)
    for _ in range(3):
        st.step(1)
        st.log_csv(tmp_path / "diag.csv", tmp_path / "budget.csv")
    d = (tmp_path / "diag.csv").read_text().splitlines()
    b = (tmp_path / "budget.csv").read_text().splitlines()
    assert d[0] == "t,total_volume,total_energy,eta_min,eta_max" and len(d) == 4
    assert b[0] == "t,stage,volume,momentum_x,momentum_y,tracer_mass,tracer_min,tracer_max" and len(b) == 7
    rows = [list(map(float, r.split(","))) for r in b[1:]]
    assert [r[1] for r in rows] == [1, 2, 1, 2, 1, 2]
    assert rows[0][0] == 20.0 and rows[1][0] == 40.0            # stage 1 at the midpoint, stage 2 at t
    vols = [float(r.split(",")[1]) for r in d[1:]]
    assert max(vols) - min(vols) <= 1e-12 * abs(vols[0])         # closed basin: volume conserved


def test_nvtx_ranges_do_not_change_the_step(pdg):
    """With NVTX ranges around every library launch (ImexStepper.nvtx / PDG_NVTX=1) the step is
    unchanged (the markers are host-side annotations for nsys / ncu --nvtx)."""
    m, om, p, s0 = _setup(pdg, nx=6, ny=4, L=4)
    out = []
    for nvtx in (False, True):
        st = pdg.stepper.ImexStepper(m, 4, p, 60.0, 4, 1e-3, 1e-4)
        st.nvtx = nvtx
        st.use_graph = False
        st.set_state(**s0)
        st.step(2)
        out.append(st.get_state())
    for k in ("eta", "ux", "T"):
        assert np.array_equal(out[0][k], out[1][k])

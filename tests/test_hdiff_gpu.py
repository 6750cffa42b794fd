"""Explicit horizontal viscosity / diffusion (internal3d.py:549-692) on the GPU (csrc/hdiff.cu).

The reference raises at internal3d.py:665 / :676; the target is the PATCHED
oracle: the reference function with those two broadcasts fixed (oracle/refops.py), whose outputs are
tests/golden/hdiff.npz (scripts/make_golden_hdiff.py).  Per-RHS bar 1e-12 (north_star), steps 1e-9
after 100 steps, partitions bitwise.
"""
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import record
from oracle import ext2d as OE
from oracle import geom as OG
from oracle import stepper as OS

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.fixture(scope="module")
def pdg():
    import paper_2605_16082_b200 as p
    return p


@pytest.fixture(scope="module")
def case(pdg, golden):
    g = golden("hdiff")
    lx, ly = float(g["lx"]), float(g["ly"])

    def bed(x, y):
        return -20.0 + 5.0 * np.sin(np.pi * x / lx) * np.cos(2.0 * np.pi * y / ly)
    m = pdg.mesh.hilbert_reorder(pdg.mesh.generate_basin_mesh(int(g["nx"]), int(g["ny"]), lx, ly, bed))
    om = OG.hilbert_reorder(OG.basin_mesh(int(g["nx"]), int(g["ny"]), lx, ly, bed))
    return g, m, om


def _params(pdg, g, **kw):
    return pdg.PhysParams(f=1e-4, cd=2.5e-3, alpha=0.2, t_ref=12.5, kappa_h=float(g["kappa_h"]),
                          kappa_v=float(g["kappa_v"]), nu_h=float(g["nu_h"]), nu_v=float(g["nu_v"]), **kw)


def test_horizontal_rhs_with_viscosity(pdg, case):
    g, m, _ = case
    grid = pdg.mesh.extrude(m, pdg.mesh.LayerPolicy(count=int(g["L"])), g["eta"])
    p = _params(pdg, g)
    M = pdg.internal3d.prism_mass(grid)
    Fh = pdg.internal3d.horizontal_rhs(grid, g["ux"], g["uy"], g["q"], g["fac"], g["r"], M, p)
    Ft = pdg.internal3d.tracer_horizontal_rhs(grid, g["T"], g["q"], g["fac"], p)
    assert record("hdiff::Fh", rel(Fh, g["Fh"])) <= 1e-12
    assert record("hdiff::Ft", rel(Ft, g["Ft"])) <= 1e-12
    Fe = pdg.internal3d.horizontal_rhs(grid, g["ux"], g["uy"], g["q"], g["fac"], g["r"], M, p, els=g["els"])
    Te = pdg.internal3d.tracer_horizontal_rhs(grid, g["T"], g["q"], g["fac"], p, els=g["els"])
    assert rel(Fe, g["Fh_els"]) <= 1e-12
    assert rel(Te, g["Ft_els"]) <= 1e-12


def test_diffusion_term_alone(pdg, case):
    """pdg_horizontal_diffusion through the C ABI: the bare D(u), D(T) and their column sums."""
    import torch
    from paper_2605_16082_b200 import _lib
    from paper_2605_16082_b200.device import c3_in, device_mesh, p6_in, ptr, stream_ptr
    g, m, _ = case
    L = int(g["L"])
    dm = device_mesh(m, L)
    nt, dev = m.nt, dm.device
    eta = c3_in(torch.as_tensor(g["eta"], device=dev), dev)
    u = torch.stack([p6_in(torch.as_tensor(g["ux"], device=dev), nt, L),
                     p6_in(torch.as_tensor(g["uy"], device=dev), nt, L)]).contiguous()
    T = p6_in(torch.as_tensor(g["T"], device=dev), nt, L).contiguous()
    lb = _lib.lib()
    for f, nc, kh, ref in ((u, 2, float(g["kappa_h"]), g["D_u"]), (T, 1, float(g["nu_h"]), g["D_T"][..., None])):
        out = torch.zeros(nc, 6, L, nt, dtype=torch.float64, device=dev)
        _lib.check(lb.pdg_horizontal_diffusion(dm.h, ptr(eta), ptr(f), nc, kh, int(nc == 2), 1.0, 0, None, 0,
                                               ptr(out), stream_ptr()), "hdiff")
        got = out.permute(3, 2, 1, 0).cpu().numpy()                     # (nt, L, 6, nc)
        assert record(f"hdiff::D{nc}", rel(got, ref)) <= 1e-12
        cs = torch.zeros(nc, 3, nt, dtype=torch.float64, device=dev)
        _lib.check(lb.pdg_horizontal_diffusion(dm.h, ptr(eta), ptr(f), nc, kh, int(nc == 2), 2.0, 1, None, 0,
                                               ptr(cs), stream_ptr()), "hdiff colsum")
        ref_cs = 2.0 * (ref[:, :, 0:3].sum(1) + ref[:, :, 3:6].sum(1))    # column_sum (internal3d.py:184-187)
        assert rel(cs.permute(2, 1, 0).cpu().numpy(), ref_cs) <= 1e-12
    dm.raise_errors()


def test_step_golden_patched_reference(pdg, case):
    """Two IMEX steps with kappa_h, nu_h != 0 against the orchestrator over the patched reference."""
    g, m, _ = case
    p = _params(pdg, g, tau_x=0.05, tau_y=-0.02)
    st = pdg.stepper.ImexStepper(m, int(g["L"]), p, float(g["dt"]), int(g["m"]), float(g["kv"]),
                                 float(g["nu_v_step"]))
    st.set_state(g["eta"], g["qx"], g["qy"], g["ux"], g["uy"], g["T0"])
    for i in range(2):
        st.step(1)
        st.check()
        s = st.get_state()
        for n in ["ux", "uy", "T", "eta", "qx", "qy"]:
            assert record(f"hdiff::step{i}", rel(s[n], g[f"s{i}_{n}"])) <= 1e-11, (i, n)


@pytest.mark.parametrize("graph", [False, True])
def test_100_steps_vs_oracle(pdg, case, graph):
    """100 steps with horizontal viscosity and diffusion on: <= 1e-9 (north_star)."""
    g, m, om = case
    L, dt, msub, kv, nu_v = int(g["L"]), 40.0, 4, 1e-3, 1e-4
    p = _params(pdg, g, tau_x=0.05, tau_y=-0.02)
    s0 = dict(eta=g["eta"], qx=g["qx"], qy=g["qy"], ux=g["ux"], uy=g["uy"], T=g["T0"])
    st = pdg.stepper.ImexStepper(m, L, p, dt, msub, kv, nu_v)
    st.use_graph = graph
    st.set_state(**s0)
    n = 100 if graph else 10
    st.step(n)
    st.check()
    s = st.get_state()
    o = SimpleNamespace(grid=OG.extrude(om, L, s0["eta"]), ux=s0["ux"], uy=s0["uy"], T=s0["T"],
                        s2d=OE.S2(s0["eta"].copy(), s0["qx"], s0["qy"], 0.0))
    for _ in range(n):
        o = OS.imex_step(o, p, dt, msub, kv, nu_v)
    for k, ref in [("ux", o.ux), ("uy", o.uy), ("T", o.T), ("eta", o.s2d.eta), ("qx", o.s2d.qx), ("qy", o.s2d.qy)]:
        assert record(f"hdiff::{n}steps", rel(s[k], ref)) <= 1e-9, k


@pytest.mark.parametrize("P", [2, 3])
def test_partition_invariance_with_diffusion(pdg, P):
    from paper_2605_16082_b200.partition import PartitionedRun
    from paper_2605_16082_b200.scenarios import make_case
    c = make_case("c4", scale=0.02, L=5)
    p = c.params.__class__(**{**c.params.__dict__, "kappa_h": 30.0, "nu_h": 10.0})
    ref = pdg.stepper.ImexStepper(c.mesh, c.L, p, c.dt, c.m, c.kv, c.nu_v)
    ref.use_graph = False
    ref.set_state(**c.state)
    ref.step(2)
    ref.check()
    g = ref.get_state()
    run = PartitionedRun(c.mesh, c.L, p, c.dt, c.m, c.kv, c.nu_v, P)
    run.set_state(**c.state)
    run.step(2)
    run.check()
    s = run.get_state()
    for k in ("eta", "qx", "qy", "ux", "uy", "T"):
        assert np.array_equal(s[k], g[k]), (P, k, float(np.abs(s[k] - g[k]).max()))

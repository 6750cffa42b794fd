"""The CPU oracle against golden vectors produced by the real reference (scripts/make_golden.py)."""
import numpy as np
import pytest

from oracle import colsolve, ext2d, geom, int3d, stepper
from paper_2605_16082_b200.params import PhysParams

P = PhysParams(f=1e-4, cd=2.5e-3, alpha=0.2, t_ref=12.5)


def same(a, b, tol=0.0):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    if tol == 0.0:
        assert np.array_equal(a, b), float(np.abs(a - b).max())
    else:
        assert np.abs(a - b).max() <= tol * max(np.abs(b).max(), 1e-300)


@pytest.fixture(scope="module")
def mesh(golden):
    g = golden("mesh")
    raw = geom.make_mesh(g["vx"], g["vy"], g["vb"], g["raw_tri"])
    return geom.hilbert_reorder(raw), raw, g


def test_mesh_bitwise(mesh):
    m, raw, g = mesh
    same(raw.nbr, g["raw_nbr"]); same(raw.nbrk, g["raw_nbrk"])
    for k in ["tri", "j2d", "dphx", "dphy", "elen", "enx", "eny", "nbr", "nbrk", "btag", "hilbert_perm", "b"]:
        same(getattr(m, k), g[k])


def test_ext2d(mesh, golden):
    m = mesh[0]
    g = golden("ext2d")
    st = ext2d.S2(g["eta"], g["qx"], g["qy"])
    same(ext2d.free_surface_residual(st, m, P, source=g["source"]), g["res_eta"])
    same(ext2d.momentum_residual(st, m, P, f3d2d=g["f3d2d"], patm=g["patm"]), g["res_q"])
    d = ext2d.tendencies(st, m, P, f3d2d=g["f3d2d"], source=g["source"], patm=g["patm"])
    same(d[0], g["d_eta"]); same(d[1], g["d_qx"]); same(d[2], g["d_qy"])
    d = ext2d.tendencies(st, m, P, els=g["els"], f3d2d=g["f3d2d"])
    same(d[0], g["d_els_eta"]); same(d[1], g["d_els_qx"]); same(d[2], g["d_els_qy"])
    s, qbx, qby, fx, fy = ext2d.subcycle(st, m, P, 10, 2.0, f3d2d=g["f3d2d"])
    for a, k in [(s.eta, "sub_eta"), (s.qx, "sub_qx"), (s.qy, "sub_qy"), (qbx, "qbar_x"), (qby, "qbar_y"),
                 (fx, "f2d_x"), (fy, "f2d_y")]:
        same(a, g[k])
    mo = geom.OMesh(**vars(m))
    mo.btag = g["open_btag"]
    d = ext2d.tendencies(st, mo, P, eta_bc=lambda t: 0.05 + 1e-3 * t)
    same(d[0], g["open_d_eta"]); same(d[1], g["open_d_qx"]); same(d[2], g["open_d_qy"])


def test_int3d(mesh, golden):
    m = mesh[0]
    g = golden("int3d")
    L = int(g["L"])
    G = geom.extrude(m, L, g["eta"])
    G1 = geom.update_moving_mesh(G, g["eta1"], float(g["dt_mesh"]))
    for k in ["z", "jz", "dzmid", "djz", "dztop", "dzbot"]:
        same(getattr(G, k), g[k])
    same(G1.w_m, g["w_m"])
    same(ext2d.eos(g["T"], P), g["rho"])
    M = int3d.prism_mass(G)
    same(M, g["mass"])
    q = int3d.project_transport(G, g["ux"], g["uy"], mass=M)
    same(q, g["q"])
    same(int3d.lateral_flux_factor(G, q, P), g["fac"])
    same(int3d.compute_r(G, g["rho"], P), g["r"])
    same(int3d.compute_w(G, q, g["ux"], g["uy"], P, g["fac"]), g["w"])
    same(int3d.consistent_transport(G, q, g["qbx"], g["qby"]), g["qb"])
    same(int3d.compute_wtilde(G, g["qb"], g["facb"]), g["wt"])
    same(int3d.horizontal_rhs(G, g["ux"], g["uy"], g["qb"], g["facb"], g["r"], M, P), g["Fh"])
    same(int3d.tracer_horizontal_rhs(G, g["T"], g["qb"], g["facb"], P), g["Ft"])
    same(int3d.stress_rhs(G, 0.1 / 1025, -0.05 / 1025, 2.5e-3, g["ux"], g["uy"]), g["stress"])
    A = int3d.assemble_vertical_operator(G, g["wt"], g["w_m"], 0.5, 1e-3)
    same(A.d, g["A_d"]); same(A.u, g["A_u"]); same(A.w, g["A_w"])
    Ai = int3d.build_implicit(int3d.prism_mass(G1), A, 20.0, G)
    same(Ai.d, g["Ai_d"]); same(Ai.u, g["Ai_u"]); same(Ai.w, g["Ai_w"])
    same(colsolve.block_thomas(Ai, g["rhs"]), g["xb"])
    same(colsolve.banded_matvec(Ai, g["rhs"]), g["yb"])
    same(int3d.mass_solve(M, g["rhs"].reshape(-1, 6, 2), G), g["ms"])
    same(int3d.compute_r(G, g["rho"], P, els=g["els"]), g["r_els"])
    same(int3d.horizontal_rhs(G, g["ux"], g["uy"], q, g["fac"], g["r"], M, P, els=g["els"]), g["Fh_els"])


def test_columns(golden):
    g = golden("columns")
    same(colsolve.sweep_r(g["rhs"], g["j2d"]), g["r_out"])
    same(colsolve.sweep_w(g["rhs"], g["j2d"]), g["w_out"])
    same(ext2d.mh_apply(g["rhs"][:, 0, 0:3], g["j2d"]), g["mh"])
    same(ext2d.mh_inv_apply(g["rhs"][:, 0, 0:3], g["j2d"]), g["mhinv"])
    same(colsolve.thomas(g["lower"], g["diag"], g["upper"], g["trhs"]), g["tri_x"])
    mh = 1.7 * np.array([[2.0, 1, 1], [1, 2, 1], [1, 1, 2]]) / 24.0
    same(colsolve.dense_sweep_matrix("r", 3, mh), g["dense_r"])
    same(colsolve.dense_sweep_matrix("w", 3, mh), g["dense_w"])


def test_step(mesh, golden):
    from types import SimpleNamespace
    m = mesh[0]
    g = golden("step")
    L = int(g["L"])
    p = PhysParams(f=1e-4, cd=2.5e-3, alpha=0.2, t_ref=12.5, tau_x=0.05, tau_y=-0.02)
    s = SimpleNamespace(grid=geom.extrude(m, L, g["eta"]), ux=g["ux"], uy=g["uy"], T=g["T0"],
                        s2d=ext2d.S2(g["eta"].copy(), g["qx"], g["qy"], 0.0))
    for i in range(2):
        s = stepper.imex_step(s, p, float(g["dt"]), int(g["m"]), float(g["kv"]), float(g["nu_v"]))
        for n, a in [("ux", s.ux), ("uy", s.uy), ("T", s.T), ("eta", s.s2d.eta), ("qx", s.s2d.qx), ("qy", s.s2d.qy)]:
            same(a, g[f"s{i}_{n}"])


def test_diagnostics(golden):
    """diagnostics_2d / budget_3d restatements vs the reference (scripts/make_golden_diag.py)."""
    g = golden("diag")
    lx, ly = float(g["lx"]), float(g["ly"])

    def bed(x, y):
        return -20.0 + 5.0 * np.sin(np.pi * x / lx) * np.cos(2.0 * np.pi * y / ly)
    m = geom.hilbert_reorder(geom.basin_mesh(int(g["nx"]), int(g["ny"]), lx, ly, bed))
    ref = dict(zip(g["keys"].tolist(), g["values"].tolist()))
    d2 = ext2d.diagnostics_2d(g["eta"], g["qx"], g["qy"], m, float(g["g"]))
    grid = geom.extrude(m, int(g["L"]), g["eta"])
    b3 = int3d.budget_3d(grid, int3d.prism_mass(grid), g["ux"], g["uy"], g["T"])
    for k, v in {**d2, **b3}.items():
        assert abs(v - ref[k]) <= 1e-13 * max(abs(ref[k]), 1.0), (k, v, ref[k])


@pytest.mark.parametrize("name", ["c2", "c3w"])
def test_oracle_first_step_of_config_fixtures(golden, name):
    """The oracle orchestrator + oracle functions reproduce the reference's first step of the
    stated-size config fixtures (tests/golden/cfg_*.npz)."""
    import os
    import sys
    from types import SimpleNamespace
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import config_states as CS
    from oracle import ext2d as OE
    from oracle import geom as OG
    from oracle import stepper as OS
    from paper_2605_16082_b200.params import PhysParams
    cfg = CS.C2 if name == "c2" else CS.C3W
    g = golden(f"cfg_{name}")
    om = OG.hilbert_reorder(OG.basin_mesh(cfg["nx"], cfg["ny"], cfg["lx"], cfg["ly"], CS.flat_bed))
    L = cfg["L"]
    s0 = CS.c2_state(om, L) if name == "c2" else CS.c3_state(om, L, cfg["lx"])
    s = SimpleNamespace(grid=OG.extrude(om, L, s0["eta"]), ux=s0["ux"], uy=s0["uy"], T=s0["T"],
                        s2d=OE.S2(s0["eta"].copy(), s0["qx"], s0["qy"], 0.0))
    s = OS.imex_step(s, PhysParams(**cfg["params"]), cfg["dt"], cfg["m"], cfg["kv"], cfg["nu_v"])
    for n, a in (("ux", s.ux), ("uy", s.uy), ("T", s.T), ("eta", s.s2d.eta), ("qx", s.s2d.qx), ("qy", s.s2d.qy)):
        ref = g[f"s1_{n}"]
        assert np.abs(a - ref).max() <= 1e-13 * max(np.abs(ref).max(), 1e-300), n


def _hdiff_case(golden):
    g = golden("hdiff")
    lx, ly = float(g["lx"]), float(g["ly"])

    def bed(x, y):
        return -20.0 + 5.0 * np.sin(np.pi * x / lx) * np.cos(2.0 * np.pi * y / ly)
    m = geom.hilbert_reorder(geom.basin_mesh(int(g["nx"]), int(g["ny"]), lx, ly, bed))
    return g, m


def test_horizontal_diffusion_patched_oracle(golden):
    """Explicit horizontal viscosity/diffusion (internal3d.py:549-692) against the PATCHED reference
    (scripts/make_golden_hdiff.py; the reference itself raises at :665).  The oracle is a closed-form
    restatement, so the bar is 1e-14 relative, not bitwise."""
    g, m = _hdiff_case(golden)
    G = geom.extrude(m, int(g["L"]), g["eta"])
    kh, kv, nh, nv = (float(g[k]) for k in ("kappa_h", "kappa_v", "nu_h", "nu_v"))
    U = np.stack([g["ux"], g["uy"]], -1)
    same(int3d.horizontal_diffusion(G, U, kh, kv, None, True), g["D_u"], 1e-14)
    same(int3d.horizontal_diffusion(G, g["T"][..., None], nh, nv, None, False)[..., 0], g["D_T"], 1e-14)
    p = PhysParams(f=1e-4, cd=2.5e-3, alpha=0.2, t_ref=12.5, kappa_h=kh, kappa_v=kv, nu_h=nh, nu_v=nv)
    M = int3d.prism_mass(G)
    same(int3d.horizontal_rhs(G, g["ux"], g["uy"], g["q"], g["fac"], g["r"], M, p), g["Fh"], 1e-14)
    same(int3d.tracer_horizontal_rhs(G, g["T"], g["q"], g["fac"], p), g["Ft"], 1e-14)
    same(int3d.horizontal_rhs(G, g["ux"], g["uy"], g["q"], g["fac"], g["r"], M, p, els=g["els"]), g["Fh_els"], 1e-14)
    same(int3d.tracer_horizontal_rhs(G, g["T"], g["q"], g["fac"], p, els=g["els"]), g["Ft_els"], 1e-14)


def test_step_with_horizontal_diffusion(golden):
    """Two IMEX steps with kappa_h, nu_h != 0: oracle vs the orchestrator over the patched reference."""
    from types import SimpleNamespace
    g, m = _hdiff_case(golden)
    p = PhysParams(f=1e-4, cd=2.5e-3, alpha=0.2, t_ref=12.5, tau_x=0.05, tau_y=-0.02, kappa_h=float(g["kappa_h"]),
                   kappa_v=float(g["kappa_v"]), nu_h=float(g["nu_h"]), nu_v=float(g["nu_v"]))
    s = SimpleNamespace(grid=geom.extrude(m, int(g["L"]), g["eta"]), ux=g["ux"], uy=g["uy"], T=g["T0"],
                        s2d=ext2d.S2(g["eta"].copy(), g["qx"], g["qy"], 0.0))
    for i in range(2):
        s = stepper.imex_step(s, p, float(g["dt"]), int(g["m"]), float(g["kv"]), float(g["nu_v_step"]))
        for n, a in [("ux", s.ux), ("uy", s.uy), ("T", s.T), ("eta", s.s2d.eta), ("qx", s.s2d.qx), ("qy", s.s2d.qy)]:
            same(a, g[f"s{i}_{n}"], 1e-13)

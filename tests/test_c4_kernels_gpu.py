"""Per-RHS parity of the fused STEPPER kernels at the full C4 size (1 M tri x 50 layers, m = 20).

north_star gate: relative L-inf <= 1e-12 per RHS evaluation.  The kernels run over the whole
1,000,000-column mesh on the GPU exactly as the stepper launches them (tile-staged r / w~ /
F3D->2D, the fused stage RHS, the block-Thomas and explicit vertical stages, the 2D sub-cycle);
the oracle evaluates the same operators on a patch around ~1,000 sampled columns (tests/patch.py:
the reference assemblies are element-subset invariant, internal3d.py:695-751, 505-541,
columns.py:292-348), and the sampled rows are compared.  The sample includes the first / last
columns and 128-column tile edges, so the L = 50 rings, the tile maps and the 32-bit plane
indices of the fused kernels are all checked numerically.
"""
from types import SimpleNamespace

import numpy as np
import pytest

from oracle import colsolve as OC
from oracle import ext2d as OE
from oracle import geom as OG
from oracle import int3d as OI
from oracle import stepper as OS
from config_states import sample_columns
from patch import build_patch, rows_c3, rows_p6, rows_pv

pytestmark = pytest.mark.gpu

TOL = 1e-12
NSAMPLE = 1024


def rel(a, b):
    """normwise relative L-inf error, recorded per test (conftest.record)."""
    import os
    from conftest import record
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    e = float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))
    return record(os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0], e)


@pytest.fixture(scope="module")
def c4():
    import torch

    from paper_2605_16082_b200.device import DeviceMesh
    from paper_2605_16082_b200.params import PenaltyParams
    from paper_2605_16082_b200.scenarios import _c4_eta, make_case
    case = make_case("c4", with_state=False)
    mesh, L, nt = case.mesh, case.L, case.mesh.nt
    dev = torch.device("cuda", torch.cuda.current_device())
    dm = DeviceMesh(mesh).set_layers(L)
    gen = torch.Generator(device=dev).manual_seed(2024)

    def rn(*shape, scale=1.0):
        return scale * torch.randn(*shape, generator=gen, device=dev, dtype=torch.float64)
    e = torch.as_tensor(_c4_eta(mesh.x + case.x0, case.lx).T.copy(), device=dev)
    f = SimpleNamespace(
        eta0=e + rn(3, nt, scale=0.01), eta_u=None, eta1=None,
        u=rn(2, 6, L, nt, scale=0.05), T=12.0 + rn(6, L, nt, scale=0.5), qbar=rn(2, 3, nt, scale=0.3),
        f2d=rn(2, 3, nt, scale=1e-4))
    f.eta_u = f.eta0 + rn(3, nt, scale=0.005)
    f.eta1 = f.eta0 + rn(3, nt, scale=0.005)
    f.u0 = f.u + rn(2, 6, L, nt, scale=0.01)
    f.T0 = f.T + rn(6, L, nt, scale=0.01)
    cols = sample_columns(nt, NSAMPLE)
    ids1, om1 = build_patch(mesh, cols, 1)
    host = SimpleNamespace(ns=cols.size, ids=ids1, om=om1)
    for k in ("eta0", "eta_u", "eta1"):
        setattr(host, k, rows_c3(getattr(f, k), ids1))
    host.u = rows_pv(f.u, ids1)
    host.u0 = rows_pv(f.u0, ids1)
    host.T = rows_p6(f.T, ids1)
    host.T0 = rows_p6(f.T0, ids1)
    host.qbar = rows_c3(f.qbar, ids1)
    host.f2d = rows_c3(f.f2d, ids1)
    host.Gu = OG.extrude(om1, L, host.eta_u)
    host.G0 = OG.extrude(om1, L, host.eta0)
    host.G1 = OG.update_moving_mesh(host.G0, host.eta1, case.dt)
    yield SimpleNamespace(case=case, mesh=mesh, L=L, nt=nt, dev=dev, dm=dm, f=f, h=host, pen=PenaltyParams(),
                          p=case.params, z=lambda *s: torch.zeros(s, dtype=torch.float64, device=dev))
    del dm


def _lib():
    from paper_2605_16082_b200 import _lib as lb
    return lb.lib(), lb.check


def _ptr(t):
    from paper_2605_16082_b200.device import ptr
    return ptr(t)


def _s():
    from paper_2605_16082_b200.device import stream_ptr
    return stream_ptr()


def _rows(h, a, L):
    """the sampled columns' rows of a patch-ordered prism array."""
    return a[:h.ns * L]


@pytest.fixture(scope="module")
def r_q(c4):
    """GPU r (EOS inline, tile-staged k_compute_r_t) and q (projection + column sum + depth)."""
    lb, check = _lib()
    c, f = c4, c4.f
    r, q = c.z(2, 6, c.L, c.nt), c.z(2, 6, c.L, c.nt)
    qsum, htot = c.z(2, 3, c.nt), c.z(3, c.nt)
    p = c.p
    check(lb.pdg_compute_r(c.dm.h, _ptr(f.eta_u), _ptr(f.T), 1, p.alpha, p.t_ref, p.g, None, 0, _ptr(r), _s()), "r")
    check(lb.pdg_project_transport(c.dm.h, _ptr(f.eta_u), _ptr(f.u[0]), _ptr(f.u[1]), None, None, 0, _ptr(q),
                                   _ptr(qsum), _ptr(htot), _s()), "project")
    c.dm.raise_errors("r/q")
    return SimpleNamespace(r=r, q=q, qsum=qsum, htot=htot)


def test_c4_compute_r_tiled(c4, r_q):
    h, p, L = c4.h, c4.p, c4.L
    ref = OI.compute_r(h.Gu, OE.eos(h.T, p), p)
    assert rel(_rows(h, rows_pv(r_q.r, h.ids), L), _rows(h, ref, L)) <= TOL


def test_c4_project_transport(c4, r_q):
    h, L = c4.h, c4.L
    q = OI.project_transport(h.Gu, h.u[..., 0], h.u[..., 1])
    assert rel(_rows(h, rows_pv(r_q.q, h.ids), L), _rows(h, q, L)) <= TOL
    qs = OI.column_sum(q, h.Gu)
    assert rel(rows_c3(r_q.qsum, h.ids)[:h.ns], qs[:h.ns]) <= TOL
    assert rel(rows_c3(r_q.htot, h.ids)[:h.ns], OG.total_thickness(h.Gu)[:h.ns]) <= TOL


def test_c4_f3d2d(c4, r_q):
    """F3D->2D = column sum of F_h(u, q, fac(q)) + stresses (k_hrhs_t<2, PRED>, tile-staged)."""
    lb, check = _lib()
    h, p, L, f = c4.h, c4.p, c4.L, c4.f
    out = c4.z(2, 3, c4.nt)
    tsx, tsy = p.wind(0.0)
    check(lb.pdg_step_f3d2d(c4.dm.h, _ptr(f.eta_u), _ptr(f.u), _ptr(r_q.q), _ptr(r_q.r), p.g, p.f, p.rho0, tsx, tsy,
                            p.cd, _ptr(out), _s()), "f3d2d")
    q, r = rows_pv(r_q.q, h.ids), rows_pv(r_q.r, h.ids)       # the kernel's own inputs
    Mu = OI.prism_mass(h.Gu)
    fac = OI.lateral_flux_factor(h.Gu, q, p)
    Fh = OI.horizontal_rhs(h.Gu, h.u[..., 0], h.u[..., 1], q, fac, r, Mu, p)
    st = OI.stress_rhs(h.Gu, tsx, tsy, p.cd, h.u[..., 0], h.u[..., 1])
    ref = OI.column_sum(Fh + st, h.Gu)
    assert rel(rows_c3(out, h.ids)[:h.ns], ref[:h.ns]) <= TOL


@pytest.fixture(scope="module")
def mis_wt(c4, r_q):
    lb, check = _lib()
    f = c4.f
    mis, wt = c4.z(2, 3, c4.nt), c4.z(6, c4.L, c4.nt)
    check(lb.pdg_mismatch(c4.dm.h, _ptr(f.qbar), _ptr(r_q.qsum), _ptr(r_q.htot), _ptr(mis), _s()), "mismatch")
    check(lb.pdg_compute_wtilde(c4.dm.h, _ptr(f.eta_u), _ptr(r_q.q), None, _ptr(mis), c4.p.g, None, 0, _ptr(wt),
                                _s()), "wtilde")
    return SimpleNamespace(mis=mis, wt=wt)


def _qbar(Gu, q, mis, L):
    """q~ = q + Jz mis (consistent_transport, internal3d.py:190-208, given the 2D mismatch)."""
    qv, jz = q.reshape(-1, L, 6, 2), Gu.jz.reshape(-1, L, 3)
    out = np.empty_like(qv)
    for lev in range(2):
        s = slice(3 * lev, 3 * lev + 3)
        out[:, :, s] = qv[:, :, s] + jz[..., None] * mis[:, None]
    return out.reshape(q.shape)


def test_c4_mismatch(c4, r_q, mis_wt):
    h = c4.h
    ref = (h.qbar - rows_c3(r_q.qsum, h.ids)) / rows_c3(r_q.htot, h.ids)[..., None]
    assert rel(rows_c3(mis_wt.mis, h.ids)[:h.ns], ref[:h.ns]) <= TOL


def test_c4_wtilde_tiled(c4, r_q, mis_wt):
    """w~ with qbar = q + Jz mis and its factor formed on the fly (k_compute_wtilde_t)."""
    h, p, L = c4.h, c4.p, c4.L
    qb = _qbar(h.Gu, rows_pv(r_q.q, h.ids), rows_c3(mis_wt.mis, h.ids), L)
    ref = OI.compute_wtilde(h.Gu, qb, OI.lateral_flux_factor(h.Gu, qb, p))
    assert rel(_rows(h, rows_p6(mis_wt.wt, h.ids), L), _rows(h, ref, L)) <= TOL


@pytest.mark.parametrize("with_w", [False, True], ids=["rhs", "rhs+wtilde"])
@pytest.mark.parametrize("same", [False, True], ids=["stage2", "stage1"])
def test_c4_stage_rhs(c4, r_q, mis_wt, same, with_w):
    """Fused momentum + tracer stage RHS (k_hrhs_s<3, 2>; stage 1: u = u0, T = T0 on G0):
    rhs_u = M0 u0 + dt (F_h(u, q~) + stress + M1 F2D/H1), rhs_T = M0 T0 + dt F_T(T, q~);
    with_w: pdg_step_rhs_ut_w, the stepper's entry, which also forms w~ (compute_wtilde of q~) in
    the same bottom-up layer loop (k_hrhs_s<3, 2, .., WT>)."""
    import torch
    lb, check = _lib()
    h, p, L, f = c4.h, c4.p, c4.L, c4.f
    out_u, out_T = torch.empty_like(f.u), torch.empty_like(f.T)
    w = c4.z(6, L, c4.nt)
    tsx, tsy = p.wind(0.0)
    eta_u, u, T = (f.eta0, f.u0, f.T0) if same else (f.eta_u, f.u, f.T)
    args = (c4.dm.h, _ptr(eta_u), _ptr(f.eta0), _ptr(f.eta1), _ptr(u), _ptr(T), _ptr(f.u0), _ptr(f.T0), _ptr(r_q.q),
            _ptr(mis_wt.mis), _ptr(r_q.r), _ptr(f.f2d), p.g, p.f, p.rho0, tsx, tsy, p.cd, c4.case.dt, _ptr(out_u),
            _ptr(out_T))
    if with_w:
        check(lb.pdg_step_rhs_ut_w(*args, _ptr(w), _s()), "rhs_ut_w")
    else:
        check(lb.pdg_step_rhs_ut(*args, _s()), "rhs_ut")
    c4.dm.raise_errors("rhs_ut")
    Gu, uh, Th = (h.G0, h.u0, h.T0) if same else (h.Gu, h.u, h.T)
    q, r = rows_pv(r_q.q, h.ids), rows_pv(r_q.r, h.ids)          # the kernel's own inputs
    qb = _qbar(Gu, q, rows_c3(mis_wt.mis, h.ids), L)
    facb = OI.lateral_flux_factor(Gu, qb, p)
    Fhb = OI.horizontal_rhs(Gu, uh[..., 0], uh[..., 1], qb, facb, r, OI.prism_mass(Gu), p)
    st = OI.stress_rhs(Gu, tsx, tsy, p.cd, uh[..., 0], uh[..., 1])
    M0, M1 = OI.prism_mass(h.G0), OI.prism_mass(h.G1)
    H1 = h.eta1 - h.om.b
    F = np.repeat(np.stack([h.f2d[..., 0] / H1, h.f2d[..., 1] / H1], -1), L, axis=0)
    F6 = np.concatenate([F, F], axis=1)
    dt = c4.case.dt
    ref_u = OI.mass_apply(M0, h.u0) + dt * (Fhb + st + OI.mass_apply(M1, F6))
    ref_t = OI.mass_apply(M0, h.T0) + dt * OI.tracer_horizontal_rhs(Gu, Th, qb, facb, p)
    assert rel(_rows(h, rows_pv(out_u, h.ids), L), _rows(h, ref_u, L)) <= TOL
    assert rel(_rows(h, rows_p6(out_T, h.ids), L), _rows(h, ref_t, L)) <= TOL
    if with_w:
        ref_w = OI.compute_wtilde(Gu, qb, facb)
        assert rel(_rows(h, rows_p6(w, h.ids), L), _rows(h, ref_w, L)) <= TOL


@pytest.mark.parametrize("implicit", [True, False], ids=["implicit", "explicit"])
@pytest.mark.parametrize("nc", [2, 1], ids=["momentum", "tracer"])
def test_c4_vertical(c4, mis_wt, implicit, nc):
    """Vertical stage in place, as the stepper calls it: implicit (M1 - dt A) x = rhs (split
    block Thomas k_vimpl_fwd + k_vimpl_bwd_r) / explicit x = M1^-1 (rhs + dt A xin) (k_vexpl2)."""
    import torch
    lb, check = _lib()
    h, p, L, f, pe = c4.h, c4.p, c4.L, c4.f, c4.pen
    dt = c4.case.dt
    kh, kv = (p.kappa_h, c4.case.kv) if nc == 2 else (p.nu_h, c4.case.nu_v)
    xin = f.u if nc == 2 else f.T
    g = torch.Generator(device=c4.dev).manual_seed(7 + nc)
    x = torch.randn(xin.shape, generator=g, device=c4.dev, dtype=torch.float64)   # rhs, solved in place
    rhs_h = rows_pv(x, h.ids) if nc == 2 else rows_p6(x, h.ids)
    check(lb.pdg_step_vertical(c4.dm.h, nc, int(implicit), _ptr(f.eta_u), _ptr(f.eta0), _ptr(f.eta1), dt,
                               _ptr(mis_wt.wt), kh, kv, pe.n0, pe.order, dt, _ptr(x), _ptr(xin), _ptr(x), _s()),
          "vertical")
    c4.dm.raise_errors("vertical")
    got = rows_pv(x, h.ids) if nc == 2 else rows_p6(x, h.ids)
    wt = rows_p6(mis_wt.wt, h.ids)
    A = OI.assemble_vertical_operator(h.Gu, wt, h.G1.w_m, kh, kv, n0=pe.n0, order=pe.order)
    M1 = OI.prism_mass(h.G1)
    if implicit:
        ref = OC.block_thomas(OI.build_implicit(M1, A, dt, h.Gu), OS._col(rhs_h, h.Gu)).reshape(rhs_h.shape)
    else:
        xh = rows_pv(xin, h.ids) if nc == 2 else rows_p6(xin, h.ids)
        ax = OC.banded_matvec(A, OS._col(xh, h.Gu)).reshape(rhs_h.shape)
        ref = OI.mass_solve(M1, rhs_h + dt * ax, h.Gu)
    assert rel(_rows(h, got, L), _rows(h, ref, L)) <= TOL


@pytest.mark.parametrize("msub", [1, 2])
def test_c4_subcycle(c4, msub):
    """2D external sub-cycle at C4 (k_rk_stage x 3 m + final): eta, Q, Qbar, F2D on sampled columns;
    the oracle runs on a patch of 3 m rings (one ring per RK stage)."""
    import torch
    lb, check = _lib()
    c, p, f = c4, c4.p, c4.f
    S = torch.stack([f.eta0, 5.0 * f.qbar[0], 5.0 * f.qbar[1]])
    f3 = c.z(2, 3, c.nt).copy_(f.f2d * 1e3)
    qbar, f2d = c.z(2, 3, c.nt), c.z(2, 3, c.nt)
    dt2 = c.case.dt2d
    S0 = S.clone()
    check(lb.pdg_ext2d_subcycle(c.dm.h, _ptr(S), msub, dt2, p.g, p.rho0, _ptr(f3), None, None, None, _ptr(qbar),
                                _ptr(f2d), 1, _s()), "subcycle")
    c.dm.raise_errors("subcycle")
    cols = sample_columns(c.nt, 256, seed=11)
    ids, om = build_patch(c.mesh, cols, 3 * msub)
    n = cols.size
    s0 = OE.S2(*(rows_c3(S0[i], ids) for i in range(3)), 0.0)
    s, qbx, qby, fx, fy = OE.subcycle(s0, om, p, msub, dt2, f3d2d=rows_c3(f3, ids))
    for k, ref in ((0, s.eta), (1, s.qx), (2, s.qy)):
        assert rel(rows_c3(S[k], ids)[:n], ref[:n]) <= TOL, k
    qb, ff = rows_c3(qbar, ids), rows_c3(f2d, ids)
    assert rel(qb[:n, :, 0], qbx[:n]) <= TOL and rel(qb[:n, :, 1], qby[:n]) <= TOL
    assert rel(ff[:n, :, 0], fx[:n]) <= TOL and rel(ff[:n, :, 1], fy[:n]) <= TOL

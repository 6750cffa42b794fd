"""The shared 2-stage IMEX internal step (E2), composed from oracle functions.

Oracle / test infrastructure only.  The reference ships no stepper
(SURVEY.md section 0.2); this is the composition defined in DESIGN.md section 3,
following SPEC.md:511-519, 529-534 and PAPER.md:372-384:

  stage(dt_s, m_s, implicit) starting from (G0, u0, T0, s2d0) with stage values (Gu, u, T):
    rho = eos(T); r = compute_r(Gu, rho); Mu = prism_mass(Gu)
    q = project_transport(Gu, u); fac = lateral_flux_factor(Gu, q)
    Fh = horizontal_rhs(Gu, u, q, fac, r, Mu); st = stress_rhs(Gu, wind, cd, u)
    f3d2d = column_sum(Fh + st)
    ext = subcycle_external(s2d0, m_s, dt_s / m_s, f3d2d)
    G1 = update_moving_mesh(G0, ext.eta, dt_s); M0, M1 = prism_mass(G0), prism_mass(G1)
    qb = consistent_transport(Gu, q, Qbar); facb = lateral_flux_factor(Gu, qb)
    wt = compute_wtilde(Gu, qb, facb); Fhb = horizontal_rhs(Gu, u, qb, facb, r, Mu)
    rhs_u = M0 u0 + dt_s (Fhb + st + M1 (F2D / H1 on all six nodes))
    A = assemble_vertical_operator(Gu, wt, G1.w_m, kappa_h, kv)
    implicit: u1 = solve_banded_column(M1 - dt_s A, rhs_u)
    explicit: u1 = mass_solve(M1, rhs_u + dt_s A u)
    tracer: same with tracer_horizontal_rhs(Gu, T, qb, facb), At(nu_h, nu_v), rhs_T = M0 T0 + dt_s Ft
  step: stage 1 (dt/2, m/2, implicit) from the step start; stage 2 (dt, m, explicit)
        with stage values = stage-1 result.
"""
from types import SimpleNamespace

import numpy as np

from . import ext2d, geom, int3d
from .colsolve import Banded, banded_matvec, block_thomas


def wind(p, t):
    """external2d.py:60-67."""
    tx, ty = p.tau_x, p.tau_y
    if p.tau_x1 is not None and p.wind_t1 > p.wind_t0:
        a = float(np.clip((t - p.wind_t0) / (p.wind_t1 - p.wind_t0), 0.0, 1.0))
        tx = (1.0 - a) * p.tau_x + a * p.tau_x1
        ty = (1.0 - a) * p.tau_y + a * (p.tau_y1 if p.tau_y1 is not None else p.tau_y)
    return tx / p.rho0, ty / p.rho0


def _col(f, grid):
    f = np.asarray(f)
    return f.reshape((grid.mesh.nt, grid.n_layers) + f.shape[1:])


def _oracle_subcycle(s2d, mesh, p, m, dt, f3d2d):
    s, qbx, qby, fx, fy = ext2d.subcycle(s2d, mesh, p, m, dt, f3d2d=f3d2d)
    return SimpleNamespace(state=s, qbar_x=qbx, qbar_y=qby, f2d_x=fx, f2d_y=fy, steps=m)


# the operator set the orchestrator is written against (reference signatures)
ORACLE_OPS = SimpleNamespace(
    eos=ext2d.eos, compute_r=int3d.compute_r, prism_mass=int3d.prism_mass,
    project_transport=int3d.project_transport, lateral_flux_factor=int3d.lateral_flux_factor,
    horizontal_rhs=int3d.horizontal_rhs, stress_rhs=int3d.stress_rhs, column_sum=int3d.column_sum,
    consistent_transport=int3d.consistent_transport, compute_wtilde=int3d.compute_wtilde,
    tracer_horizontal_rhs=int3d.tracer_horizontal_rhs,
    assemble_vertical_operator=int3d.assemble_vertical_operator, build_implicit=int3d.build_implicit,
    mass_apply=int3d.mass_apply, mass_solve=int3d.mass_solve, solve_banded_column=block_thomas,
    apply_banded=banded_matvec, update_moving_mesh=geom.update_moving_mesh, subcycle=_oracle_subcycle)


def stage(ops, st0, Gu, ux, uy, T, p, kv, nu_v, dt_s, m_s, implicit, t_wind):
    G0, mesh = st0.grid, st0.grid.mesh
    rho = ops.eos(T, p)
    r = ops.compute_r(Gu, rho, p)
    Mu = ops.prism_mass(Gu)
    q = ops.project_transport(Gu, ux, uy, mass=Mu)
    fac = ops.lateral_flux_factor(Gu, q, p)
    Fh = ops.horizontal_rhs(Gu, ux, uy, q, fac, r, Mu, p)
    tsx, tsy = wind(p, t_wind)
    st = ops.stress_rhs(Gu, tsx, tsy, p.cd, ux, uy)
    f3d2d = ops.column_sum(Fh + st, Gu)
    ext = ops.subcycle(st0.s2d, mesh, p, m_s, dt_s / m_s, f3d2d)
    G1 = ops.update_moving_mesh(G0, ext.state.eta, dt_s)
    M0, M1 = ops.prism_mass(G0), ops.prism_mass(G1)
    qb = ops.consistent_transport(Gu, q, ext.qbar_x, ext.qbar_y)
    facb = ops.lateral_flux_factor(Gu, qb, p)
    wt = ops.compute_wtilde(Gu, qb, facb)
    Fhb = ops.horizontal_rhs(Gu, ux, uy, qb, facb, r, Mu, p)
    H1 = ext.state.eta - mesh.b
    F = np.repeat(np.stack([ext.f2d_x / H1, ext.f2d_y / H1], -1), G0.n_layers, axis=0)   # (P, 3, 2)
    F6 = np.concatenate([F, F], axis=1)                                                  # (P, 6, 2)
    U0 = np.stack([st0.ux, st0.uy], -1)
    U = np.stack([ux, uy], -1)
    rhs_u = ops.mass_apply(M0, U0) + dt_s * (Fhb + st + ops.mass_apply(M1, F6))
    A = ops.assemble_vertical_operator(Gu, wt, G1.w_m, p.kappa_h, kv)
    Ft = ops.tracer_horizontal_rhs(Gu, T, qb, facb, p)
    At = ops.assemble_vertical_operator(Gu, wt, G1.w_m, p.nu_h, nu_v)
    rhs_t = ops.mass_apply(M0, st0.T) + dt_s * Ft
    if implicit:
        u1 = ops.solve_banded_column(ops.build_implicit(M1, A, dt_s, Gu), _col(rhs_u, Gu)).reshape(-1, 6, 2)
        T1 = ops.solve_banded_column(ops.build_implicit(M1, At, dt_s, Gu), _col(rhs_t, Gu)).reshape(-1, 6)
    else:
        au = ops.apply_banded(A, _col(U, Gu)).reshape(-1, 6, 2)
        u1 = ops.mass_solve(M1, rhs_u + dt_s * au, Gu)
        at = ops.apply_banded(At, _col(T, Gu)).reshape(-1, 6)
        T1 = ops.mass_solve(M1, rhs_t + dt_s * at, Gu)
    return SimpleNamespace(grid=G1, ux=np.ascontiguousarray(u1[..., 0]), uy=np.ascontiguousarray(u1[..., 1]),
                           T=T1, s2d=ext.state,
                           diag=dict(qbar=(ext.qbar_x, ext.qbar_y), f2d=(ext.f2d_x, ext.f2d_y), r=r, q=q, qb=qb,
                                     wt=wt, f3d2d=f3d2d))


def imex_step_ops(ops, st, p, dt, m, kv, nu_v):
    """One internal step: stage 1 (dt/2, m/2, implicit), stage 2 (dt, m, explicit)."""
    if m % 2:
        raise ValueError("m must be even (stage 1 uses m/2 substeps)")
    t0 = st.s2d.t
    h = stage(ops, st, st.grid, st.ux, st.uy, st.T, p, kv, nu_v, 0.5 * dt, m // 2, True, t0)
    return stage(ops, st, h.grid, h.ux, h.uy, h.T, p, kv, nu_v, dt, m, False, t0 + 0.5 * dt)


def imex_step(st, p, dt, m, kv, nu_v):
    return imex_step_ops(ORACLE_OPS, st, p, dt, m, kv, nu_v)

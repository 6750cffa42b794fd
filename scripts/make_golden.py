"""Generate tests/golden/*.npz from the REAL reference package.

Run in the build container only (needs /root/reference):
    python scripts/make_golden.py
The fixtures pin the CPU oracle (oracle/) -- tests/test_oracle_golden.py --
and, through it, the CUDA path.  Each fixture stores its inputs as well as
the reference outputs, so nothing depends on RNG reproducibility.
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def main():
    sys.path.insert(0, REF)
    from prismdg import columns as RC
    from prismdg import external2d as RE
    from prismdg import internal3d as RI
    from prismdg import mesh as RM

    os.makedirs(OUT, exist_ok=True)
    lx, ly = 1e4, 8e3

    def bed(x, y):
        return -20.0 + 5.0 * np.sin(np.pi * x / lx) * np.cos(2.0 * np.pi * y / ly)

    # ---------------------------------------------------------------- mesh
    raw = RM.generate_basin_mesh(6, 4, lx, ly, bed)
    mesh = RM.hilbert_reorder(raw)
    keys = ["vx", "vy", "vb", "tri", "j2d", "dphx", "dphy", "elen", "enx", "eny", "nbr", "nbrk", "btag",
            "hilbert_perm", "b", "x", "y"]
    np.savez_compressed(os.path.join(OUT, "mesh.npz"), raw_tri=raw.tri, raw_nbr=raw.nbr, raw_nbrk=raw.nbrk,
                        **{k: getattr(mesh, k) for k in keys})
    nt = mesh.nt
    rng = np.random.default_rng(2605)

    # ---------------------------------------------------------------- 2D
    p = RE.PhysParams(f=1e-4, cd=2.5e-3, alpha=0.2, t_ref=12.5)
    eta = 0.1 * np.cos(np.pi * mesh.x / lx) + 0.01 * rng.standard_normal((nt, 3))
    qx, qy = rng.standard_normal((nt, 3)), rng.standard_normal((nt, 3))
    f3 = rng.standard_normal((nt, 3, 2))
    src = 1e-3 * rng.standard_normal((nt, 3))
    patm = 10.0 * rng.standard_normal((nt, 3))
    st = RE.State2D(eta, qx, qy)
    res_eta = RE.rhs_free_surface(st, mesh, p, source=src)
    res_q = RE.rhs_depth_momentum(st, mesh, p, f3d2d=f3, patm=patm)
    d = RE.external_tendencies(st, mesh, p, f3d2d=f3, source=src, patm=patm)
    els = np.array([3, 0, 17, 40, 41, 12])
    d_els = RE.external_tendencies(st, mesh, p, els=els, f3d2d=f3)
    ex = RE.subcycle_external(st, mesh, p, 10, 2.0, f3d2d=f3)
    # open boundary variant: tag the west wall open with a prescribed level
    mo = RM.hilbert_reorder(RM.generate_basin_mesh(6, 4, lx, ly, bed))
    west = (mo.btag != 0) & (np.abs(mo.x[:, RM.EDGE_V0_] + mo.x[:, RM.EDGE_V1_]) < 1e-9)
    mo.btag[west] = RM.BTAG_OPEN
    d_open = RE.external_tendencies(st, mo, p, eta_bc=lambda t: 0.05 + 1e-3 * t)
    np.savez_compressed(os.path.join(OUT, "ext2d.npz"), eta=eta, qx=qx, qy=qy, f3d2d=f3, source=src, patm=patm,
                        res_eta=res_eta, res_q=res_q, d_eta=d[0], d_qx=d[1], d_qy=d[2], els=els,
                        d_els_eta=d_els[0], d_els_qx=d_els[1], d_els_qy=d_els[2],
                        sub_eta=ex.state.eta, sub_qx=ex.state.qx, sub_qy=ex.state.qy, qbar_x=ex.qbar_x,
                        qbar_y=ex.qbar_y, f2d_x=ex.f2d_x, f2d_y=ex.f2d_y, open_btag=mo.btag,
                        open_d_eta=d_open[0], open_d_qx=d_open[1], open_d_qy=d_open[2])

    # ---------------------------------------------------------------- 3D
    L = 3
    grid = RM.extrude(mesh, RM.LayerPolicy(count=L), eta)
    eta1 = eta + 0.01 * rng.standard_normal((nt, 3))
    grid1 = RM.update_moving_mesh(grid, eta1, 5.0)
    P = nt * L
    ux, uy = 0.1 * rng.standard_normal((P, 6)), 0.1 * rng.standard_normal((P, 6))
    T = 12.5 + rng.standard_normal((P, 6))
    rho = RE.eos_density(T, p)
    M = RI.prism_mass(grid)
    q = RI.project_transport(grid, ux, uy, mass=M)
    fac = RI.lateral_flux_factor(grid, q, p)
    r = RI.compute_r(grid, rho, p)
    w = RI.compute_w(grid, q, ux, uy, p, fac)
    qbx, qby = rng.standard_normal((nt, 3)), rng.standard_normal((nt, 3))
    qb = RI.consistent_transport(grid, q, qbx, qby)
    facb = RI.lateral_flux_factor(grid, qb, p)
    wt = RI.compute_wtilde(grid, qb, facb)
    Fh = RI.horizontal_rhs(grid, ux, uy, qb, facb, r, M, p)
    Ft = RI.tracer_horizontal_rhs(grid, T, qb, facb, p)
    st3 = RI.stress_rhs(grid, 0.1 / 1025, -0.05 / 1025, 2.5e-3, ux, uy)
    A = RI.assemble_vertical_operator(grid, wt, grid1.w_m, 0.5, 1e-3)
    Ai = RI.build_implicit(RI.prism_mass(grid1), A, 20.0, grid)
    rhs = rng.standard_normal((nt, L, 6, 2))
    xb = RC.solve_banded_column(Ai, rhs)
    yb = RC.apply_banded(Ai, rhs)
    ms = RI.mass_solve(M, rhs.reshape(P, 6, 2), grid)
    els3 = np.array([5, 1, 30])
    r_els = RI.compute_r(grid, rho, p, els=els3)
    Fh_els = RI.horizontal_rhs(grid, ux, uy, q, fac, r, M, p, els=els3)
    np.savez_compressed(os.path.join(OUT, "int3d.npz"), L=L, eta=eta, eta1=eta1, dt_mesh=5.0, ux=ux, uy=uy, T=T,
                        rho=rho, mass=M, q=q, fac=fac, r=r, w=w, qbx=qbx, qby=qby, qb=qb, facb=facb, wt=wt,
                        Fh=Fh, Ft=Ft, stress=st3, w_m=grid1.w_m, A_d=A.d, A_u=A.u, A_w=A.w, Ai_d=Ai.d,
                        Ai_u=Ai.u, Ai_w=Ai.w, rhs=rhs, xb=xb, yb=yb, ms=ms, els=els3, r_els=r_els,
                        Fh_els=Fh_els, z=grid.z, jz=grid.jz, dzmid=grid.dzmid, djz=grid.djz,
                        dztop=grid.dztop, dzbot=grid.dzbot, z1=grid1.z)

    # ---------------------------------------------------------------- column solvers
    Lc = 7
    j2dc = 1.0 + rng.random(5)
    rr = rng.standard_normal((5, Lc, 6, 2))
    lo, di, up, rt = (rng.standard_normal((4, 9)), 4.0 + rng.random((4, 9)),
                      rng.standard_normal((4, 9)), rng.standard_normal((4, 9)))
    np.savez_compressed(os.path.join(OUT, "columns.npz"), j2d=j2dc, rhs=rr,
                        r_out=RC.solve_r_column(rr, j2dc), w_out=RC.solve_w_column(rr, j2dc),
                        mh=RC.apply_mh(rr[:, 0, 0:3], j2dc), mhinv=RC.apply_mh_inv(rr[:, 0, 0:3], j2dc),
                        lower=lo, diag=di, upper=up, trhs=rt, tri_x=RC.solve_tridiagonal(lo, di, up, rt),
                        dense_r=RC.assemble_dense_oracle("r", 3, RC.mh_matrix(1.7)),
                        dense_w=RC.assemble_dense_oracle("w", 3, RC.mh_matrix(1.7)))

    # ---------------------------------------------------------------- two IMEX steps (reference functions
    # composed by the orchestrator of oracle/stepper.py; the reference ships no stepper)
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
    import oracle.stepper as OS
    from types import SimpleNamespace

    ref_ops = SimpleNamespace(
        eos=RE.eos_density, compute_r=RI.compute_r, prism_mass=RI.prism_mass,
        project_transport=RI.project_transport, lateral_flux_factor=RI.lateral_flux_factor,
        horizontal_rhs=RI.horizontal_rhs, stress_rhs=RI.stress_rhs, column_sum=RI.column_sum,
        consistent_transport=RI.consistent_transport, compute_wtilde=RI.compute_wtilde,
        tracer_horizontal_rhs=RI.tracer_horizontal_rhs, assemble_vertical_operator=RI.assemble_vertical_operator,
        build_implicit=RI.build_implicit, mass_apply=RI.mass_apply, mass_solve=RI.mass_solve,
        solve_banded_column=RC.solve_banded_column, apply_banded=RC.apply_banded,
        update_moving_mesh=RM.update_moving_mesh,
        subcycle=lambda s, m_, pp, ms_, dt_, f3d2d: RE.subcycle_external(s, m_, pp, ms_, dt_, f3d2d=f3d2d))
    pstep = RE.PhysParams(f=1e-4, cd=2.5e-3, alpha=0.2, t_ref=12.5, tau_x=0.05, tau_y=-0.02)
    T0 = np.where(np.repeat(mesh.x, L, axis=0).mean(1, keepdims=True) < lx / 2, 15.0, 10.0) * np.ones((1, 6))
    s = SimpleNamespace(grid=grid, ux=ux, uy=uy, T=T0, s2d=RE.State2D(eta.copy(), qx * 0.1, qy * 0.1, 0.0))
    traj = []
    for _ in range(2):
        s = OS.imex_step_ops(ref_ops, s, pstep, 40.0, 4, 1e-3, 1e-4)
        traj.append((s.ux.copy(), s.uy.copy(), s.T.copy(), s.s2d.eta.copy(), s.s2d.qx.copy(), s.s2d.qy.copy()))
    np.savez_compressed(os.path.join(OUT, "step.npz"), L=L, eta=eta, ux=ux, uy=uy, T0=T0, qx=qx * 0.1,
                        qy=qy * 0.1, dt=40.0, m=4, kv=1e-3, nu_v=1e-4,
                        **{f"s{i}_{n}": a for i, t in enumerate(traj)
                           for n, a in zip(["ux", "uy", "T", "eta", "qx", "qy"], t)})
    print("golden fixtures written to", os.path.abspath(OUT))


if __name__ == "__main__":
    main()

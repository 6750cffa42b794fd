"""Golden vectors of the explicit horizontal viscosity / diffusion from the PATCHED reference.

    python scripts/make_golden_hdiff.py      -> tests/golden/hdiff.npz

The reference's `_horizontal_diffusion` (internal3d.py:549-692) raises at internal3d.py:665 for
every mesh (a 4-D broadcast of the edge normals against a 5-D array).
oracle/refops.patch_horizontal_diffusion re-compiles the reference's own function with that one
broadcast fixed ("Hard parts" item 2): these vectors are the "patched
oracle".  Everything else -- horizontal_rhs, tracer_horizontal_rhs, the vertical operator, the
orchestrator's composition -- is the unmodified reference.

Contents: a 6x4 basin (48 tri, bumpy bed, noisy free surface) x 4 layers; seeded u, T, transports;
  D_u, D_T      _horizontal_diffusion(u, kappa_h, wall_mirror=True) / (T, nu_h, wall_mirror=False)
  Fh, Ft        horizontal_rhs / tracer_horizontal_rhs with kappa_h, kappa_v, nu_h, nu_v != 0
  Fh_els, Ft_els  the same on an element subset
  s{0,1}_*      two IMEX steps of oracle/stepper.imex_step_ops composed from the patched reference
Runs in the build container only (needs /root/reference).
"""
import os
import sys
from types import SimpleNamespace

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
REF = "/root/reference/pkg/src"
OUT = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)

KAPPA_H, KAPPA_V, NU_H, NU_V = 40.0, 1e-3, 25.0, 1e-4


def main():
    from oracle import refops
    import oracle.stepper as OS
    r = refops.load_patched(REF)
    RE, RI, RM = r.RE, r.RI, r.RM
    lx, ly = 1e4, 8e3

    def bed(x, y):
        return -20.0 + 5.0 * np.sin(np.pi * x / lx) * np.cos(2.0 * np.pi * y / ly)

    mesh = RM.hilbert_reorder(RM.generate_basin_mesh(6, 4, lx, ly, bed))
    nt, L = mesh.nt, 4
    rng = np.random.default_rng(16082)
    eta = 0.2 * np.cos(np.pi * mesh.x / lx) + 0.05 * rng.standard_normal((nt, 3))
    grid = RM.extrude(mesh, RM.LayerPolicy(count=L), eta)
    P = nt * L
    p = RE.PhysParams(f=1e-4, cd=2.5e-3, alpha=0.2, t_ref=12.5, kappa_h=KAPPA_H, kappa_v=KAPPA_V, nu_h=NU_H,
                      nu_v=NU_V)
    ux, uy = 0.1 * rng.standard_normal((P, 6)), 0.1 * rng.standard_normal((P, 6))
    T = 12.5 + rng.standard_normal((P, 6))
    U = np.stack([ux, uy], -1)
    D_u = RI._horizontal_diffusion(grid, U, KAPPA_H, KAPPA_V, None, True)
    D_T = RI._horizontal_diffusion(grid, T[..., None], NU_H, NU_V, None, False)[..., 0]
    M = RI.prism_mass(grid)
    q = RI.project_transport(grid, ux, uy, mass=M)
    fac = RI.lateral_flux_factor(grid, q, p)
    rho = RE.eos_density(T, p)
    rr = RI.compute_r(grid, rho, p)
    Fh = RI.horizontal_rhs(grid, ux, uy, q, fac, rr, M, p)
    Ft = RI.tracer_horizontal_rhs(grid, T, q, fac, p)
    els = np.array([7, 0, 33, 21, 46])
    Fh_els = RI.horizontal_rhs(grid, ux, uy, q, fac, rr, M, p, els=els)
    Ft_els = RI.tracer_horizontal_rhs(grid, T, q, fac, p, els=els)

    # two IMEX steps with horizontal viscosity / diffusion on (and the vertical operator's kh)
    pstep = RE.PhysParams(f=1e-4, cd=2.5e-3, alpha=0.2, t_ref=12.5, tau_x=0.05, tau_y=-0.02, kappa_h=KAPPA_H,
                          kappa_v=KAPPA_V, nu_h=NU_H, nu_v=NU_V)
    T0 = np.where(np.repeat(mesh.x, L, axis=0).mean(1, keepdims=True) < lx / 2, 15.0, 10.0) * np.ones((1, 6))
    qx, qy = 0.1 * rng.standard_normal((nt, 3)), 0.1 * rng.standard_normal((nt, 3))
    s = SimpleNamespace(grid=grid, ux=ux, uy=uy, T=T0, s2d=RE.State2D(eta.copy(), qx, qy, 0.0))
    traj = []
    for _ in range(2):
        s = OS.imex_step_ops(r.ops, s, pstep, 40.0, 4, 1e-3, 1e-4)
        traj.append((s.ux.copy(), s.uy.copy(), s.T.copy(), s.s2d.eta.copy(), s.s2d.qx.copy(), s.s2d.qy.copy()))
    np.savez_compressed(os.path.join(OUT, "hdiff.npz"), lx=lx, ly=ly, nx=6, ny=4, L=L, eta=eta, ux=ux, uy=uy, T=T,
                        kappa_h=KAPPA_H, kappa_v=KAPPA_V, nu_h=NU_H, nu_v=NU_V, D_u=D_u, D_T=D_T, q=q, fac=fac,
                        r=rr, Fh=Fh, Ft=Ft, els=els, Fh_els=Fh_els, Ft_els=Ft_els, T0=T0, qx=qx, qy=qy, dt=40.0,
                        m=4, kv=1e-3, nu_v_step=1e-4,
                        **{f"s{i}_{n}": a for i, t in enumerate(traj)
                           for n, a in zip(["ux", "uy", "T", "eta", "qx", "qy"], t)})
    print("wrote", os.path.abspath(os.path.join(OUT, "hdiff.npz")), "|D_u|", np.abs(D_u).max(), "|D_T|",
          np.abs(D_T).max(), "|Fh|", np.abs(Fh).max())


if __name__ == "__main__":
    main()

"""Generate tests/golden/diag.npz from the REAL reference package: diagnostics_2d
(external2d.py:366-380) and budget_3d (internal3d.py:942-951) of a seeded state.

Run in the build container only (needs /root/reference):  python scripts/make_golden_diag.py
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "diag.npz")


def main():
    sys.path.insert(0, REF)
    from prismdg import external2d as RE
    from prismdg import internal3d as RI
    from prismdg import mesh as RM

    lx, ly, L = 1.2e4, 8e3, 5

    def bed(x, y):
        return -20.0 + 5.0 * np.sin(np.pi * x / lx) * np.cos(2.0 * np.pi * y / ly)

    mesh = RM.hilbert_reorder(RM.generate_basin_mesh(9, 5, lx, ly, bed))
    nt, P = mesh.nt, mesh.nt * L
    rng = np.random.default_rng(16082)
    eta = 0.1 * np.cos(np.pi * mesh.x / lx) + 0.01 * rng.standard_normal((nt, 3))
    qx, qy = rng.standard_normal((nt, 3)), rng.standard_normal((nt, 3))
    ux, uy = 0.1 * rng.standard_normal((P, 6)), 0.1 * rng.standard_normal((P, 6))
    T = 12.0 + rng.standard_normal((P, 6))
    p = RE.PhysParams(f=1e-4, alpha=0.2, t_ref=12.5)
    d2 = RE.diagnostics_2d(RE.State2D(eta, qx, qy, 0.0), mesh, p)
    grid = RM.extrude(mesh, RM.LayerPolicy(count=L), eta)
    b3 = RI.budget_3d(grid, RI.prism_mass(grid), ux, uy, T)
    keys2 = ["total_volume", "total_energy", "eta_min", "eta_max"]
    keys3 = ["volume", "momentum_x", "momentum_y", "tracer_mass", "tracer_min", "tracer_max"]
    np.savez_compressed(OUT, nx=9, ny=5, lx=lx, ly=ly, L=L, g=p.g, eta=eta, qx=qx, qy=qy, ux=ux, uy=uy, T=T,
                        keys=np.array(keys2 + keys3), values=np.array([d2[k] for k in keys2] + [b3[k] for k in keys3]))
    print(OUT, dict(zip(keys2 + keys3, [d2[k] for k in keys2] + [b3[k] for k in keys3])))


if __name__ == "__main__":
    main()

"""Seeded initial states of the BASELINE configs' parity variants.

Pure numpy, shared by scripts/make_golden_configs.py (which steps them with the REAL reference
functions) and the GPU parity tests (which step them with the CUDA path), so both start from
bit-identical inputs.  `mesh` is any object with the Mesh2D fields (the product's and the
reference's generators build bitwise-equal meshes, tests/test_mesh.py).
"""
import numpy as np

C2 = dict(nx=32, ny=32, lx=1e4, ly=1e4, L=10, dt=40.0, m=20, kv=1e-3, nu_v=1e-4, steps=100,
          params=dict(f=1e-4, cd=2.5e-3))
# C3 lock exchange: 250 x 100 squares (50,000 tri) x 20 layers, dt2d = 1 s, m = 20
C3 = dict(nx=250, ny=100, lx=25e3, ly=10e3, L=20, dt=20.0, m=20, kv=1e-4, nu_v=1e-5,
          params=dict(f=1e-4, cd=2.5e-3, alpha=0.2, t_ref=12.5))
# a window of the C3 basin at the same 100 m resolution, stepped 100 times
C3W = dict(C3, nx=20, ny=8, lx=2e3, ly=8e2, steps=100)


def flat_bed(x, y):
    return -20.0 + 0.0 * x


def c2_state(mesh, L):
    """C2 as stated: eta0 = 0.1 cos(pi x / Lx), Q0 = 0, u0 = 0, T = 12.5.
    (The section's 0.1 N(0,1) u0 "parity variant" is not a usable 100-step case: the reference
    itself runs dry -- DryColumn -- at step 38 from it.)"""
    P = mesh.nt * L
    z = np.zeros((mesh.nt, 3))
    return dict(eta=0.1 * np.cos(np.pi * np.asarray(mesh.x) / C2["lx"]), qx=z.copy(), qy=z.copy(),
                ux=np.zeros((P, 6)), uy=np.zeros((P, 6)), T=np.full((P, 6), 12.5))


def c3_state(mesh, L, lx, seed=1):
    """C3 parity variant: lock-exchange front (T = 15 for x < Lx/2 else 10) plus seeded noise in
    every prognostic field so every column and every term is out of equilibrium."""
    rng = np.random.default_rng(seed)
    nt, P = mesh.nt, mesh.nt * L
    xc = np.repeat(np.asarray(mesh.x), L, axis=0)
    x6 = np.concatenate([xc, xc], axis=1)
    return dict(eta=0.01 * rng.standard_normal((nt, 3)), qx=0.05 * rng.standard_normal((nt, 3)),
                qy=0.05 * rng.standard_normal((nt, 3)), ux=0.05 * rng.standard_normal((P, 6)),
                uy=0.05 * rng.standard_normal((P, 6)),
                T=np.where(x6 < lx / 2, 15.0, 10.0) + 0.01 * rng.standard_normal((P, 6)))


def sample_columns(nt, n, seed=7):
    """Seeded sorted column sample that always includes the first and last columns and the edges
    of the 128-column tiles of the staged kernels."""
    rng = np.random.default_rng(seed)
    fixed = np.array([0, 1, 127, 128, nt // 2, nt - 129, nt - 128, nt - 2, nt - 1])
    fixed = fixed[(fixed >= 0) & (fixed < nt)]
    rest = rng.choice(nt, size=min(n, nt), replace=False)
    return np.unique(np.concatenate([fixed, rest]))

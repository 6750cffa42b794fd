"""Synthetic workloads of BASELINE.json `configs`.

C1  2D seiche, 32x32 basin (2,048 tri), dt2d = 2 s, 100 SSP-RK3 steps
C2  same basin, 10 sigma layers, barotropic, dt = 40 s, m = 20
C3  lock exchange, 250x100 (50,000 tri) x 20 layers, dt2d = 1 s, m = 20
C4  synthetic coastal mesh 1000x500 (1,000,000 tri) x 50 layers, dt2d = 0.25 s, m = 20  <- bench workload
    (SURVEY proposed dt2d = 0.5 s: c dt/dx = 0.235 passes check_cfl's 1/3 but P1-DG SSP-RK3 on these
    right triangles blows up in the 200 m deep part within 2 steps; 0.25 s gives 0.118.  Work per step
    -- the metric's unit -- does not depend on dt)
    (shelf 20-200 m with seeded banks, >= 15 m; density front + linear stratification; seeded smooth u0)
All meshes are Hilbert-reordered `generate_basin_mesh` meshes (mesh.py:150-228).
Random fields are seeded.  `make_case(name)` returns the mesh (host setup) and
numpy initial state in reference layouts; `device_state_c4` builds the C4 3D
fields directly on the GPU (600 M random numbers are not worth a host round trip).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .mesh import generate_basin_mesh, hilbert_reorder
from .params import PhysParams


@dataclass
class Case:
    name: str
    mesh: object
    L: int
    params: PhysParams
    dt: float
    m: int
    kv: float
    nu_v: float
    dt2d: float
    state: dict = field(default_factory=dict)

    @property
    def prisms(self):
        return self.mesh.nt * self.L


def coastal_bed(lx, ly, seed=42, nbump=8):
    rng = np.random.default_rng(seed)
    cx, cy = rng.uniform(0, lx, nbump), rng.uniform(0, ly, nbump)
    amp, rad = rng.uniform(-5.0, 30.0, nbump), rng.uniform(0.05, 0.12, nbump) * lx

    def bed(x, y):
        # shelf 20 m -> 200 m deep plus seeded Gaussian banks/holes; >= 15 m everywhere so the 50
        # sigma layers stay >= 0.3 m thick (the explicit stage-2 vertical advection needs it)
        b = -(20.0 + 180.0 * x / lx)
        for i in range(nbump):
            b = b - amp[i] * np.exp(-((x - cx[i]) ** 2 + (y - cy[i]) ** 2) / rad[i] ** 2)
        return np.minimum(b, -15.0)
    return bed


def smooth_velocity(x, y, lx, ly, seed=42, nmode=4, amp=0.05):
    """Seeded smooth horizontal velocity (sum of Fourier modes), uniform over the column."""
    rng = np.random.default_rng(seed)
    kx, ky = rng.integers(1, 4, (2, nmode)), rng.integers(1, 4, (2, nmode))
    ph, a = rng.uniform(0, 2 * np.pi, (2, nmode)), rng.uniform(-1, 1, (2, nmode))
    u = sum(a[0, i] * np.sin(np.pi * kx[0, i] * x / lx + ph[0, i]) * np.cos(np.pi * ky[0, i] * y / ly)
            for i in range(nmode))
    v = sum(a[1, i] * np.cos(np.pi * kx[1, i] * x / lx) * np.sin(np.pi * ky[1, i] * y / ly + ph[1, i])
            for i in range(nmode))
    return amp * u / nmode, amp * v / nmode


def make_case(name: str, scale: float = 1.0, with_state: bool = True, L: int | None = None) -> Case:
    """Build a config; `scale` < 1 shrinks nx, ny (used for bounded CPU samples)."""
    name = name.lower()
    if name in ("c1", "c2"):
        lx = ly = 1e4
        mesh = hilbert_reorder(generate_basin_mesh(32, 32, lx, ly, lambda x, y: -20.0 + 0.0 * x))
        p = PhysParams(f=1e-4 if name == "c2" else 0.0, cd=2.5e-3 if name == "c2" else 0.0)
        c = Case(name, mesh, L or (10 if name == "c2" else 1), p, 40.0, 20, 1e-3, 1e-4, 2.0)
        if with_state:
            nt, P = mesh.nt, mesh.nt * c.L
            z = np.zeros((nt, 3))
            c.state = dict(eta=0.1 * np.cos(np.pi * mesh.x / lx), qx=z.copy(), qy=z.copy(), ux=np.zeros((P, 6)),
                           uy=np.zeros((P, 6)), T=np.full((P, 6), 12.5))
        return c
    if name == "c3":
        nx, ny = max(2, int(250 * scale)), max(2, int(100 * scale))
        lx, ly = 25e3 * nx / 250, 10e3 * ny / 100
        mesh = hilbert_reorder(generate_basin_mesh(nx, ny, lx, ly, lambda x, y: -20.0 + 0.0 * x))
        p = PhysParams(f=1e-4, cd=2.5e-3, alpha=0.2, t_ref=12.5)
        c = Case(name, mesh, L or 20, p, 20.0, 20, 1e-4, 1e-5, 1.0)
        if with_state:
            nt, P = mesh.nt, mesh.nt * c.L
            xc = np.repeat(mesh.x, c.L, axis=0)
            xnode = np.concatenate([xc, xc], axis=1)
            z = np.zeros((nt, 3))
            c.state = dict(eta=z.copy(), qx=z.copy(), qy=z.copy(), ux=np.zeros((P, 6)), uy=np.zeros((P, 6)),
                           T=np.where(xnode < lx / 2, 15.0, 10.0))
        return c
    if name == "c4":
        # scale < 1: a window of the full C4 basin at the SAME resolution (100 m squares), centred
        # on the shelf, so per-prism cost and dynamics match the full workload (bounded CPU samples)
        nx, ny = max(2, int(1000 * scale)), max(2, int(500 * scale))
        LX, LY = 1e5, 5e4
        dx = LX / 1000
        x0 = 0.0 if nx == 1000 else 0.45 * LX
        y0 = 0.0 if ny == 500 else 0.45 * LY
        full = coastal_bed(LX, LY)
        mesh = hilbert_reorder(generate_basin_mesh(nx, ny, nx * dx, ny * dx, lambda x, y: full(x + x0, y + y0)))
        p = PhysParams(f=1e-4, cd=2.5e-3, alpha=0.2, t_ref=12.5, tau_x=0.1, tau_y=0.02)
        c = Case(name, mesh, L or 50, p, 5.0, 20, 1e-4, 1e-5, 0.25)
        c.x0, c.y0, c.lx, c.ly = x0, y0, LX, LY
        if with_state:
            c.state = c4_host_state(c)
        return c
    raise ValueError(name)


def _c4_eta(x, lx):
    return 0.05 * np.exp(-((x - 0.3 * lx) ** 2) / (0.05 * lx) ** 2)


def c4_host_state(c: Case, seed=42):
    """Host numpy C4 initial state (used for bounded CPU samples and small-scale parity)."""
    mesh, L = c.mesh, c.L
    nt, P = mesh.nt, mesh.nt * L
    lx, x0 = c.lx, c.x0
    eta = _c4_eta(mesh.x + x0, lx)
    H = eta - mesh.b
    fr = np.linspace(0.0, 1.0, L + 1)
    zt = (eta[:, None, :] - fr[None, :-1, None] * H[:, None, :]).reshape(P, 3)
    zb = (eta[:, None, :] - fr[None, 1:, None] * H[:, None, :]).reshape(P, 3)
    z = np.concatenate([zt, zb], axis=1)
    xc = np.repeat(mesh.x + x0, L, axis=0)
    x6 = np.concatenate([xc, xc], axis=1)
    T = 12.0 + 3.0 * np.tanh((x6 - 0.5 * lx) / (0.05 * lx)) + 0.02 * z
    u, v = smooth_velocity(mesh.x + x0, mesh.y + c.y0, lx, c.ly, seed)
    ux = np.repeat(np.concatenate([u, u], axis=1), L, axis=0)
    uy = np.repeat(np.concatenate([v, v], axis=1), L, axis=0)
    z2 = np.zeros((nt, 3))
    return dict(eta=eta, qx=z2.copy(), qy=z2.copy(), ux=ux, uy=uy, T=T)


def device_state_c4(c: Case, stepper, seed=42):
    """Fill a stepper with the C4 initial state generated on device, in device layouts
    (works for a partition's local mesh too: every value is a function of the node position)."""
    import torch
    mesh, L = stepper.mesh, c.L
    dev = stepper.dev
    lx, x0 = c.lx, c.x0
    eta = _c4_eta(mesh.x + x0, lx)
    S = stepper.S
    S.zero_()
    S[0].copy_(torch.as_tensor(eta.T.copy(), device=dev))
    u = stepper.U[stepper.cur]
    uu, vv = smooth_velocity(mesh.x + x0, mesh.y + c.y0, lx, c.ly, seed)
    for comp, f in ((0, uu), (1, vv)):
        ft = torch.as_tensor(f.T.copy(), device=dev)                # [3][nt]
        u[comp, 0:3] = ft[:, None, :]
        u[comp, 3:6] = ft[:, None, :]
    fr = torch.as_tensor(np.linspace(0.0, 1.0, L + 1), device=dev, dtype=torch.float64)
    e = S[0]                                    # [3][nt]
    b = torch.as_tensor(mesh.b.T.copy(), device=dev)
    H = e - b
    x = torch.as_tensor((mesh.x + x0).T.copy(), device=dev)
    T = stepper.T[stepper.cur]
    for lev, f in ((0, fr[:-1]), (1, fr[1:])):
        z = e[:, None, :] - f[None, :, None] * H[:, None, :]      # [3][L][nt]
        T[3 * lev:3 * lev + 3] = 12.0 + 3.0 * torch.tanh((x[:, None, :] - 0.5 * lx) / (0.05 * lx)) + 0.02 * z
    stepper.t = 0.0

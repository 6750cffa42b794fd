"""Mesh / column-grid restatement (prismdg/mesh.py).  Oracle / test infrastructure only.

Objects are plain attribute bags with the reference's field names, so the
product's Mesh2D / ColumnGrid can be handed to oracle functions and vice versa.
"""
from types import SimpleNamespace

import numpy as np

from paper_2605_16082_b200.errors import (DegenerateLayer, DryColumn, NonConforming,
                                          NonPositiveArea, NonPositiveLength)
from .tables import BTAG_INTERIOR, BTAG_WALL, EV0, EV1


class OMesh(SimpleNamespace):
    @property
    def nt(self):
        return self.tri.shape[0]

    @property
    def nv(self):
        return self.vx.shape[0]

    @property
    def min_edge(self):
        return float(self.elen.min())


def pair_edges(tri):
    """Edge pairing of mesh.py:107-127 (dict pass in element order).

    Restated as a stable sort of the sorted vertex-pair keys followed by pairing
    consecutive equal keys, which reproduces the dict's first-come pairing
    (occurrences 1&2, 3&4, ...) exactly.
    """
    nt = tri.shape[0]
    a = tri[:, EV0].ravel()
    b = tri[:, EV1].ravel()
    lo, hi = np.minimum(a, b), np.maximum(a, b)
    order = np.lexsort((hi, lo))            # stable: ties keep flat (e*3+k) order
    klo, khi = lo[order], hi[order]
    nbr = np.full(3 * nt, -1, dtype=np.int64)
    nbrk = np.full(3 * nt, -1, dtype=np.int64)
    same = (klo[1:] == klo[:-1]) & (khi[1:] == khi[:-1])
    # run-position parity: pair run members (0,1), (2,3), ...
    start = np.ones(order.size, dtype=bool)
    start[1:] = ~same
    run_id = np.cumsum(start) - 1
    first_idx = np.flatnonzero(start)
    pos = np.arange(order.size) - first_idx[run_id]
    run_len = np.diff(np.append(first_idx, order.size))[run_id]
    left = (pos % 2 == 0) & (pos + 1 < run_len)
    i = np.flatnonzero(left)
    f1, f2 = order[i], order[i + 1]
    nbr[f1], nbrk[f1] = f2 // 3, f2 % 3
    nbr[f2], nbrk[f2] = f1 // 3, f1 % 3
    nbr, nbrk = nbr.reshape(nt, 3), nbrk.reshape(nt, 3)
    btag = np.where(nbr >= 0, BTAG_INTERIOR, BTAG_WALL).astype(np.int64)
    return nbr, nbrk, btag


def make_mesh(vx, vy, vb, tri, perm=None):
    """mesh.py:79-105, 140-147: nodal coordinates, J2D, grad(phi), edges, adjacency."""
    m = OMesh(vx=np.asarray(vx, float), vy=np.asarray(vy, float),
              vb=np.asarray(vb, float), tri=np.asarray(tri, np.int64))
    t = m.tri
    x, y = m.vx[t], m.vy[t]
    m.x, m.y, m.b = x, y, m.vb[t]
    m.j2d = (x[:, 1] - x[:, 0]) * (y[:, 2] - y[:, 0]) - (x[:, 2] - x[:, 0]) * (y[:, 1] - y[:, 0])
    if np.any(m.j2d <= 0.0):
        bad = int(np.argmin(m.j2d))
        raise NonPositiveArea(f"triangle {bad} has signed area {m.j2d[bad] / 2.0:g}")
    nxt, prv = [1, 2, 0], [2, 0, 1]
    m.dphx = (y[:, nxt] - y[:, prv]) / m.j2d[:, None]
    m.dphy = (x[:, prv] - x[:, nxt]) / m.j2d[:, None]
    dx = x[:, EV1] - x[:, EV0]
    dy = y[:, EV1] - y[:, EV0]
    m.elen = np.hypot(dx, dy)
    if np.any(m.elen <= 0.0):
        raise NonPositiveLength("zero-length edge")
    m.enx = dy / m.elen
    m.eny = -dx / m.elen
    m.nbr, m.nbrk, m.btag = pair_edges(t)
    m.hilbert_perm = np.arange(m.nt) if perm is None else perm
    return m


def basin_mesh(nx, ny, lx, ly, bed):
    """mesh.py:150-179: 2 nx ny CCW triangles, row-major squares."""
    if nx < 1 or ny < 1:
        raise NonPositiveArea("nx and ny must be >= 1")
    if lx <= 0.0 or ly <= 0.0:
        raise NonPositiveArea("lx and ly must be positive")
    gx, gy = np.meshgrid(np.linspace(0.0, lx, nx + 1), np.linspace(0.0, ly, ny + 1), indexing="xy")
    vx, vy = gx.ravel(), gy.ravel()
    vb = np.asarray(bed(vx, vy), float)
    j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    v00 = (j * (nx + 1) + i).ravel()
    v10, v11, v01 = v00 + 1, v00 + nx + 2, v00 + nx + 1
    tri = np.empty((2 * nx * ny, 3), np.int64)
    tri[0::2] = np.stack([v00, v10, v11], 1)
    tri[1::2] = np.stack([v00, v11, v01], 1)
    return make_mesh(vx, vy, vb, tri)


def hilbert_d(order, ix, iy):
    """mesh.py:187-207: distance along the order-`order` Hilbert curve."""
    x = np.array(ix, dtype=np.int64)
    y = np.array(iy, dtype=np.int64)
    n = np.int64(1) << order
    d = np.zeros_like(x)
    s = n >> 1
    while s > 0:
        rx = (x & s) > 0
        ry = (y & s) > 0
        d += s * s * ((3 * rx.astype(np.int64)) ^ ry.astype(np.int64))
        flip = (~ry) & rx
        x = np.where(flip, n - 1 - x, x)
        y = np.where(flip, n - 1 - y, y)
        x, y = np.where(~ry, y, x), np.where(~ry, x, y)
        s >>= 1
    return d


def hilbert_reorder(mesh, order=16):
    """mesh.py:210-228: stable argsort of the centroid Hilbert index."""
    cx, cy = mesh.x.mean(axis=1), mesh.y.mean(axis=1)
    n = np.int64(1) << order
    sx = max(cx.max() - cx.min(), 1e-300)
    sy = max(cy.max() - cy.min(), 1e-300)
    ix = np.minimum(n - 1, ((cx - cx.min()) / sx * (n - 1)).astype(np.int64))
    iy = np.minimum(n - 1, ((cy - cy.min()) / sy * (n - 1)).astype(np.int64))
    perm = np.argsort(hilbert_d(order, ix, iy), kind="stable")
    return make_mesh(mesh.vx, mesh.vy, mesh.vb, mesh.tri[perm], perm=perm)


class OGrid(SimpleNamespace):
    @property
    def n_prisms(self):
        return self.z.shape[0]

    @property
    def n_layers(self):
        return int(self.layers[0])


def extrude(mesh, L, eta=None):
    """mesh.py:371-408 (uniform policy) + ColumnGrid._finish (:343-356)."""
    nt = mesh.nt
    eta = np.zeros((nt, 3)) if eta is None else np.asarray(eta, float)
    H = eta - mesh.b
    if np.any(H <= 0.0):
        c = int(np.argmin(H.min(axis=1)))
        raise DryColumn(c, float(H[c].min()))
    fr = np.linspace(0.0, 1.0, L + 1)
    zi = eta[:, None, :] - fr[None, :, None] * H[:, None, :]       # (nt, L+1, 3)
    zt = zi[:, :-1].reshape(nt * L, 3)
    zb = zi[:, 1:].reshape(nt * L, 3)
    jz = 0.5 * (zt - zb)
    if np.any(jz <= 0.0):
        raise DegenerateLayer("non-positive layer thickness after extrusion")
    g = OGrid(mesh=mesh, layers=np.full(nt, L, np.int64), fracs=fr, eta=eta.copy(),
              z=np.concatenate([zt, zb], 1), jz=jz, w_m=np.zeros((nt * L, 6)))
    g.offsets = np.arange(nt + 1, dtype=np.int64) * L
    dx = np.repeat(mesh.dphx, L, axis=0)
    dy = np.repeat(mesh.dphy, L, axis=0)

    def grad(f):
        return np.stack([(f * dx).sum(1), (f * dy).sum(1)], -1)
    g.dzmid = grad(0.5 * (zt + zb))
    g.djz = grad(jz)
    g.dztop = grad(zt)
    g.dzbot = grad(zb)
    return g


def update_moving_mesh(grid, eta_new, dt):
    """mesh.py:411-419."""
    new = extrude(grid.mesh, grid.n_layers, eta_new)
    new.w_m = (new.z - grid.z) / float(dt)
    return new


def total_thickness(grid):
    """mesh.py:422-426."""
    nt, L = grid.mesh.nt, grid.n_layers
    return 2.0 * grid.jz.reshape(nt, L, 3).sum(axis=1)

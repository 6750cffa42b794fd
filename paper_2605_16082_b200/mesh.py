"""Triangle mesh and sigma column grid -- drop-in for prismdg/mesh.py.

Mesh2D keeps the reference's field names (mesh.py:35-54) so existing user code
works.  Connectivity is built with a stable sort of the edge keys, which
reproduces the reference's dict pairing (mesh.py:107-127) bit-exactly (pinned by
tests/test_mesh.py against golden vectors) at O(nt log nt) instead of a Python
loop.  This is one-time setup on the host; everything per step runs on device.

ColumnGrid carries only what the device path needs -- the free surface it was
extruded from, the layer count and the sigma fractions.  The prism geometry
(z, Jz, grad z, w_m; mesh.py:308-356, 389-419) is recomputed on the fly inside
the kernels; the array attributes exist for API compatibility and are derived
lazily on the host only if a caller reads them.
"""
from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Callable, Optional

import numpy as np

from .errors import DegenerateLayer, DryColumn, NonConforming, NonPositiveArea, NonPositiveLength
from .params import LayerPolicy

BTAG_INTERIOR = 0
BTAG_WALL = 1
BTAG_OPEN = 2
EDGE_V0_ = np.array([0, 1, 2])
EDGE_V1_ = np.array([1, 2, 0])


@dataclass
class Mesh2D:
    vx: np.ndarray
    vy: np.ndarray
    vb: np.ndarray
    tri: np.ndarray
    x: np.ndarray = None
    y: np.ndarray = None
    b: np.ndarray = None
    j2d: np.ndarray = None
    dphx: np.ndarray = None
    dphy: np.ndarray = None
    nbr: np.ndarray = None
    nbrk: np.ndarray = None
    btag: np.ndarray = None
    elen: np.ndarray = None
    enx: np.ndarray = None
    eny: np.ndarray = None
    hilbert_perm: np.ndarray = None

    @property
    def nt(self) -> int:
        return self.tri.shape[0]

    @property
    def nv(self) -> int:
        return self.vx.shape[0]

    @property
    def area(self) -> np.ndarray:
        return 0.5 * self.j2d

    @property
    def min_edge(self) -> float:
        return float(self.elen.min())

    def n_interior_edges(self) -> int:
        return int(np.count_nonzero(self.nbr >= 0)) // 2

    def n_edges(self) -> int:
        return self.n_interior_edges() + int(np.count_nonzero(self.nbr < 0))

    def _finish(self) -> "Mesh2D":
        """Geometry + adjacency: on the GPU (csrc/mesh.cu) when one is present, else on the host."""
        if _gpu():
            return self._finish_device()
        return self._finish_host()

    def _finish_device(self) -> "Mesh2D":
        import ctypes

        import torch

        from . import _lib
        from .device import stream_ptr
        from .errors import raise_for_code
        dev = torch.device("cuda", torch.cuda.current_device())
        nt = self.nt
        f = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)  # noqa: E731
        vx, vy, vb = f(self.vx), f(self.vy), f(self.vb)
        tri = torch.as_tensor(np.ascontiguousarray(self.tri, dtype=np.int64), device=dev)
        out = {k: torch.empty((nt, 3), dtype=torch.float64, device=dev)
               for k in ("x", "y", "b", "dphx", "dphy", "elen", "enx", "eny")}
        out["j2d"] = torch.empty(nt, dtype=torch.float64, device=dev)
        ints = {k: torch.empty((nt, 3), dtype=torch.int64, device=dev) for k in ("nbr", "nbrk", "btag")}
        err = torch.zeros(4, dtype=torch.int64, device=dev)
        p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        _lib.check(_lib.lib().pdg_mesh_build(nt, self.nv, p(vx), p(vy), p(vb), p(tri), p(out["x"]), p(out["y"]),
                                             p(out["b"]), p(out["j2d"]), p(out["dphx"]), p(out["dphy"]),
                                             p(out["elen"]), p(out["enx"]), p(out["eny"]), p(ints["nbr"]),
                                             p(ints["nbrk"]), p(ints["btag"]), p(err), stream_ptr()), "mesh_build")
        h = err.cpu()
        if int(h[0]) & 0xFFFFFFFF:
            raise_for_code(int(h[0]) & 0xFFFFFFFF, int(h[1]), int(h[2]), float(h[3:4].view(torch.float64).item()))
        for k, v in out.items():
            setattr(self, k, v.cpu().numpy())
        for k, v in ints.items():
            setattr(self, k, v.cpu().numpy())
        if self.hilbert_perm is None:
            self.hilbert_perm = np.arange(self.nt)
        return self

    def _finish_host(self) -> "Mesh2D":
        t = self.tri
        X, Y = self.vx[t], self.vy[t]
        self.x, self.y, self.b = X, Y, self.vb[t]
        # J2D = 2 area (mesh.py:85), grad(phi_i) = (y_j - y_k, x_k - x_j)/J2D, (i,j,k) cyclic
        self.j2d = (X[:, 1] - X[:, 0]) * (Y[:, 2] - Y[:, 0]) - (X[:, 2] - X[:, 0]) * (Y[:, 1] - Y[:, 0])
        if np.any(self.j2d <= 0.0):
            bad = int(np.argmin(self.j2d))
            raise NonPositiveArea(f"triangle {bad} has signed area {self.j2d[bad] / 2.0:g}")
        cyc1, cyc2 = np.array([1, 2, 0]), np.array([2, 0, 1])
        self.dphx = (Y[:, cyc1] - Y[:, cyc2]) / self.j2d[:, None]
        self.dphy = (X[:, cyc2] - X[:, cyc1]) / self.j2d[:, None]
        ex = X[:, EDGE_V1_] - X[:, EDGE_V0_]
        ey = Y[:, EDGE_V1_] - Y[:, EDGE_V0_]
        self.elen = np.hypot(ex, ey)
        if np.any(self.elen <= 0.0):
            raise NonPositiveLength("zero-length edge")
        self.enx = ey / self.elen
        self.eny = -ex / self.elen
        self._build_adjacency()
        if self.hilbert_perm is None:
            self.hilbert_perm = np.arange(self.nt)
        return self

    def _build_adjacency(self):
        nt = self.nt
        a = self.tri[:, EDGE_V0_].reshape(-1)
        b = self.tri[:, EDGE_V1_].reshape(-1)
        key = np.minimum(a, b) * (int(max(a.max(), b.max())) + 1) + np.maximum(a, b)
        order = np.argsort(key, kind="stable")          # first-come order inside equal keys
        ks = key[order]
        brk = np.ones(ks.size, dtype=bool)
        brk[1:] = ks[1:] != ks[:-1]
        first = np.flatnonzero(brk)
        grp = np.cumsum(brk) - 1
        rank = np.arange(ks.size) - first[grp]
        size = np.diff(np.append(first, ks.size))[grp]
        lead = np.flatnonzero((rank & 1 == 0) & (rank + 1 < size))
        f1, f2 = order[lead], order[lead + 1]
        nbr = np.full(3 * nt, -1, dtype=np.int64)
        nbrk = np.full(3 * nt, -1, dtype=np.int64)
        nbr[f1], nbrk[f1], nbr[f2], nbrk[f2] = f2 // 3, f2 % 3, f1 // 3, f1 % 3
        self.nbr, self.nbrk = nbr.reshape(nt, 3), nbrk.reshape(nt, 3)
        self.btag = np.where(self.nbr >= 0, BTAG_INTERIOR, BTAG_WALL).astype(np.int64)

    def astype(self, dtype) -> "Mesh2D":
        m = replace(self)
        for name in ("vx", "vy", "vb", "x", "y", "b", "j2d", "dphx", "dphy", "elen", "enx", "eny"):
            setattr(m, name, getattr(self, name).astype(dtype))
        return m


def _gpu() -> bool:
    """Mesh setup runs on the GPU (csrc/mesh.cu).  The host restatement is used only when it is
    asked for explicitly (PDG_MESH_HOST=1: CPU-only processes such as the oracle baseline workers
    and the CPU test suite); without it a missing GPU or a broken library raises."""
    import os
    if os.environ.get("PDG_MESH_HOST"):
        return False
    import torch
    from . import _lib
    if not torch.cuda.is_available():
        raise RuntimeError("Mesh2D setup needs a CUDA device (csrc/mesh.cu); set PDG_MESH_HOST=1 to build "
                           "the connectivity on the host instead")
    _lib.lib()                                 # raises if the sm_100a library is missing
    return True


def make_mesh(vx, vy, vb, tri) -> Mesh2D:
    """mesh.py:140-147."""
    return Mesh2D(vx=np.asarray(vx, float), vy=np.asarray(vy, float), vb=np.asarray(vb, float),
                  tri=np.asarray(tri, np.int64))._finish()


def generate_basin_mesh(nx, ny, lx, ly, bed: Callable) -> Mesh2D:
    """mesh.py:150-179: structured 2 nx ny CCW triangles over [0,lx]x[0,ly], walls everywhere."""
    if nx < 1 or ny < 1:
        raise NonPositiveArea("nx and ny must be >= 1")
    if lx <= 0.0 or ly <= 0.0:
        raise NonPositiveArea("lx and ly must be positive")
    gx, gy = np.meshgrid(np.linspace(0.0, lx, nx + 1), np.linspace(0.0, ly, ny + 1), indexing="xy")
    vx, vy = gx.ravel(), gy.ravel()
    base = (np.arange(ny)[:, None] * (nx + 1) + np.arange(nx)[None, :]).ravel()
    quads = np.stack([base, base + 1, base + nx + 2, base + nx + 1], axis=1)
    tri = np.empty((2 * base.size, 3), np.int64)
    tri[0::2] = quads[:, [0, 1, 2]]
    tri[1::2] = quads[:, [0, 2, 3]]
    return make_mesh(vx, vy, np.asarray(bed(vx, vy), float), tri)


def hilbert_index(order: int, ix, iy) -> np.ndarray:
    """Distance along the order-`order` Hilbert curve (mesh.py:187-207)."""
    x = np.asarray(ix, np.int64).copy()
    y = np.asarray(iy, np.int64).copy()
    n = np.int64(1) << order
    d = np.zeros_like(x)
    s = n >> 1
    while s > 0:
        rx = (x & s) != 0
        ry = (y & s) != 0
        d += s * s * ((3 * rx) ^ ry)
        low = ~ry
        mirror = low & rx
        x[mirror] = n - 1 - x[mirror]
        y[mirror] = n - 1 - y[mirror]
        x[low], y[low] = y[low], x[low].copy()
        s >>= 1
    return d


def hilbert_reorder(mesh: Mesh2D, order: int = 16) -> Mesh2D:
    """mesh.py:210-228 (stable, idempotent); the permutation is computed on the GPU when present."""
    if _gpu():
        perm = hilbert_perm_device(mesh, order)
        out = make_mesh(mesh.vx, mesh.vy, mesh.vb, mesh.tri[perm])
        out.hilbert_perm = perm
        return out
    cx, cy = mesh.x.mean(axis=1), mesh.y.mean(axis=1)
    n = np.int64(1) << order
    sx = max(cx.max() - cx.min(), 1e-300)
    sy = max(cy.max() - cy.min(), 1e-300)
    ix = np.minimum(n - 1, ((cx - cx.min()) / sx * (n - 1)).astype(np.int64))
    iy = np.minimum(n - 1, ((cy - cy.min()) / sy * (n - 1)).astype(np.int64))
    perm = np.argsort(hilbert_index(order, ix, iy), kind="stable")
    out = make_mesh(mesh.vx, mesh.vy, mesh.vb, mesh.tri[perm])
    out.hilbert_perm = perm
    return out


def hilbert_perm_device(mesh, order: int = 16) -> np.ndarray:
    """hilbert_reorder's permutation computed on the GPU (csrc/mesh.cu: pdg_hilbert_perm)."""
    import ctypes

    import torch

    from . import _lib
    from .device import stream_ptr
    dev = torch.device("cuda", torch.cuda.current_device())
    x = torch.as_tensor(np.ascontiguousarray(mesh.x), device=dev)
    y = torch.as_tensor(np.ascontiguousarray(mesh.y), device=dev)
    perm = torch.empty(mesh.nt, dtype=torch.int64, device=dev)
    _lib.check(_lib.lib().pdg_hilbert_perm(mesh.nt, order, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                                           ctypes.c_void_p(perm.data_ptr()), stream_ptr()), "hilbert_perm")
    return perm.cpu().numpy()


def hilbert_reorder_host(mesh: Mesh2D, order: int = 16) -> Mesh2D:
    cx, cy = mesh.x.mean(axis=1), mesh.y.mean(axis=1)
    n = np.int64(1) << order
    sx = max(cx.max() - cx.min(), 1e-300)
    sy = max(cy.max() - cy.min(), 1e-300)
    ix = np.minimum(n - 1, ((cx - cx.min()) / sx * (n - 1)).astype(np.int64))
    iy = np.minimum(n - 1, ((cy - cy.min()) / sy * (n - 1)).astype(np.int64))
    perm = np.argsort(hilbert_index(order, ix, iy), kind="stable")
    out = make_mesh(mesh.vx, mesh.vy, mesh.vb, mesh.tri[perm])
    out.hilbert_perm = perm
    return out


def mesh_locality(mesh: Mesh2D) -> float:
    """mesh.py:231-238."""
    e, k = np.nonzero(mesh.nbr >= 0)
    j = mesh.nbr[e, k]
    keep = e < j
    return float(np.abs(e[keep] - j[keep]).mean()) if np.any(keep) else 0.0


def write_mesh(path, mesh: Mesh2D) -> None:
    """PRISMDG-MESH 1 (mesh.py:246-253); plain-float repr (the reference's
    `!r` of numpy scalars writes `np.float64(...)` under numpy 2, which its own reader rejects)."""
    with open(path, "w") as f:
        f.write("PRISMDG-MESH 1\n")
        f.write(f"{mesh.nv} {mesh.nt}\n")
        for i in range(mesh.nv):
            f.write(f"{float(mesh.vx[i])!r} {float(mesh.vy[i])!r} {float(mesh.vb[i])!r}\n")
        for t in mesh.tri:
            f.write(f"{t[0]} {t[1]} {t[2]}\n")


def read_mesh(path) -> Mesh2D:
    """mesh.py:256-271."""
    with open(path) as f:
        head = f.readline().split()
        if head[:2] != ["PRISMDG-MESH", "1"]:
            raise ValueError(f"not a PRISMDG-MESH 1 file: {path}")
        nv, nt = (int(t) for t in f.readline().split())
        v = np.array([[float(t) for t in f.readline().split()[:3]] for _ in range(nv)]).reshape(nv, 3)
        tri = np.array([[int(t) for t in f.readline().split()[:3]] for _ in range(nt)], np.int64).reshape(nt, 3)
    return make_mesh(v[:, 0], v[:, 1], v[:, 2], tri)


# --------------------------------------------------------------------------- column grid

class ColumnGrid:
    """Sigma column grid for one free-surface snapshot (mesh.py:308-356).

    Device kernels rebuild z / Jz / grad z from (eta, b, fracs); the array
    attributes below are computed lazily on the host only for API users.
    """

    def __init__(self, mesh: Mesh2D, layers=None, offsets=None, fracs=None, eta=None, z=None, jz=None, w_m=None,
                 dzmid=None, djz=None, dztop=None, dzbot=None, *, L: int | None = None, eta_prev=None,
                 dt_prev=None):
        """The reference dataclass's field order (mesh.py:308-325): (mesh, layers, offsets, fracs,
        eta, z, jz, w_m, dzmid, djz, dztop, dzbot).  Array fields left out are derived from
        (eta, fracs) on first access; ones passed in are kept as given (the device kernels always
        rebuild the geometry from eta, b and fracs).  Keyword-only extras: L (uniform layer count
        instead of `layers`) and eta_prev / dt_prev (the previous free surface and step, from which
        w_m is derived, mesh.py:418)."""
        if layers is None:
            if L is None:
                raise TypeError("ColumnGrid needs `layers` (per-column counts) or L=")
            layers = np.full(mesh.nt, int(L), dtype=np.int64)
        elif np.ndim(layers) == 0:          # a bare layer count
            layers = np.full(mesh.nt, int(layers), dtype=np.int64)
        self.mesh = mesh
        self.layers = np.asarray(layers, dtype=np.int64)
        if self.layers.size and self.layers.min() != self.layers.max():
            raise NonConforming("the device path needs one layer count for every column")
        Lc = self.n_layers
        self.offsets = np.arange(mesh.nt + 1, dtype=np.int64) * Lc if offsets is None else np.asarray(offsets)
        self.fracs = np.linspace(0.0, 1.0, Lc + 1) if fracs is None else np.asarray(fracs, dtype=float)
        self.eta = np.zeros((mesh.nt, 3)) if eta is None else eta
        self._eta_prev = eta_prev
        self._dt_prev = dt_prev
        self._geo = None
        given = dict(z=z, jz=jz, dzmid=dzmid, djz=djz, dztop=dztop, dzbot=dzbot)
        self._given = {k: v for k, v in given.items() if v is not None}
        self._w_m = w_m

    @property
    def n_layers(self) -> int:
        return int(self.layers[0]) if self.layers.size else 0

    @property
    def n_prisms(self) -> int:
        return self.mesh.nt * self.n_layers

    @property
    def depth(self) -> np.ndarray:
        return np.asarray(self.eta) - self.mesh.b

    def column_slice(self, c: int) -> slice:
        return slice(self.offsets[c], self.offsets[c + 1])

    def _z(self, eta):
        eta = np.asarray(eta)
        H = eta - self.mesh.b
        zi = eta[:, None, :] - self.fracs[None, :, None] * H[:, None, :]
        nt, L = self.mesh.nt, self.n_layers
        return zi[:, :-1].reshape(nt * L, 3), zi[:, 1:].reshape(nt * L, 3)

    def _geometry(self):
        if self._geo is None:
            zt, zb = self._z(self.eta)
            L = self.n_layers
            dx, dy = np.repeat(self.mesh.dphx, L, axis=0), np.repeat(self.mesh.dphy, L, axis=0)

            def grad(f):
                return np.stack([(f * dx).sum(axis=1), (f * dy).sum(axis=1)], axis=-1)
            jz = 0.5 * (zt - zb)
            self._geo = dict(z=np.concatenate([zt, zb], axis=1), jz=jz, dzmid=grad(0.5 * (zt + zb)), djz=grad(jz),
                             dztop=grad(zt), dzbot=grad(zb))
        return self._geo

    def _field(self, k):
        v = self._given.get(k)
        return v if v is not None else self._geometry()[k]

    z = property(lambda self: self._field("z"))
    jz = property(lambda self: self._field("jz"))
    dzmid = property(lambda self: self._field("dzmid"))
    djz = property(lambda self: self._field("djz"))
    dztop = property(lambda self: self._field("dztop"))
    dzbot = property(lambda self: self._field("dzbot"))

    @property
    def w_m(self) -> np.ndarray:
        """Nodal mesh velocity (z - z_prev)/dt (mesh.py:418); zero for a fresh extrusion."""
        if self._w_m is not None:
            return self._w_m
        if self._eta_prev is None:
            return np.zeros((self.n_prisms, 6))
        zt, zb = self._z(self._eta_prev)
        return (self.z - np.concatenate([zt, zb], axis=1)) / float(self._dt_prev)


def _check_conforming(mesh: Mesh2D, counts: np.ndarray) -> None:
    e, k = np.nonzero(mesh.nbr >= 0)
    j = mesh.nbr[e, k]
    bad = counts[e] != counts[j]
    if np.any(bad):
        i = int(np.argmax(bad))
        raise NonConforming(f"columns {e[i]} and {j[i]} share an edge but have {counts[e[i]]} vs {counts[j[i]]} layers")


def extrude(mesh: Mesh2D, policy: LayerPolicy, eta=None) -> ColumnGrid:
    """mesh.py:371-408."""
    eta = np.zeros((mesh.nt, 3)) if eta is None else np.asarray(eta, dtype=float)
    counts = policy.counts(mesh, eta)
    _check_conforming(mesh, counts)
    if counts.size and counts.min() != counts.max():
        raise NonConforming("layer counts differ between mesh components")
    H = eta - mesh.b
    if np.any(H <= 0.0):
        c = int(np.argmin(H.min(axis=1)))
        raise DryColumn(c, float(H[c].min()))
    L = int(counts[0])
    g = ColumnGrid(mesh, L=L, eta=eta.copy())
    if L > 1 and np.any(np.diff(g.fracs) <= 0.0):
        raise DegenerateLayer("non-positive layer thickness after extrusion")
    return g


def update_moving_mesh(grid: ColumnGrid, eta_new, dt: float) -> ColumnGrid:
    """mesh.py:411-419: new grid following eta_new, w_m = (z_new - z_old)/dt."""
    new = extrude(grid.mesh, LayerPolicy(mode="uniform", count=grid.n_layers), np.asarray(eta_new, dtype=float))
    new._eta_prev = np.asarray(grid.eta)
    new._dt_prev = float(dt)
    return new


def total_thickness(grid: ColumnGrid) -> np.ndarray:
    """mesh.py:422-426."""
    nt, L = grid.mesh.nt, grid.n_layers
    return 2.0 * grid.jz.reshape(nt, L, 3).sum(axis=1)

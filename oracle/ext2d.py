"""External (2D) mode restatement (prismdg/external2d.py).  Oracle / test infrastructure only.

States are attribute bags with eta, qx, qy (nt, 3) and t.
"""
from types import SimpleNamespace

import numpy as np

from paper_2605_16082_b200.errors import CflViolation, DryColumn, SingularMass
from .tables import BARY, BTAG_INTERIOR, BTAG_OPEN, ES, EV0, EV1, QW, ZQW


def mh_apply(v, j2d):
    """columns.py:45-56: (J2D/24)(v + sum v), component axis optional (last)."""
    v = np.asarray(v)
    if v.shape[-1] == 3:
        return (v + v.sum(-1)[..., None]) * (np.asarray(j2d)[..., None] / 24.0)
    return (v + v.sum(-2)[..., None, :]) * (np.asarray(j2d)[..., None, None] / 24.0)


def mh_inv_apply(v, j2d):
    """columns.py:59-69: (6/J2D)(4 v - sum v)."""
    v = np.asarray(v)
    j2d = np.asarray(j2d, dtype=v.dtype)
    if np.any(j2d <= 0.0):
        raise SingularMass("J2D must be positive")
    if v.shape[-1] == 3:
        return (4.0 * v - v.sum(-1)[..., None]) * (6.0 / j2d)[..., None]
    return (4.0 * v - v.sum(-2)[..., None, :]) * (6.0 / j2d)[..., None, None]


def eos(T, p, S=None):
    """external2d.py:81-87 linear EOS."""
    rho = -p.alpha * (np.asarray(T) - p.t_ref)
    if p.beta != 0.0:
        s = p.s_ref if S is None else np.asarray(S)
        rho = rho + p.beta * (s - p.s_ref)
    return rho


def own_trace(f, rows, k):
    """external2d.py:95-99: (n, 2) values at the edge Gauss points."""
    return f[rows, EV0[k]][:, None] * ES[:, 0] + f[rows, EV1[k]][:, None] * ES[:, 1]


def nbr_trace(f, e2, k2):
    """external2d.py:102-107: neighbour trace, mirrored point order."""
    e2 = np.maximum(e2, 0)
    return f[e2, EV0[k2]][:, None] * ES[:, 1] + f[e2, EV1[k2]][:, None] * ES[:, 0]


def _edge_states(st, mesh, rows, k, eta_bc):
    """Interior/exterior traces incl. wall and open closures (external2d.py:150-173)."""
    e2, k2, tag = mesh.nbr[rows, k], mesh.nbrk[rows, k], mesh.btag[rows, k]
    nx, ny = mesh.enx[rows, k][:, None], mesh.eny[rows, k][:, None]
    tr = {n: own_trace(f, rows, k) for n, f in (("e", st.eta), ("x", st.qx), ("y", st.qy), ("b", mesh.b))}
    ex = {n: nbr_trace(f, e2, k2) for n, f in (("e", st.eta), ("x", st.qx), ("y", st.qy), ("b", mesh.b))}
    bnd = (tag != BTAG_INTERIOR)[:, None]
    if np.any(bnd):
        opn = (tag == BTAG_OPEN)[:, None]
        qn = nx * tr["x"] + ny * tr["y"]
        ew = tr["e"] if eta_bc is None else np.full_like(tr["e"], eta_bc(st.t))
        ex["e"] = np.where(bnd, np.where(opn, ew, tr["e"]), ex["e"])
        ex["x"] = np.where(bnd, np.where(opn, tr["x"], tr["x"] - 2.0 * qn * nx), ex["x"])
        ex["y"] = np.where(bnd, np.where(opn, tr["y"], tr["y"] - 2.0 * qn * ny), ex["y"])
        ex["b"] = np.where(bnd, tr["b"], ex["b"])
    return tr, ex, nx, ny


def _celerity(tr, ex, g):
    """external2d.py:110-116."""
    hi, he = tr["e"] - tr["b"], ex["e"] - ex["b"]
    if np.any(hi <= 0.0) or np.any(he <= 0.0):
        raise DryColumn(-1, float(min(hi.min(), he.min())))
    return np.maximum(np.sqrt(g * hi), np.sqrt(g * he))


def _edge_scatter(res, k, flux, elen):
    """external2d.py:119-125: res[:, edge nodes] -= Jedge sum_q w_q phi flux."""
    je = 0.5 * elen
    for q in range(2):
        wq = ZQW[q] * je * flux[:, q]
        res[:, EV0[k]] -= wq * ES[q, 0]
        res[:, EV1[k]] -= wq * ES[q, 1]


def _rows(mesh, els):
    return np.arange(mesh.nt) if els is None else np.asarray(els)


def free_surface_residual(st, mesh, p, els=None, source=None, eta_bc=None):
    """external2d.py:128-184 (residual before Mh^-1), shape (nel, 3)."""
    rows = _rows(mesh, els)
    j2d = mesh.j2d[rows]
    qxi = (st.qx[rows] @ BARY.T) @ QW
    qyi = (st.qy[rows] @ BARY.T) @ QW
    res = j2d[:, None] * (mesh.dphx[rows] * qxi[:, None] + mesh.dphy[rows] * qyi[:, None])
    for k in range(3):
        tr, ex, nx, ny = _edge_states(st, mesh, rows, k, eta_bc)
        c = _celerity(tr, ex, p.g)
        flux = nx * 0.5 * (tr["x"] + ex["x"]) + ny * 0.5 * (tr["y"] + ex["y"]) + c * 0.5 * (tr["e"] - ex["e"])
        _edge_scatter(res, k, flux, mesh.elen[rows, k])
    if source is not None:
        res += mh_apply(np.asarray(source)[rows], j2d)
    return res


def momentum_residual(st, mesh, p, els=None, f3d2d=None, patm=None, eta_bc=None):
    """external2d.py:187-256, shape (nel, 3, 2)."""
    rows = _rows(mesh, els)
    g = p.g
    j2d = mesh.j2d[rows]
    e = st.eta[rows]
    gx = (e * mesh.dphx[rows]).sum(1)
    gy = (e * mesh.dphy[rows]).sum(1)
    hq = (e - mesh.b[rows]) @ BARY.T
    if np.any(hq <= 0.0):
        raise DryColumn(int(rows[np.argmin(hq.min(axis=1))]), float(hq.min()))
    hphi = (hq * QW) @ BARY
    rx = -(g * j2d[:, None] * gx[:, None] * hphi)
    ry = -(g * j2d[:, None] * gy[:, None] * hphi)
    if patm is not None:
        pa = np.asarray(patm)[rows]
        rx = rx - j2d[:, None] * (pa * mesh.dphx[rows]).sum(1)[:, None] * hphi / p.rho0
        ry = ry - j2d[:, None] * (pa * mesh.dphy[rows]).sum(1)[:, None] * hphi / p.rho0
    for k in range(3):
        tr, ex, nx, ny = _edge_states(st, mesh, rows, k, eta_bc)
        c = _celerity(tr, ex, g)
        hm = 0.5 * ((tr["e"] - tr["b"]) + (ex["e"] - ex["b"]))
        de = 0.5 * (tr["e"] - ex["e"])
        _edge_scatter(rx, k, -(g * nx * hm * de) + c * 0.5 * (tr["x"] - ex["x"]), mesh.elen[rows, k])
        _edge_scatter(ry, k, -(g * ny * hm * de) + c * 0.5 * (tr["y"] - ex["y"]), mesh.elen[rows, k])
    if f3d2d is not None:
        rx = rx + f3d2d[rows, :, 0]
        ry = ry + f3d2d[rows, :, 1]
    return np.stack([rx, ry], -1)


def tendencies(st, mesh, p, els=None, f3d2d=None, source=None, patm=None, eta_bc=None):
    """external2d.py:259-268."""
    rows = _rows(mesh, els)
    j2d = mesh.j2d[rows]
    re = free_surface_residual(st, mesh, p, rows, source=source, eta_bc=eta_bc)
    rq = momentum_residual(st, mesh, p, rows, f3d2d=f3d2d, patm=patm, eta_bc=eta_bc)
    return mh_inv_apply(re, j2d), mh_inv_apply(rq[..., 0], j2d), mh_inv_apply(rq[..., 1], j2d)


def cfl_ratio(st, mesh, p, dt2d):
    """external2d.py:271-283."""
    h = st.eta - mesh.b
    if np.any(h <= 0.0):
        raise DryColumn(int(np.argmin(h.min(axis=1))), float(h.min()))
    cmax = float(np.sqrt(p.g * h.max()))
    r = dt2d * cmax / mesh.min_edge
    if r > 1.0 / 3.0:
        raise CflViolation(f"dt2d = {dt2d:g} gives c dt / dx = {r:.3f} > 1/3")
    return r


def S2(eta, qx, qy, t=0.0):
    return SimpleNamespace(eta=eta, qx=qx, qy=qy, t=t)


def subcycle(st, mesh, p, m, dt, f3d2d=None, source=None, patm=None, eta_bc=None):
    """external2d.py:296-353: m SSP-RK3 substeps, Qbar and F2D.

    Returns (state, qbar_x, qbar_y, f2d_x, f2d_y).
    """
    cfl_ratio(st, mesh, p, dt)
    s = S2(st.eta.copy(), st.qx.copy(), st.qy.copy(), st.t)
    q0x, q0y = s.qx.copy(), s.qy.copy()
    qbx, qby = np.zeros_like(s.qx), np.zeros_like(s.qy)

    def rhs(x):
        return tendencies(x, mesh, p, f3d2d=f3d2d, source=source, patm=patm, eta_bc=eta_bc)
    for _ in range(m):
        e0, x0, y0, t0 = s.eta, s.qx, s.qy, s.t
        d = rhs(s)
        s1 = S2(e0 + dt * d[0], x0 + dt * d[1], y0 + dt * d[2], t0 + dt)
        d = rhs(s1)
        s2 = S2(0.75 * e0 + 0.25 * (s1.eta + dt * d[0]), 0.75 * x0 + 0.25 * (s1.qx + dt * d[1]),
                0.75 * y0 + 0.25 * (s1.qy + dt * d[2]), t0 + 0.5 * dt)
        d = rhs(s2)
        s = S2(e0 / 3.0 + (2.0 / 3.0) * (s2.eta + dt * d[0]), x0 / 3.0 + (2.0 / 3.0) * (s2.qx + dt * d[1]),
               y0 / 3.0 + (2.0 / 3.0) * (s2.qy + dt * d[2]), t0 + dt)
        qbx += s.qx
        qby += s.qy
    qbx /= m
    qby /= m
    T = m * dt
    fx, fy = (s.qx - q0x) / T, (s.qy - q0y) / T
    if f3d2d is not None:
        fx = fx - mh_inv_apply(f3d2d[:, :, 0], mesh.j2d)
        fy = fy - mh_inv_apply(f3d2d[:, :, 1], mesh.j2d)
    return s, qbx, qby, fx, fy


def diagnostics(st, mesh, p):
    """external2d.py:361-380."""
    hq = (st.eta - mesh.b) @ BARY.T
    eq, xq, yq = st.eta @ BARY.T, st.qx @ BARY.T, st.qy @ BARY.T
    dens = 0.5 * p.g * eq ** 2 + 0.5 * (xq ** 2 + yq ** 2) / hq
    return {"t": st.t,
            "total_volume": float(mh_apply(st.eta - mesh.b, mesh.j2d).sum()),
            "total_energy": float((mesh.j2d[:, None] * dens * QW).sum()),
            "eta_min": float(st.eta.min()), "eta_max": float(st.eta.max())}


def diagnostics_2d(eta, qx, qy, mesh, g):
    """external2d.py:366-380: total volume (exact P1 integral of eta - b), quadrature energy, eta range."""
    h_q = (eta - mesh.b) @ BARY.T
    eta_q, qx_q, qy_q = eta @ BARY.T, qx @ BARY.T, qy @ BARY.T
    dens = 0.5 * g * eta_q ** 2 + 0.5 * (qx_q ** 2 + qy_q ** 2) / h_q
    return {"total_volume": float(mh_apply(eta - mesh.b, mesh.j2d).sum()),
            "total_energy": float((mesh.j2d[:, None] * dens * QW[None, :]).sum()),
            "eta_min": float(eta.min()), "eta_max": float(eta.max())}

"""Internal (3D) mode restatement (prismdg/internal3d.py).  Oracle / test infrastructure only.

Prism fields are (P, 6[, nc]) with p = c * L + l (layer 0 = surface); nodes
0-2 top face, 3-5 bottom face.  `grid` is any object with the ColumnGrid
attributes (mesh, eta, jz, dzmid, djz, dztop, dzbot, n_layers, n_prisms).
"""
import numpy as np

from paper_2605_16082_b200.errors import ZeroPivot
from .colsolve import Banded, lu6, lu6_solve, sweep_r, sweep_w
from .ext2d import mh_apply, nbr_trace, own_trace
from .geom import total_thickness
from .tables import BARY, DPHIZ, DV, ES, EV0, EV1, MH, PHI12, QW, VS, W12, ZQP, ZQW, penalty_sigma


def _cols(grid, els):
    return np.arange(grid.mesh.nt) if els is None else np.asarray(els)


def _cv(f, grid):
    """(P, ...) -> (nt, L, ...)."""
    f = np.asarray(f)
    return f.reshape((grid.mesh.nt, grid.n_layers) + f.shape[1:])


def _hq(c3):
    return c3 @ BARY.T


def _tensor_pts(f6):
    """(..., 6) nodal -> (..., 2v, 6q) at the 12 tensor points (internal3d.py:83-90)."""
    t, b = _hq(f6[..., 0:3]), _hq(f6[..., 3:6])
    return VS[:, 0][:, None] * t[..., None, :] + VS[:, 1][:, None] * b[..., None, :]


def _lev_grad(f6, dx, dy):
    """iso-zeta gradient per level (internal3d.py:98-106): (..., 2lev, 2d)."""
    out = []
    for lev in range(2):
        s = f6[..., 3 * lev:3 * lev + 3]
        out.append(np.stack([(s * dx).sum(-1), (s * dy).sum(-1)], -1))
    return np.stack(out, -2)


def _metric(grid, cols):
    """(jzq (n,L,6), mid2 (n,L,2v,2), m_h (n,L,2v,6q,2)) -- internal3d.py:413-421."""
    jzq = _hq(_cv(grid.jz, grid)[cols])
    mid2 = _cv(grid.dzmid, grid)[cols][:, :, None, :] + ZQP[None, None, :, None] * _cv(grid.djz, grid)[cols][:, :, None, :]
    m_h = -mid2[:, :, :, None, :] / jzq[:, :, None, :, None]
    return jzq, mid2, m_h


# ----------------------------------------------------------------------------- mass

def prism_mass(grid, els=None):
    """internal3d.py:114-123: 6x6 mass via the 12-point rule, measure J2D Jz."""
    cols = _cols(grid, els)
    meas = grid.mesh.j2d[cols][:, None, None] * _hq(_cv(grid.jz, grid)[cols])
    blk = np.einsum("vq,nlq,vqi,vqj->nlij", W12, meas, PHI12, PHI12)
    out = np.zeros((grid.mesh.nt, grid.n_layers, 6, 6))
    out[cols] = blk
    return out.reshape(-1, 6, 6)


def mass_apply(mass, f):
    """internal3d.py:126-131."""
    f = np.asarray(f)
    return np.einsum("pij,pj->pi", mass, f) if f.ndim == 2 else np.einsum("pij,pjc->pic", mass, f)


def mass_solve(mass, rhs, grid, els=None):
    """internal3d.py:134-151: per-prism unpivoted LU, ZeroPivot(layer, k)."""
    cols = _cols(grid, els)
    f = np.asarray(rhs)
    vec = f.ndim == 3
    f3 = f if vec else f[..., None]
    out = np.zeros_like(f3)
    mv, fv, ov = _cv(mass, grid), _cv(f3, grid), _cv(out, grid)
    for l in range(grid.n_layers):
        a = mv[cols, l].copy()
        b = fv[cols, l].copy()
        lu6(a, l)
        ov[cols, l] = lu6_solve(a, b)
    return out if vec else out[..., 0]


# ----------------------------------------------------------------------------- transport

def project_transport(grid, ux, uy, els=None, mass=None):
    """internal3d.py:164-181: M q = <phi Jz u J2D Jz>."""
    cols = _cols(grid, els)
    if mass is None:
        mass = prism_mass(grid, els)
    jzq = _hq(_cv(grid.jz, grid)[cols])
    meas = grid.mesh.j2d[cols][:, None, None] * jzq * jzq
    uq = np.stack([_tensor_pts(_cv(ux, grid)[cols]), _tensor_pts(_cv(uy, grid)[cols])], -1)
    rhs = np.zeros((grid.mesh.nt, grid.n_layers, 6, 2))
    rhs[cols] = np.einsum("vq,nlq,nlvqc,vqi->nlic", W12, meas, uq, PHI12)
    return mass_solve(mass, rhs.reshape(-1, 6, 2), grid, els)


def column_sum(f, grid):
    """internal3d.py:184-187: sum over both levels of every layer."""
    fv = _cv(f, grid)
    return fv[:, :, 0:3].sum(axis=1) + fv[:, :, 3:6].sum(axis=1)


def consistent_transport(grid, q, qbx, qby, els=None):
    """internal3d.py:190-208: qbar = q + Jz (Qbar - sum_col q) / H."""
    cols = _cols(grid, els)
    Qb = np.stack([np.asarray(qbx), np.asarray(qby)], -1)
    mis = (Qb - column_sum(q, grid)) / total_thickness(grid)[..., None]
    out = np.zeros_like(np.asarray(q))
    qv, ov, jz = _cv(q, grid), _cv(out, grid), _cv(grid.jz, grid)
    for lev in range(2):
        s = slice(3 * lev, 3 * lev + 3)
        ov[cols, :, s] = qv[cols, :, s] + jz[cols][..., None] * mis[cols][:, None]
    return out


# ----------------------------------------------------------------------------- lateral faces

def _pair(x0, x1, mirror):
    a, b = (1, 0) if mirror else (0, 1)
    return x0[..., None] * ES[:, a] + x1[..., None] * ES[:, b]


def lat_trace(f6, grid, rows, k, mirror):
    """internal3d.py:229-258: (n, L, 2v, 2h[, c]) values on edge-k lateral faces."""
    mesh = grid.mesh
    fv = _cv(f6, grid)
    if not mirror:
        src, i0, i1 = fv[rows], EV0[k], EV1[k]
        t0, t1, b0, b1 = src[:, :, i0], src[:, :, i1], src[:, :, 3 + i0], src[:, :, 3 + i1]
    else:
        e2 = np.maximum(mesh.nbr[rows, k], 0)
        k2 = mesh.nbrk[rows, k]
        src = fv[e2]
        r = np.arange(rows.size)
        t0, t1 = src[r, :, EV0[k2]], src[r, :, EV1[k2]]
        b0, b1 = src[r, :, 3 + EV0[k2]], src[r, :, 3 + EV1[k2]]
    comp = np.asarray(f6).ndim == 3
    if comp:
        t0, t1, b0, b1 = (np.moveaxis(a, -1, 0) for a in (t0, t1, b0, b1))
    ht, hb = _pair(t0, t1, mirror), _pair(b0, b1, mirror)
    out = VS[:, 0][:, None] * ht[..., None, :] + VS[:, 1][:, None] * hb[..., None, :]
    return np.moveaxis(out, 0, -1) if comp else out


def lat_gather_add(acc, rows, k, x, jedge, sign):
    """internal3d.py:261-272: acc[rows, :, node] += sign Jedge sum_vh w phi x."""
    for lev in range(2):
        for hn in range(2):
            node = 3 * lev + (EV0[k] if hn == 0 else EV1[k])
            coef = (VS[:, lev] * ZQW)[:, None] * (ES[:, hn] * ZQW)[None, :]
            acc[rows, :, node] += sign * jedge[:, None] * np.einsum("vh,nlvh->nl", coef, x)


def _dup(c3):
    return np.concatenate([c3, c3], axis=1)


def lateral_flux_factor(grid, q, p, els=None):
    """internal3d.py:275-314: n.{q} + {Jz/H} max(c) [[eta]] on interior faces."""
    cols = _cols(grid, els)
    mesh, L = grid.mesh, grid.n_layers
    eta, b = grid.eta, mesh.b
    jzh = grid.jz / np.repeat(eta - b, L, axis=0)
    out = np.zeros((mesh.nt, L, 3, 2, 2))
    for k in range(3):
        rows = cols[mesh.btag[cols, k] == 0]
        if rows.size == 0:
            continue
        e2, k2 = mesh.nbr[rows, k], mesh.nbrk[rows, k]
        ei, ee = own_trace(eta, rows, k), nbr_trace(eta, e2, k2)
        hi, he = ei - own_trace(b, rows, k), ee - nbr_trace(b, e2, k2)
        stab = 0.5 * (ei - ee) * np.maximum(np.sqrt(p.g * hi), np.sqrt(p.g * he))
        qm = 0.5 * (lat_trace(q, grid, rows, k, False) + lat_trace(q, grid, rows, k, True))
        jm = 0.5 * (lat_trace(_dup(jzh), grid, rows, k, False) + lat_trace(_dup(jzh), grid, rows, k, True))
        out[rows, :, k] = (mesh.enx[rows, k][:, None, None, None] * qm[..., 0]
                           + mesh.eny[rows, k][:, None, None, None] * qm[..., 1]
                           + jm * stab[:, None, None, :])
    return out


# ----------------------------------------------------------------------------- baroclinic head

def compute_r(grid, rho, p, els=None):
    """internal3d.py:327-405: weak RHS of the head, then the top-down sweep."""
    cols = _cols(grid, els)
    mesh, L, g = grid.mesh, grid.n_layers, p.g
    j2d = mesh.j2d[cols]
    rv = _cv(rho, grid)
    dx, dy = mesh.dphx[cols], mesh.dphy[cols]
    jzq, mid2, m_h = _metric(grid, cols)
    gl = _lev_grad(rv[cols], dx[:, None, :], dy[:, None, :])            # (n, L, lev, d)
    giso = np.einsum("vm,nlmd->nlvd", VS, gl)[:, :, :, None, :]         # (n, L, v, 1, d)
    dzr = 0.5 * (_hq(rv[cols][..., 0:3]) - _hq(rv[cols][..., 3:6]))     # (n, L, q)
    gfull = giso + m_h * dzr[:, :, None, :, None]
    meas = j2d[:, None, None] * jzq
    acc = np.zeros((mesh.nt, L, 6, 2))
    acc[cols] = -g * np.einsum("vq,nlq,vqi,nlvqd->nlid", W12, meas, PHI12, gfull)
    if L > 1:
        jump = 0.5 * (rv[cols][:, 1:, 0:3] - rv[cols][:, :-1, 3:6])
        fint = jump @ MH.T
        dzf = _cv(grid.dztop, grid)[cols][:, 1:]
        acc[cols, 1:, 0:3] += 2.0 * g * j2d[:, None, None, None] * (-dzf[:, :, None, :]) * fint[..., None]
    jz6 = _dup(grid.jz)
    for k in range(3):
        rows = cols[mesh.btag[cols, k] == 0]
        if rows.size == 0:
            continue
        dr = 0.5 * (lat_trace(rho, grid, rows, k, False) - lat_trace(rho, grid, rows, k, True))
        jm = 0.5 * (lat_trace(jz6, grid, rows, k, False) + lat_trace(jz6, grid, rows, k, True))
        je = 0.5 * mesh.elen[rows, k]
        for d, nrm in ((0, mesh.enx), (1, mesh.eny)):
            lat_gather_add(acc[..., d], rows, k, nrm[rows, k][:, None, None, None] * dr * jm, je, g)
    ex = (grid.eta[cols] * dx).sum(1)
    ey = (grid.eta[cols] * dy).sum(1)
    mr = mh_apply(rv[cols, 0, 0:3], j2d)
    acc[cols, 0, 0:3, 0] -= g * mr * ex[:, None]
    acc[cols, 0, 0:3, 1] -= g * mr * ey[:, None]
    out = np.zeros((mesh.nt, L, 6, 2))
    out[cols] = sweep_r(acc[cols], j2d)
    return out.reshape(-1, 6, 2)


# ----------------------------------------------------------------------------- vertical velocities

def _iso_div(acc, cols, s, dx, dy, j2d):
    for lev in range(2):
        for i in range(3):
            acc[cols, :, 3 * lev + i] += j2d[:, None] * (dx[:, i, None] * s[:, :, lev, 0] + dy[:, i, None] * s[:, :, lev, 1])


def _lat_factor_terms(acc, grid, cols, factor):
    mesh = grid.mesh
    for k in range(3):
        rows = cols[mesh.btag[cols, k] == 0]
        if rows.size:
            lat_gather_add(acc, rows, k, factor[rows, :, k], 0.5 * mesh.elen[rows, k], -1.0)


def compute_w(grid, q, ux, uy, p, factor, els=None):
    """internal3d.py:434-502: continuity RHS then the bottom-up sweep."""
    cols = _cols(grid, els)
    mesh, L = grid.mesh, grid.n_layers
    j2d, dx, dy = mesh.j2d[cols], mesh.dphx[cols], mesh.dphy[cols]
    jzq, mid2, m_h = _metric(grid, cols)
    qv = _cv(q, grid)[cols]
    qq = np.einsum("nljc,vqj->nlvqc", qv, PHI12)
    acc = np.zeros((mesh.nt, L, 6))
    _iso_div(acc, cols, np.einsum("vq,vm,nlvqc->nlmc", W12, VS, qq), dx, dy, j2d)
    met = np.einsum("vq,nlvq,qi->nli", W12, (qq * m_h).sum(-1), BARY)
    acc[cols, :, 0:3] += j2d[:, None, None] * DV[0] * met
    acc[cols, :, 3:6] += j2d[:, None, None] * DV[1] * met
    ut = np.einsum("nljc,qj->nlqc", qv[:, :, 0:3], BARY) / jzq[..., None]
    ub = np.einsum("nljc,qj->nlqc", qv[:, :, 3:6], BARY) / jzq[..., None]
    mt, mb = ut.copy(), ub.copy()
    mt[:, 1:] = 0.5 * (ut[:, 1:] + ub[:, :-1])
    mb[:, :-1] = 0.5 * (ub[:, :-1] + ut[:, 1:])
    ft = np.einsum("nlqc,nlc->nlq", mt, _cv(grid.dztop, grid)[cols])
    fb = np.einsum("nlqc,nlc->nlq", mb, _cv(grid.dzbot, grid)[cols])
    acc[cols, :, 0:3] += j2d[:, None, None] * np.einsum("q,nlq,qi->nli", QW, ft, BARY)
    acc[cols, :, 3:6] -= j2d[:, None, None] * np.einsum("q,nlq,qi->nli", QW, fb, BARY)
    _lat_factor_terms(acc, grid, cols, factor)
    bx, by = (mesh.b[cols] * dx).sum(1), (mesh.b[cols] * dy).sum(1)
    uxb, uyb = _cv(ux, grid)[cols, L - 1, 3:6], _cv(uy, grid)[cols, L - 1, 3:6]
    acc[cols, L - 1, 3:6] += mh_apply(uxb * bx[:, None] + uyb * by[:, None], j2d)
    out = np.zeros((mesh.nt, L, 6))
    out[cols] = sweep_w(acc[cols], j2d)
    return out.reshape(-1, 6)


def compute_wtilde(grid, qbar, factor, els=None):
    """internal3d.py:505-541: iso-zeta volume term + lateral factor, bed-anchored sweep."""
    cols = _cols(grid, els)
    mesh, L = grid.mesh, grid.n_layers
    j2d, dx, dy = mesh.j2d[cols], mesh.dphx[cols], mesh.dphy[cols]
    qq = np.einsum("nljc,vqj->nlvqc", _cv(qbar, grid)[cols], PHI12)
    acc = np.zeros((mesh.nt, L, 6))
    _iso_div(acc, cols, np.einsum("vq,vm,nlvqc->nlmc", W12, VS, qq), dx, dy, j2d)
    _lat_factor_terms(acc, grid, cols, factor)
    out = np.zeros((mesh.nt, L, 6))
    out[cols] = sweep_w(acc[cols], j2d)
    return out.reshape(-1, 6)


# ----------------------------------------------------------------------------- horizontal RHS

W1 = QW @ BARY                                           # sum_q QW BARY_i (the P1 face moments)


def horizontal_diffusion(grid, f, kh, kv, els=None, wall_mirror=True):
    """internal3d.py:549-692 (_horizontal_diffusion), PATCHED ORACLE: the reference raises at
    :665 and :676 (two (n,) per-edge arrays broadcast without their trailing axes; SURVEY.md
    section 0.3); this is the function with those broadcasts as evidently intended
    (oracle/refops.patch_horizontal_diffusion, pinned by tests/golden/hdiff.npz).

    Restated in closed form.  With gv the iso-zeta gradient at the vertical points, mid2 = -m_h Jz
    (internal3d.py:413-421) and dz = 0.5 (f_top - f_bot) per corner:
      volume   sum_vq QW Jz gh = gv sum QW Jz - mid2 sum QW dz against grad_h phi; the m_h parts of
               the phi_z test (:603-611) cancel to +kh J2D DV (sum_v gv . mid2) W1
      top/bottom faces: the -kh |grad z_f|^2 dz/Jz remainder cancels the metric part of n.D.grad
               (:624-636), leaving -kh J2D grad_iso . grad z_f, constant over the face
      lateral  kh Jz n.gv - kh (n.mid2) dz per side, mean of both sides, plus the interior penalty
               sigma kh {Jz} [[f]] (:644-678); walls: the penalty on the normal velocity only when
               wall_mirror (:679-691).
    f: (P, 6, nc) -> (nt, L, 6, nc) residual (rows outside els zero)."""
    cols = _cols(grid, els)
    mesh, L = grid.mesh, grid.n_layers
    f = np.asarray(f, dtype=float)
    nc = f.shape[-1]
    acc = np.zeros((mesh.nt, L, 6, nc))
    if kh == 0.0 and kv == 0.0:
        return acc
    fv = _cv(f, grid)                                                   # (nt, L, 6, c)
    dxa, dya = mesh.dphx[:, None, :, None], mesh.dphy[:, None, :, None]
    giso = np.stack([np.stack([(fv[:, :, 3 * lev:3 * lev + 3] * dxa).sum(2),
                               (fv[:, :, 3 * lev:3 * lev + 3] * dya).sum(2)], 2) for lev in range(2)], 2)
    gv_all = np.einsum("vm,nlmdc->nlvdc", VS, giso)                     # (nt, L, v, d, c)
    allc = np.arange(mesh.nt)
    jzq_all, mid2_all, _ = _metric(grid, allc)                           # mid2: (nt, L, v, d)
    dz_all = 0.5 * (fv[:, :, 0:3] - fv[:, :, 3:6])                     # (nt, L, 3, c)
    j2d = mesh.j2d[cols]
    dx, dy = mesh.dphx[cols], mesh.dphy[cols]
    gv, mid2, jzq, dz = gv_all[cols], mid2_all[cols], jzq_all[cols], dz_all[cols]

    # volume
    A = jzq @ QW                                                        # (n, L)
    B = np.einsum("q,qj,nljc->nlc", QW, BARY, dz)                       # (n, L, c)
    sv = np.einsum("vm,nlvdc->nlmdc", VS, gv * A[:, :, None, None, None]
                   - mid2[..., None] * B[:, :, None, None, :])
    for lev in range(2):
        for i in range(3):
            acc[cols, :, 3 * lev + i] -= kh * j2d[:, None, None] * (dx[:, None, i, None] * sv[:, :, lev, 0]
                                                                    + dy[:, None, i, None] * sv[:, :, lev, 1])
    gm = np.einsum("nlvdc,nlvd->nlc", gv, mid2)
    for lev in range(2):
        acc[cols, :, 3 * lev:3 * lev + 3] += (kh * DV[lev]) * j2d[:, None, None, None] * W1[None, None, :, None] \
            * gm[:, :, None, :]

    # interior top / bottom faces between layers l-1 and l
    if L > 1:
        dzt = _cv(grid.dztop, grid)[cols][:, 1:]                         # (n, L-1, d)
        dzb = _cv(grid.dzbot, grid)[cols][:, :-1]
        gsi = giso[cols]
        f_lo = -kh * np.einsum("nldc,nld->nlc", gsi[:, 1:, 0], dzt)
        f_hi = -kh * np.einsum("nldc,nld->nlc", gsi[:, :-1, 1], dzb)
        face = (0.5 * j2d[:, None, None] * (f_lo + f_hi))[:, :, None, :] * W1[None, None, :, None]
        acc[cols, 1:, 0:3] += face
        acc[cols, :-1, 3:6] -= face

    # lateral faces
    jz6 = _dup(grid.jz)
    dz6 = np.concatenate([dz_all, dz_all], axis=2).reshape(-1, 6, nc)
    for k in range(3):
        tag = mesh.btag[cols, k]
        je_all = 0.5 * mesh.elen[cols, k]
        rows = cols[tag == 0]
        if rows.size:
            e2 = mesh.nbr[rows, k]
            nx, ny = mesh.enx[rows, k], mesh.eny[rows, k]
            jzi, jze = lat_trace(jz6, grid, rows, k, False), lat_trace(jz6, grid, rows, k, True)   # (n, L, v, h)
            dzi, dze = lat_trace(dz6, grid, rows, k, False), lat_trace(dz6, grid, rows, k, True)   # (n, L, v, h, c)

            def side(src, jt, dt):
                ng = nx[:, None, None, None] * gv_all[src][:, :, :, 0] + ny[:, None, None, None] * gv_all[src][:, :, :, 1]
                nm = nx[:, None, None] * mid2_all[src][..., 0] + ny[:, None, None] * mid2_all[src][..., 1]
                # (n, L, v, h, c): kh Jz (n.gv - (n.mid2) dz / Jz(v=0))
                return kh * jt[..., None] * (ng[:, :, :, None, :] - nm[:, :, :, None, None] * dt
                                             / jt[:, :, :1, :, None])

            mean = 0.5 * (side(rows, jzi, dzi) + side(e2, jze, dze))
            sig = penalty_sigma(0.5 * mesh.j2d[rows] / mesh.elen[rows, k], 0.5 * mesh.j2d[e2] / mesh.elen[rows, k], 3)
            pen = sig[:, None, None, None] * kh * 0.5 * (jzi + jze) * 0.5
            tri, tre = lat_trace(f, grid, rows, k, False), lat_trace(f, grid, rows, k, True)
            je = 0.5 * mesh.elen[rows, k]
            for c in range(nc):
                lat_gather_add(acc[..., c], rows, k, mean[..., c], je, 1.0)
                lat_gather_add(acc[..., c], rows, k, pen * (tri[..., c] - tre[..., c]), je, -1.0)
        wr = cols[tag != 0]
        if wall_mirror and wr.size:
            nx, ny = mesh.enx[wr, k], mesh.eny[wr, k]
            tri = lat_trace(f, grid, wr, k, False)
            jzi = lat_trace(jz6, grid, wr, k, False)
            ln = 0.5 * mesh.j2d[wr] / mesh.elen[wr, k]
            pen = penalty_sigma(ln, ln, 3)[:, None, None, None] * kh * jzi
            un = nx[:, None, None, None] * tri[..., 0] + ny[:, None, None, None] * tri[..., 1]
            je = je_all[tag != 0]
            lat_gather_add(acc[..., 0], wr, k, pen * un * nx[:, None, None, None], je, -1.0)
            lat_gather_add(acc[..., 1], wr, k, pen * un * ny[:, None, None, None], je, -1.0)
    return acc


def horizontal_rhs(grid, ux, uy, q_adv, factor, r, mass, p, els=None):
    """internal3d.py:695-751 (explicit viscosity: the patched horizontal_diffusion above)."""
    cols = _cols(grid, els)
    mesh, L = grid.mesh, grid.n_layers
    j2d, dx, dy = mesh.j2d[cols], mesh.dphx[cols], mesh.dphy[cols]
    U = np.stack([np.asarray(ux), np.asarray(uy)], -1)
    acc = np.zeros((mesh.nt, L, 6, 2))
    uq = np.einsum("nljc,vqj->nlvqc", _cv(U, grid)[cols], PHI12)
    qq = np.einsum("nljd,vqj->nlvqd", _cv(q_adv, grid)[cols], PHI12)
    s = np.einsum("vq,vm,nlvqc,nlvqd->nlmcd", W12, VS, uq, qq)
    for lev in range(2):
        for i in range(3):
            acc[cols, :, 3 * lev + i] += j2d[:, None, None] * (dx[:, None, i, None] * s[:, :, lev, :, 0]
                                                               + dy[:, None, i, None] * s[:, :, lev, :, 1])
    for k in range(3):
        rows = cols[mesh.btag[cols, k] == 0]
        if rows.size == 0:
            continue
        fac = factor[rows, :, k]
        up = np.where(fac[..., None] >= 0.0, lat_trace(U, grid, rows, k, False), lat_trace(U, grid, rows, k, True))
        for c in range(2):
            lat_gather_add(acc[..., c], rows, k, up[..., c] * fac, 0.5 * mesh.elen[rows, k], -1.0)
    acc += horizontal_diffusion(grid, U, p.kappa_h, p.kappa_v, els, wall_mirror=True)
    out = acc.reshape(-1, 6, 2)
    if p.f != 0.0:
        mu = mass_apply(mass, U)
        out[..., 0] += p.f * mu[..., 1]
        out[..., 1] -= p.f * mu[..., 0]
    out -= mass_apply(mass, np.asarray(r)) / p.rho0
    return out


def tracer_horizontal_rhs(grid, tr, qbar, factor, p, els=None):
    """internal3d.py:754-792 (explicit diffusion: the patched horizontal_diffusion above)."""
    cols = _cols(grid, els)
    mesh, L = grid.mesh, grid.n_layers
    j2d, dx, dy = mesh.j2d[cols], mesh.dphx[cols], mesh.dphy[cols]
    acc = np.zeros((mesh.nt, L, 6))
    tq = np.einsum("nlj,vqj->nlvq", _cv(tr, grid)[cols], PHI12)
    qq = np.einsum("nljd,vqj->nlvqd", _cv(qbar, grid)[cols], PHI12)
    _iso_div(acc, cols, np.einsum("vq,vm,nlvq,nlvqd->nlmd", W12, VS, tq, qq), dx, dy, j2d)
    for k in range(3):
        rows = cols[mesh.btag[cols, k] == 0]
        if rows.size == 0:
            continue
        fac = factor[rows, :, k]
        up = np.where(fac >= 0.0, lat_trace(tr, grid, rows, k, False), lat_trace(tr, grid, rows, k, True))
        lat_gather_add(acc, rows, k, up * fac, 0.5 * mesh.elen[rows, k], -1.0)
    acc += horizontal_diffusion(grid, np.asarray(tr)[..., None], p.nu_h, p.nu_v, els, wall_mirror=False)[..., 0]
    return acc.reshape(-1, 6)


def stress_rhs(grid, tsx, tsy, cd, ux, uy, els=None):
    """internal3d.py:919-934."""
    cols = _cols(grid, els)
    mesh, L = grid.mesh, grid.n_layers
    j2d = mesh.j2d[cols]
    acc = np.zeros((mesh.nt, L, 6, 2))
    acc[cols, 0, 0:3, 0] += j2d[:, None] / 6.0 * tsx
    acc[cols, 0, 0:3, 1] += j2d[:, None] / 6.0 * tsy
    if cd != 0.0:
        bx, by = _cv(ux, grid)[cols, L - 1, 3:6], _cv(uy, grid)[cols, L - 1, 3:6]
        sp = np.sqrt(bx ** 2 + by ** 2)
        acc[cols, L - 1, 3:6, 0] += mh_apply(-cd * sp * bx, j2d)
        acc[cols, L - 1, 3:6, 1] += mh_apply(-cd * sp * by, j2d)
    return acc.reshape(-1, 6, 2)


# ----------------------------------------------------------------------------- vertical operator

def _face(w, a, b):
    """sum_q w[..., q] a[q, i] b[q, j] -> (..., 3 or 6, 3 or 6)."""
    return np.einsum("q,...q,qi,qj->...ij", QW, w, a, b)


def assemble_vertical_operator(grid, wtilde, w_m, kh, kv, els=None, n0=5.0, order=1):
    """internal3d.py:800-899: banded A (d, u, w) per column."""
    cols = _cols(grid, els)
    L = grid.n_layers
    n = cols.size
    j2d = grid.mesh.j2d[cols]
    jzq, mid2, _ = _metric(grid, cols)
    d = np.zeros((n, L, 6, 6))
    u = np.zeros((n, L, 3, 6))
    w = np.zeros((n, L, 3, 6))
    wt, wm = _cv(wtilde, grid)[cols], _cv(w_m, grid)[cols]
    spd = np.einsum("nlj,vqj->nlvq", wt - wm, PHI12)
    d += np.einsum("vq,nlvq,qi,vqj->nlij", W12, j2d[:, None, None, None] * spd, DPHIZ, PHI12)
    ki = kv + kh * (mid2 ** 2).sum(-1)
    d -= np.einsum("vq,nlv,nlq,qi,qj->nlij", W12, ki, j2d[:, None, None] / jzq, DPHIZ, DPHIZ)
    wtt = np.einsum("nlj,qj->nlq", wt[:, :, 0:3], BARY)
    wmt = np.einsum("nlj,qj->nlq", wm[:, :, 0:3], BARY)
    wmb = np.einsum("nlj,qj->nlq", wm[:, :, 3:6], BARY)
    d[:, 0, 0:3, 0:3] -= _face(j2d[:, None] * (wtt[:, 0] - wmt[:, 0]), BARY, BARY)
    if L > 1:
        st = wtt[:, 1:] - wmt[:, 1:]
        d[:, 1:, 0:3, 0:3] -= _face(j2d[:, None, None] * np.where(st >= 0.0, st, 0.0), BARY, BARY)
        u[:, 1:, :, 3:6] -= _face(j2d[:, None, None] * np.where(st < 0.0, st, 0.0), BARY, BARY)
        sb = wtt[:, 1:] - wmb[:, :-1]
        d[:, :-1, 3:6, 3:6] += _face(j2d[:, None, None] * np.where(sb <= 0.0, sb, 0.0), BARY, BARY)
        w[:, :-1, :, 0:3] += _face(j2d[:, None, None] * np.where(sb > 0.0, sb, 0.0), BARY, BARY)
        dzt, dzb = _cv(grid.dztop, grid)[cols], _cv(grid.dzbot, grid)[cols]
        kt = kv + kh * (dzt ** 2).sum(-1)
        kb = kv + kh * (dzb ** 2).sum(-1)
        hi = 0.5 * j2d[:, None, None] * kt[:, 1:, None] / jzq[:, 1:]      # face seen from below (layer l top)
        he = 0.5 * j2d[:, None, None] * kb[:, :-1, None] / jzq[:, :-1]    # face seen from above (layer l-1 bottom)
        d[:, 1:, 0:3, :] += _face(hi, BARY, DPHIZ)
        u[:, 1:] += _face(he, BARY, DPHIZ)
        d[:, :-1, 3:6, :] -= _face(he, BARY, DPHIZ)
        w[:, :-1] -= _face(hi, BARY, DPHIZ)
        hgt = 2.0 * _cv(grid.jz, grid)[cols].mean(axis=2)
        sig = penalty_sigma(hgt[:, 1:], hgt[:, :-1], 3, n0, order)
        nz = 1.0 / np.sqrt(1.0 + (dzt[:, 1:] ** 2).sum(-1))
        mf = np.einsum("q,qi,qj->ij", QW, BARY, BARY)
        pf = (sig * np.maximum(kt[:, 1:], kb[:, :-1]) * nz * j2d[:, None])[..., None, None]
        d[:, 1:, 0:3, 0:3] -= 0.5 * pf * mf
        u[:, 1:, :, 3:6] += 0.5 * pf * mf
        d[:, :-1, 3:6, 3:6] -= 0.5 * pf * mf
        w[:, :-1, :, 0:3] += 0.5 * pf * mf
    return Banded(d, u, w)


def build_implicit(mass, op, dt, grid, els=None):
    """internal3d.py:902-906: M - dt A."""
    cols = _cols(grid, els)
    mv = _cv(mass, grid)[cols]
    return Banded(mv - dt * op.d, -dt * op.u, -dt * op.w)


def scatter_columns(x, grid, els=None):
    """internal3d.py:909-916."""
    cols = _cols(grid, els)
    x = np.asarray(x)
    shape = (grid.n_prisms, 6) if x.ndim == 3 else (grid.n_prisms, 6, x.shape[-1])
    out = np.zeros(shape)
    out.reshape((grid.mesh.nt, grid.n_layers) + shape[1:])[cols] = x
    return out


def budget_3d(grid, mass, ux, uy, tr):
    """internal3d.py:942-951: integrals of 1, u_x, u_y, T against the prism masses; T range."""
    integ = lambda f: float(mass_apply(mass, f).sum())  # noqa: E731
    return {"volume": integ(np.ones((mass.shape[0], 6))), "momentum_x": integ(ux), "momentum_y": integ(uy),
            "tracer_mass": integ(tr), "tracer_min": float(np.min(tr)), "tracer_max": float(np.max(tr))}

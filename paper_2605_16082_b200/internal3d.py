"""Drop-in for prismdg/internal3d.py: the 3D internal mode on the B200.

Same names, signatures, shapes and exceptions as the reference; numpy in ->
numpy out (parity path), torch CUDA in -> torch CUDA out.  Every assembly is
one thread-per-column kernel in csrc/int3d.cu / csrc/columns.cu; the grid's
prism geometry is rebuilt on device from (grid.eta, mesh.b, sigma fractions).

Explicit horizontal viscosity / diffusivity (kappa_h, nu_h != 0) is the
"patched oracle" of _horizontal_diffusion (internal3d.py:549-692): the reference
raises at internal3d.py:665 / :676 for every mesh (two per-edge broadcasts miss
an axis); with those fixed (oracle/refops.py) its output
is tests/golden/hdiff.npz, which csrc/hdiff.cu matches.  Vertical diffusion
(assemble_vertical_operator's kh / kv) is the reference's own.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .columns import _err_check, _err_word
from .device import Arr, c3_in, c3_out, device_mesh, els_dev, p6_in, p6_out, ptr, stream_ptr
from .params import BandedColumnMatrix, PenaltyParams, PhysParams

F64 = torch.float64


def _dm(grid):
    return device_mesh(grid.mesh, grid.n_layers, getattr(grid, "fracs", None))


def _eta(grid, A, dev):
    """grid free surface on device; does not decide the caller's result kind (fields do)."""
    e = grid.eta
    e = e.to(device=dev, dtype=F64) if isinstance(e, torch.Tensor) else torch.as_tensor(np.asarray(e, np.float64),
                                                                                       device=dev)
    return c3_in(e, dev)


def _nsel(dm, el):
    return dm.nt if el is None else el.numel()


def _fac_in(f, nt, L):
    """(nt, L, 3, 2, 2) -> [3][2][2][L][nt]."""
    return f.reshape(nt, L, 3, 2, 2).permute(2, 3, 4, 1, 0).contiguous()


def _fac_out(t):
    return t.permute(4, 3, 0, 1, 2).contiguous()


def _mass_in(mass, nt, L):
    return mass.reshape(nt, L, 36).permute(2, 1, 0).contiguous()


def _mass_out(t, nt, L):
    return t.permute(2, 1, 0).reshape(nt * L, 6, 6).contiguous()


def _zeros(*shape, dev):
    return torch.zeros(shape, dtype=F64, device=dev)


def _add_diffusion(dm, eta, f, nc, kh, el, out, scale=1.0, mode=0):
    """out += scale * _horizontal_diffusion(f) (internal3d.py:549-692, patched; csrc/hdiff.cu).
    Every term carries kh, so kh == 0 adds nothing (the reference returns zeros when kh == kv == 0)."""
    if kh != 0.0:
        _lib.check(_lib.lib().pdg_horizontal_diffusion(dm.h, ptr(eta), ptr(f), nc, float(kh), int(nc == 2),
                                                       float(scale), mode, ptr(el), _nsel(dm, el), ptr(out),
                                                       stream_ptr()), "horizontal_diffusion")


# ----------------------------------------------------------------------------- mass

def prism_mass(grid, els=None):
    """(P, 6, 6) prism masses, rows outside `els` zero (internal3d.py:114-123)."""
    dm = _dm(grid)
    dev, nt, L = dm.device, dm.nt, dm.L
    A = Arr()
    A.numpy = not isinstance(grid.eta, torch.Tensor)
    with torch.cuda.device(dev):
        el = els_dev(els, dev)
        out = _zeros(36, L, nt, dev=dev)
        _lib.check(_lib.lib().pdg_prism_mass(dm.h, ptr(_eta(grid, A, dev)), ptr(el), _nsel(dm, el), ptr(out),
                                             stream_ptr()), "prism_mass")
        return A.out(_mass_out(out, nt, L))


def _mass_dev(mass, A, dev):
    m = A.dev(mass, dev)
    P = m.shape[0]
    return m.reshape(P, 36).t().contiguous(), P


def mass_apply(mass, field):
    """M f per prism (internal3d.py:126-131)."""
    A = Arr()
    dev = torch.device("cuda", torch.cuda.current_device())
    m, P = _mass_dev(mass, A, dev)
    f = A.dev(field, dev)
    vec = f.dim() == 3
    nc = f.shape[2] if vec else 1
    fd = (f.permute(2, 1, 0) if vec else f.t()[None]).contiguous()
    out = torch.empty_like(fd)
    err = _err_word(dev)
    _lib.check(_lib.lib().pdg_mass_op(1, P, nc, 0, ptr(m), ptr(fd), ptr(out), ptr(err), stream_ptr()), "mass_apply")
    res = out.permute(2, 1, 0) if vec else out[0].t()
    return A.out(res.contiguous())


def mass_solve(mass, rhs, grid, els=None):
    """Per-prism unpivoted 6x6 LU solve, ZeroPivot(layer, k) (internal3d.py:134-151)."""
    dm = _dm(grid)
    dev, nt, L = dm.device, dm.nt, dm.L
    A = Arr()
    with torch.cuda.device(dev):
        m = A.dev(mass, dev).reshape(nt, L, 36)
        f = A.dev(rhs, dev)
        vec = f.dim() == 3
        nc = f.shape[2] if vec else 1
        fv = f.reshape(nt, L, 6, nc)
        cols = torch.arange(nt, device=dev) if els is None else els_dev(els, dev).long()
        n = cols.numel()
        ms = m[cols].reshape(n * L, 36).t().contiguous()           # [36][n*L], prism = col*L + l
        # lay the selected prisms out as [..][L][n] so the kernel's layer index is l
        ms = ms.reshape(36, n, L).permute(0, 2, 1).contiguous()
        fs = fv[cols].permute(3, 2, 1, 0).contiguous()              # [nc][6][L][n]
        out = torch.empty_like(fs)
        err = _err_word(dev)
        _lib.check(_lib.lib().pdg_mass_op(L, n, nc, 1, ptr(ms), ptr(fs), ptr(out), ptr(err), stream_ptr()),
                   "mass_solve")
        _err_check(err)
        res = torch.zeros((nt, L, 6, nc), dtype=F64, device=dev)
        res[cols] = out.permute(3, 2, 1, 0)
        res = res.reshape(nt * L, 6, nc)
        return A.out(res if vec else res[..., 0].contiguous())


def integrate_prism(mass, field) -> float:
    """Exact integral of a nodal prism field (internal3d.py:154-156)."""
    r = mass_apply(mass, field)
    return float(r.sum()) if isinstance(r, np.ndarray) else float(r.sum().item())


# ----------------------------------------------------------------------------- transport

def project_transport(grid, ux, uy, els=None, mass=None):
    """q = M^-1 <phi Jz u J2D Jz>, (P, 6, 2) (internal3d.py:164-181)."""
    dm = _dm(grid)
    dev, nt, L = dm.device, dm.nt, dm.L
    A = Arr()
    with torch.cuda.device(dev):
        el = els_dev(els, dev)
        x, y = p6_in(A.dev(ux, dev), nt, L), p6_in(A.dev(uy, dev), nt, L)
        md = None if mass is None else _mass_in(A.dev(mass, dev), nt, L)
        q = _zeros(2, 6, L, nt, dev=dev)
        _lib.check(_lib.lib().pdg_project_transport(dm.h, ptr(_eta(grid, A, dev)), ptr(x), ptr(y), ptr(md), ptr(el),
                                                    _nsel(dm, el), ptr(q), None, None, stream_ptr()), "project")
        dm.raise_errors()
        return A.out(p6_out(q, nt, L))


def column_sum(field, grid):
    """Sum over both levels of every layer, (nt, 3[, nc]) (internal3d.py:184-187)."""
    nt, L = grid.mesh.nt, grid.n_layers
    dev = torch.device("cuda", torch.cuda.current_device())
    A = Arr()
    f = A.dev(field, dev)
    vec = f.dim() == 3
    fd = p6_in(f, nt, L)
    nc = fd.shape[0] if vec else 1
    out = torch.empty((nc, 3, nt), dtype=F64, device=dev)
    _lib.check(_lib.lib().pdg_column_sum(nt, L, nc, ptr(fd), ptr(out), stream_ptr()), "column_sum")
    return A.out(c3_out(out) if vec else c3_out(out[0]))


def consistent_transport(grid, q, qbar_x, qbar_y, els=None):
    """qbar = q + Jz (Qbar - sum_col q) / H (internal3d.py:190-208)."""
    dm = _dm(grid)
    dev, nt, L = dm.device, dm.nt, dm.L
    A = Arr()
    with torch.cuda.device(dev):
        el = els_dev(els, dev)
        eta = _eta(grid, A, dev)
        qd = p6_in(A.dev(q, dev), nt, L)
        qb = torch.stack([c3_in(A.dev(qbar_x, dev), dev), c3_in(A.dev(qbar_y, dev), dev)])
        qsum = torch.empty((2, 3, nt), dtype=F64, device=dev)
        htot = torch.empty((3, nt), dtype=F64, device=dev)
        mis = torch.empty((2, 3, nt), dtype=F64, device=dev)
        lb = _lib.lib()
        s = stream_ptr()
        _lib.check(lb.pdg_column_sum(nt, L, 2, ptr(qd), ptr(qsum), s), "colsum")
        _lib.check(lb.pdg_total_thickness(dm.h, ptr(eta), ptr(htot), s), "htot")
        _lib.check(lb.pdg_mismatch(dm.h, ptr(qb), ptr(qsum), ptr(htot), ptr(mis), s), "mismatch")
        out = _zeros(2, 6, L, nt, dev=dev)
        _lib.check(lb.pdg_consistent_transport(dm.h, ptr(eta), ptr(qd), ptr(mis), ptr(el), _nsel(dm, el), ptr(out), s),
                   "consistent_transport")
        return A.out(p6_out(out, nt, L))


def lateral_flux_factor(grid, qfield, params: PhysParams, els=None):
    """n.{q} + {Jz/H} max(c) [[eta]], (nt, L, 3, 2, 2) (internal3d.py:275-314)."""
    dm = _dm(grid)
    dev, nt, L = dm.device, dm.nt, dm.L
    A = Arr()
    with torch.cuda.device(dev):
        el = els_dev(els, dev)
        qd = p6_in(A.dev(qfield, dev), nt, L)
        fac = _zeros(3, 2, 2, L, nt, dev=dev)
        _lib.check(_lib.lib().pdg_lateral_flux_factor(dm.h, ptr(_eta(grid, A, dev)), ptr(qd), params.g, ptr(el),
                                                      _nsel(dm, el), ptr(fac), stream_ptr()), "factor")
        return A.out(_fac_out(fac))


# ----------------------------------------------------------------------------- r, w, w~

def compute_r(grid, rho, params: PhysParams, els=None):
    """Baroclinic head (P, 6, 2): weak RHS + top-down sweep (internal3d.py:327-405)."""
    dm = _dm(grid)
    dev, nt, L = dm.device, dm.nt, dm.L
    A = Arr()
    with torch.cuda.device(dev):
        el = els_dev(els, dev)
        rd = p6_in(A.dev(rho, dev), nt, L)
        r = _zeros(2, 6, L, nt, dev=dev)
        _lib.check(_lib.lib().pdg_compute_r(dm.h, ptr(_eta(grid, A, dev)), ptr(rd), 0, 0.0, 0.0, params.g, ptr(el),
                                            _nsel(dm, el), ptr(r), stream_ptr()), "compute_r")
        dm.raise_errors()
        return A.out(p6_out(r, nt, L))


def compute_w(grid, q, ux, uy, params: PhysParams, factor, els=None):
    """Vertical velocity from continuity (P, 6) (internal3d.py:434-502)."""
    dm = _dm(grid)
    dev, nt, L = dm.device, dm.nt, dm.L
    A = Arr()
    with torch.cuda.device(dev):
        el = els_dev(els, dev)
        qd = p6_in(A.dev(q, dev), nt, L)
        x, y = p6_in(A.dev(ux, dev), nt, L), p6_in(A.dev(uy, dev), nt, L)
        fac = _fac_in(A.dev(factor, dev), nt, L)
        w = _zeros(6, L, nt, dev=dev)
        _lib.check(_lib.lib().pdg_compute_w(dm.h, ptr(_eta(grid, A, dev)), ptr(qd), ptr(x), ptr(y), ptr(fac),
                                            ptr(el), _nsel(dm, el), ptr(w), stream_ptr()), "compute_w")
        dm.raise_errors()
        return A.out(p6_out(w, nt, L))


def compute_wtilde(grid, qbar, factor, els=None):
    """Grid-relative vertical transport (P, 6) (internal3d.py:505-541)."""
    dm = _dm(grid)
    dev, nt, L = dm.device, dm.nt, dm.L
    A = Arr()
    with torch.cuda.device(dev):
        el = els_dev(els, dev)
        qd = p6_in(A.dev(qbar, dev), nt, L)
        fac = _fac_in(A.dev(factor, dev), nt, L)
        w = _zeros(6, L, nt, dev=dev)
        _lib.check(_lib.lib().pdg_compute_wtilde(dm.h, ptr(_eta(grid, A, dev)), ptr(qd), ptr(fac), None, 0.0,
                                                 ptr(el), _nsel(dm, el), ptr(w), stream_ptr()), "compute_wtilde")
        dm.raise_errors()
        return A.out(p6_out(w, nt, L))


# ----------------------------------------------------------------------------- horizontal RHS

def horizontal_rhs(grid, ux, uy, q_adv, factor, r, mass, params: PhysParams, els=None):
    """Explicit horizontal momentum forcing (P, 6, 2) (internal3d.py:695-751)."""
    dm = _dm(grid)
    dev, nt, L = dm.device, dm.nt, dm.L
    A = Arr()
    with torch.cuda.device(dev):
        el = els_dev(els, dev)
        u = torch.stack([p6_in(A.dev(ux, dev), nt, L), p6_in(A.dev(uy, dev), nt, L)])
        qd = p6_in(A.dev(q_adv, dev), nt, L)
        fac = _fac_in(A.dev(factor, dev), nt, L)
        rd = p6_in(A.dev(r, dev), nt, L)
        md = _mass_in(A.dev(mass, dev), nt, L)
        out = _zeros(2, 6, L, nt, dev=dev)
        lb, s = _lib.lib(), stream_ptr()
        _lib.check(lb.pdg_horizontal_rhs(dm.h, ptr(_eta(grid, A, dev)), ptr(u), 2, ptr(qd), ptr(fac), ptr(rd), ptr(md),
                                         params.f, params.rho0, int(el is None), ptr(el), _nsel(dm, el), ptr(out), s),
                   "horizontal_rhs")
        _add_diffusion(dm, _eta(grid, A, dev), u, 2, params.kappa_h, el, out)
        if el is not None:   # the reference adds Coriolis and -M r / rho0 to ALL rows (internal3d.py:745-750)
            _lib.check(lb.pdg_mass_terms(L, nt, ptr(md), ptr(u), ptr(rd), params.f, params.rho0, ptr(out), s),
                       "mass_terms")
        return A.out(p6_out(out, nt, L))


def tracer_horizontal_rhs(grid, tr, qbar, factor, params: PhysParams, els=None):
    """Explicit horizontal tracer forcing (P, 6) (internal3d.py:754-792)."""
    dm = _dm(grid)
    dev, nt, L = dm.device, dm.nt, dm.L
    A = Arr()
    with torch.cuda.device(dev):
        el = els_dev(els, dev)
        t = p6_in(A.dev(tr, dev), nt, L)
        qd = p6_in(A.dev(qbar, dev), nt, L)
        fac = _fac_in(A.dev(factor, dev), nt, L)
        out = _zeros(6, L, nt, dev=dev)
        _lib.check(_lib.lib().pdg_horizontal_rhs(dm.h, ptr(_eta(grid, A, dev)), ptr(t), 1, ptr(qd), ptr(fac), None,
                                                 None, 0.0, 1.0, 0, ptr(el), _nsel(dm, el), ptr(out), stream_ptr()),
                   "tracer_horizontal_rhs")
        _add_diffusion(dm, _eta(grid, A, dev), t, 1, params.nu_h, el, out)
        dm.raise_errors()
        return A.out(p6_out(out, nt, L))


def stress_rhs(grid, tau_sx: float, tau_sy: float, cd: float, ux, uy, els=None):
    """Surface wind stress and quadratic bottom drag (P, 6, 2) (internal3d.py:919-934)."""
    dm = _dm(grid)
    dev, nt, L = dm.device, dm.nt, dm.L
    A = Arr()
    with torch.cuda.device(dev):
        el = els_dev(els, dev)
        x, y = p6_in(A.dev(ux, dev), nt, L), p6_in(A.dev(uy, dev), nt, L)
        out = _zeros(2, 6, L, nt, dev=dev)
        _lib.check(_lib.lib().pdg_stress_rhs(dm.h, ptr(x), ptr(y), float(tau_sx), float(tau_sy), float(cd), ptr(el),
                                             _nsel(dm, el), ptr(out), stream_ptr()), "stress_rhs")
        return A.out(p6_out(out, nt, L))


# ----------------------------------------------------------------------------- vertical operator

def _band_out(t, n, L, rows):
    return t.permute(2, 1, 0).reshape(n, L, rows, 6).contiguous()


def assemble_vertical_operator(grid, wtilde, w_m, kh: float, kv: float, els=None,
                               pen: PenaltyParams = PenaltyParams()) -> BandedColumnMatrix:
    """Banded vertical advection-diffusion operator (internal3d.py:800-899)."""
    dm = _dm(grid)
    dev, nt, L = dm.device, dm.nt, dm.L
    A = Arr()
    with torch.cuda.device(dev):
        el = els_dev(els, dev)
        n = _nsel(dm, el)
        wt = p6_in(A.dev(wtilde, dev), nt, L)
        wm = p6_in(A.dev(w_m, dev), nt, L)
        d = torch.empty((36, L, n), dtype=F64, device=dev)
        u = torch.empty((18, L, n), dtype=F64, device=dev)
        w = torch.empty((18, L, n), dtype=F64, device=dev)
        _lib.check(_lib.lib().pdg_assemble_vertical(dm.h, ptr(_eta(grid, A, dev)), ptr(wt), ptr(wm), float(kh),
                                                    float(kv), float(pen.n0), int(pen.order), ptr(el), n, ptr(d),
                                                    ptr(u), ptr(w), stream_ptr()), "assemble_vertical_operator")
        dm.raise_errors()
        return BandedColumnMatrix(d=A.out(_band_out(d, n, L, 6)), u=A.out(_band_out(u, n, L, 3)),
                                  w=A.out(_band_out(w, n, L, 3)))


def build_implicit(mass, op: BandedColumnMatrix, dt: float, grid, els=None) -> BandedColumnMatrix:
    """(M - dt A) over the same column subset (internal3d.py:902-906)."""
    nt, L = grid.mesh.nt, grid.n_layers
    dev = torch.device("cuda", torch.cuda.current_device())
    A = Arr()
    mv = A.dev(mass, dev).reshape(nt, L, 36)
    if els is not None:
        mv = mv[els_dev(els, dev).long()]
    n = mv.shape[0]
    P = n * L
    d, u, w = A.dev(op.d, dev), A.dev(op.u, dev), A.dev(op.w, dev)
    dd = d.reshape(P, 36).t().contiguous()
    uu = u.reshape(P, 18).t().contiguous()
    ww = w.reshape(P, 18).t().contiguous()
    md = mv.reshape(P, 36).t().contiguous()
    od, ou, ow = torch.empty_like(dd), torch.empty_like(uu), torch.empty_like(ww)
    _lib.check(_lib.lib().pdg_build_implicit(P, ptr(md), ptr(dd), ptr(uu), ptr(ww), float(dt), ptr(od), ptr(ou),
                                             ptr(ow), stream_ptr()), "build_implicit")
    return BandedColumnMatrix(d=A.out(od.t().reshape(n, L, 6, 6)), u=A.out(ou.t().reshape(n, L, 3, 6)),
                              w=A.out(ow.t().reshape(n, L, 3, 6)))


def scatter_columns(x, grid, els=None, ncomp=None):
    """(n, L, 6[, nc]) column data back to (P, 6[, nc]) storage (internal3d.py:909-916)."""
    nt, L = grid.mesh.nt, grid.n_layers
    is_np = not isinstance(x, torch.Tensor)
    xt = torch.as_tensor(np.asarray(x)) if is_np else x
    shape = (nt, L) + tuple(xt.shape[2:])
    out = torch.zeros(shape, dtype=xt.dtype, device=xt.device)
    cols = torch.arange(nt) if els is None else torch.as_tensor(np.asarray(els), dtype=torch.long)
    out[cols.to(xt.device)] = xt
    out = out.reshape((nt * L,) + tuple(xt.shape[2:]))
    return out.numpy() if is_np else out


def budget_3d(grid, mass, ux, uy, tr) -> dict:
    """Integral budgets (internal3d.py:942-951) -- reporting."""
    P = grid.n_prisms
    ones = np.ones((P, 6))
    to = (lambda a: a.cpu().numpy()) if isinstance(tr, torch.Tensor) else np.asarray
    return {"volume": integrate_prism(mass, ones), "momentum_x": integrate_prism(mass, ux),
            "momentum_y": integrate_prism(mass, uy), "tracer_mass": integrate_prism(mass, tr),
            "tracer_min": float(to(tr).min()), "tracer_max": float(to(tr).max())}

"""Drop-in for prismdg/external2d.py: 2D external mode on the B200.

Same function names, signatures, shapes and exceptions as the reference.
Arrays may be numpy (copied in/out -- parity path) or torch CUDA tensors
(zero-copy -- performance path); results come back in the caller's kind.
All arithmetic runs in libprismdg_b200.so (csrc/ext2d.cu); nothing is computed
on the host.
"""
from __future__ import annotations

import ctypes
import math
from typing import Callable, Optional

import numpy as np
import torch

from . import _lib
from .device import Arr, c3_in, c3_out, device_mesh, els_dev, ptr, require_cuda, stream_ptr
from .params import ExternalResult, PhysParams, State2D

__all__ = ["PhysParams", "State2D", "ExternalResult", "eos_density", "trace_int", "trace_ext", "edge_celerity",
           "rhs_free_surface", "rhs_depth_momentum", "external_tendencies", "check_cfl", "subcycle_external",
           "integrate_nodal", "diagnostics_2d"]

# edge-point shapes in the edge's own traversal order (dg.py:76-81): ES[h][s]
_GZ = 1.0 / math.sqrt(3.0)
_ES = ((0.5 * (1.0 + _GZ), 0.5 * (1.0 - _GZ)), (0.5 * (1.0 - _GZ), 0.5 * (1.0 + _GZ)))
_EV0, _EV1 = (0, 1, 2), (1, 2, 0)


def _cuda():
    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def _idx(a, device):
    return torch.as_tensor(np.asarray(a.cpu() if isinstance(a, torch.Tensor) else a, dtype=np.int64), device=device)


def trace_int(field2d, els, k):
    """Interior trace of a (nt, 3) nodal field on local edge k at the 2 Gauss points: (nel, 2)
    (external2d.py:95-99)."""
    A = Arr()
    f = A.dev(field2d, _cuda())
    r = _idx(els, f.device)
    n0, n1 = f[r, _EV0[k]], f[r, _EV1[k]]
    return A.out(torch.stack([n0 * _ES[q][0] + n1 * _ES[q][1] for q in range(2)], dim=-1))


def trace_ext(field2d, nbr_e, nbr_k):
    """Exterior trace at the same physical points, mirrored point order (external2d.py:102-107)."""
    A = Arr()
    f = A.dev(field2d, _cuda())
    e = _idx(nbr_e, f.device).clamp_min(0)
    kk = _idx(nbr_k, f.device)
    ev0 = torch.as_tensor(_EV0, device=f.device)[kk]
    ev1 = torch.as_tensor(_EV1, device=f.device)[kk]
    m0, m1 = f[e, ev0], f[e, ev1]
    t = torch.stack([m0 * _ES[q][1] + m1 * _ES[q][0] for q in range(2)], dim=-1)
    return A.out(t)


def edge_celerity(eta_i, eta_e, b_i, b_e, g):
    """max over both sides of sqrt(g H) per point; DryColumn(-1, min H) if either side is dry
    (external2d.py:110-116)."""
    A = Arr()
    dev = _cuda()
    hi = A.dev(eta_i, dev) - A.dev(b_i, dev)
    he = A.dev(eta_e, dev) - A.dev(b_e, dev)
    lo = float(torch.minimum(hi.min(), he.min()).item()) if hi.numel() else 1.0
    if lo <= 0.0:
        from .errors import DryColumn
        raise DryColumn(-1, lo)
    return A.out(torch.maximum(torch.sqrt(g * hi), torch.sqrt(g * he)))


def eos_density(T, params: PhysParams, S=None):
    """rho' = -alpha (T - t_ref) + beta (S - s_ref)  (external2d.py:81-87), on device."""
    require_cuda()
    A = Arr()
    dev = torch.device("cuda", torch.cuda.current_device())
    t = A.dev(T, dev).contiguous()
    s = None
    if params.beta != 0.0 and S is not None:
        s = torch.broadcast_to(A.dev(S, dev), t.shape).contiguous()
    out = torch.empty_like(t)
    if t.numel():
        _lib.check(_lib.lib().pdg_eos(ptr(t), ptr(s), t.numel(), params.alpha, params.beta, params.t_ref,
                                      params.s_ref, ptr(out), stream_ptr()), "eos")
    return A.out(out)


def _state_dev(state, A, dev):
    return (c3_in(A.dev(state.eta, dev), dev), c3_in(A.dev(state.qx, dev), dev), c3_in(A.dev(state.qy, dev), dev))


def _eval(state, mesh, params, els, f3d2d, source, patm, eta_bc, mode):
    dm = device_mesh(mesh)
    dev = dm.device
    A = Arr()
    with torch.cuda.device(dev):
        e, x, y = _state_dev(state, A, dev)
        f3 = None if f3d2d is None else c3_in(A.dev(f3d2d, dev), dev)
        src = None if source is None else c3_in(A.dev(source, dev), dev)
        pa = None if patm is None else c3_in(A.dev(patm, dev), dev)
        el = els_dev(els, dev)
        n = dm.nt if el is None else el.numel()
        out = torch.empty((3, 3, n), dtype=torch.float64, device=dev)
        has_bc = eta_bc is not None
        bc = float(eta_bc(state.t)) if has_bc else 0.0
        if n:
            _lib.check(_lib.lib().pdg_ext2d_eval(dm.h, ptr(e), ptr(x), ptr(y), ptr(f3), ptr(src), ptr(pa), int(has_bc),
                                                 bc, params.g, params.rho0, ptr(el), n, mode, ptr(out[0]),
                                                 ptr(out[1]), ptr(out[2]), stream_ptr()), "ext2d_eval")
        dm.raise_errors("external2d")
    return A, out


def rhs_free_surface(state: State2D, mesh, params: PhysParams, els=None, source=None,
                     eta_bc: Optional[Callable[[float], float]] = None):
    """Weak free-surface residual before Mh^-1, (nel, 3) (external2d.py:128-184)."""
    A, out = _eval(state, mesh, params, els, None, source, None, eta_bc, 1)
    return A.out(c3_out(out[0]))


def rhs_depth_momentum(state: State2D, mesh, params: PhysParams, els=None, f3d2d=None, patm=None,
                       eta_bc: Optional[Callable[[float], float]] = None):
    """Weak depth-momentum residual, (nel, 3, 2) (external2d.py:187-256)."""
    A, out = _eval(state, mesh, params, els, f3d2d, None, patm, eta_bc, 1)
    return A.out(torch.stack([c3_out(out[1]), c3_out(out[2])], dim=-1))


def external_tendencies(state, mesh, params, els=None, f3d2d=None, source=None, patm=None, eta_bc=None):
    """(d eta/dt, d Qx/dt, d Qy/dt) on the selected elements (external2d.py:259-268)."""
    A, out = _eval(state, mesh, params, els, f3d2d, source, patm, eta_bc, 0)
    return A.out(c3_out(out[0])), A.out(c3_out(out[1])), A.out(c3_out(out[2]))


def check_cfl(state: State2D, mesh, params: PhysParams, dt2d: float) -> float:
    """Raise DryColumn / CflViolation, return c dt / dx (external2d.py:271-283)."""
    dm = device_mesh(mesh)
    dev = dm.device
    A = Arr()
    with torch.cuda.device(dev):
        e = c3_in(A.dev(state.eta, dev), dev)
        r = torch.zeros(1, dtype=torch.float64, device=dev)
        _lib.check(_lib.lib().pdg_ext2d_cfl(dm.h, ptr(e), params.g, float(dt2d), ptr(r), stream_ptr()), "cfl")
        try:
            dm.raise_errors()
        except Exception as exc:
            from .errors import CflViolation
            if isinstance(exc, CflViolation):
                ratio = float(r.item())
                raise CflViolation(f"dt2d = {dt2d:g} gives c dt / dx = {ratio:.3f} > 1/3 "
                                   f"(min edge = {mesh.min_edge:g})") from None
            raise
        return float(r.item())


def subcycle_external(state: State2D, mesh, params: PhysParams, m: int, dt2d: float, f3d2d=None, source=None,
                      patm=None, eta_bc=None) -> ExternalResult:
    """m SSP-RK3 substeps with Qbar / F2D accumulation (external2d.py:296-353), one launch per RK stage."""
    dm = device_mesh(mesh)
    dev = dm.device
    A = Arr()
    nt = dm.nt
    with torch.cuda.device(dev):
        S = torch.empty((3, 3, nt), dtype=torch.float64, device=dev)
        e, x, y = _state_dev(state, A, dev)
        S[0].copy_(e)
        S[1].copy_(x)
        S[2].copy_(y)
        f3 = None if f3d2d is None else c3_in(A.dev(f3d2d, dev), dev)
        src = None if source is None else c3_in(A.dev(source, dev), dev)
        pa = None if patm is None else c3_in(A.dev(patm, dev), dev)
        qbar = torch.empty((2, 3, nt), dtype=torch.float64, device=dev)
        f2d = torch.empty((2, 3, nt), dtype=torch.float64, device=dev)
        bc = None
        if eta_bc is not None:
            t0 = state.t
            vals = []
            t = t0
            for _ in range(m):   # stage times t, t + dt, t + dt/2 (external2d.py:325-331)
                vals += [eta_bc(t), eta_bc(t + dt2d), eta_bc(t + 0.5 * dt2d)]
                t = t + dt2d
            bc = np.asarray(vals, dtype=np.float64)
        _lib.check(_lib.lib().pdg_ext2d_subcycle(dm.h, ptr(S), int(m), float(dt2d), params.g, params.rho0, ptr(f3),
                                                 ptr(src), ptr(pa), None if bc is None else bc.ctypes.data,
                                                 ptr(qbar), ptr(f2d), 1, stream_ptr()), "subcycle")
        try:
            dm.raise_errors()
        except Exception as exc:
            from .errors import CflViolation
            if isinstance(exc, CflViolation):
                raise CflViolation(f"dt2d = {dt2d:g} gives c dt / dx > 1/3 (min edge = {mesh.min_edge:g})") from None
            raise
    t_end = state.t
    for _ in range(m):
        t_end = t_end + dt2d
    st = State2D(A.out(c3_out(S[0])), A.out(c3_out(S[1])), A.out(c3_out(S[2])), t_end)
    return ExternalResult(state=st, qbar_x=A.out(c3_out(qbar[0])), qbar_y=A.out(c3_out(qbar[1])),
                          f2d_x=A.out(c3_out(f2d[0])), f2d_y=A.out(c3_out(f2d[1])), steps=m)


# ------------------------------------------------------------------ diagnostics (reporting, not hot path)

def integrate_nodal(field2d, mesh) -> float:
    """Exact integral of a P1 field (external2d.py:361-363): sum (J2D/24)(v + sum v) = sum J2D/6 sum v."""
    f = torch.as_tensor(np.asarray(field2d) if not isinstance(field2d, torch.Tensor) else field2d,
                        dtype=torch.float64, device="cuda")
    j = torch.as_tensor(mesh.j2d, dtype=torch.float64, device=f.device)
    s = f.sum(dim=-1, keepdim=True)
    return float(((f + s) * (j[:, None] / 24.0)).sum().item())


def diagnostics_2d(state: State2D, mesh, params: PhysParams) -> dict:
    """Volume, energy and eta range (external2d.py:366-380)."""
    from .tables import BARY_T, QW_T
    dev = torch.device("cuda")
    e = torch.as_tensor(np.asarray(state.eta) if not isinstance(state.eta, torch.Tensor) else state.eta,
                        dtype=torch.float64, device=dev)
    x = torch.as_tensor(np.asarray(state.qx) if not isinstance(state.qx, torch.Tensor) else state.qx,
                        dtype=torch.float64, device=dev)
    y = torch.as_tensor(np.asarray(state.qy) if not isinstance(state.qy, torch.Tensor) else state.qy,
                        dtype=torch.float64, device=dev)
    b = torch.as_tensor(mesh.b, dtype=torch.float64, device=dev)
    j = torch.as_tensor(mesh.j2d, dtype=torch.float64, device=dev)
    B = BARY_T.to(dev)
    hq = (e - b) @ B.T
    dens = 0.5 * params.g * (e @ B.T) ** 2 + 0.5 * ((x @ B.T) ** 2 + (y @ B.T) ** 2) / hq
    energy = float((j[:, None] * dens * QW_T.to(dev)[None, :]).sum().item())
    return {"t": state.t, "total_volume": integrate_nodal(e - b, mesh), "total_energy": energy,
            "eta_min": float(e.min().item()), "eta_max": float(e.max().item())}

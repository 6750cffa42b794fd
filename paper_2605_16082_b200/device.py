"""Device context (one pdg_ctx per mesh per CUDA device) and layout plumbing.

torch owns every field buffer; the library only receives raw device pointers.
Reference layouts ((nt,3), (P,6[,nc]), (ncol,L,6[,nc])) are converted to the
device layouts of include/prismdg_b200.h with torch permutes -- that is
plumbing for the drop-in per-function API; the stepper keeps all state in the
device layouts and never converts on the hot path.
"""
from __future__ import annotations

import ctypes
import hashlib

import numpy as np
import torch

from . import _lib
from .errors import raise_for_code

F64 = torch.float64


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2605_16082_b200 needs a CUDA device (B200); there is no CPU fallback")


def ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def stream_ptr():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class DeviceMesh:
    """Uploads Mesh2D geometry/connectivity once; owns the C context."""

    def __init__(self, mesh, device=None):
        require_cuda()
        _drain_pending()
        self.mesh = mesh
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.nt = mesh.nt
        L = _lib.lib()
        arrs = {k: np.ascontiguousarray(getattr(mesh, k), dtype=np.float64)
                for k in ("j2d", "dphx", "dphy", "elen", "enx", "eny", "b")}
        ints = {k: np.ascontiguousarray(getattr(mesh, k), dtype=np.int64) for k in ("nbr", "nbrk", "btag")}
        desc = _lib.MeshDesc(self.nt, *[arrs[k].ctypes.data for k in ("j2d", "dphx", "dphy", "elen", "enx", "eny",
                                                                         "b")],
                             *[ints[k].ctypes.data for k in ("nbr", "nbrk", "btag")], float(mesh.min_edge))
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(L.pdg_ctx_create(ctypes.byref(desc), self.device.index, ctypes.byref(h)), "pdg_ctx_create")
        self.h = h
        self.L = 0
        self._fracs = None
        self.fingerprint = mesh_fingerprint(mesh)
        # device copies used by host-side glue (Python never reads them per step)
        self.j2d = torch.as_tensor(arrs["j2d"], device=self.device)
        self.b3 = torch.as_tensor(arrs["b"].T.copy(), device=self.device)

    def set_layers(self, L: int, fracs=None):
        """Layer count and sigma fractions (default: uniform, as extrude builds them, mesh.py:389)."""
        fr = np.linspace(0.0, 1.0, L + 1) if fracs is None else np.ascontiguousarray(fracs, dtype=np.float64)
        if fr.shape != (L + 1,):
            from .errors import ShapeMismatch
            raise ShapeMismatch(f"fracs has shape {fr.shape}, expected ({L + 1},)")
        if L != self.L or not np.array_equal(fr, self._fracs):
            _lib.check(_lib.lib().pdg_ctx_set_layers(self.h, int(L), fr.ctypes.data), "pdg_ctx_set_layers")
            self.L, self._fracs = L, fr.copy()
        return self

    def raise_errors(self, what=""):
        code, i0, i1, val = ctypes.c_int(), ctypes.c_longlong(), ctypes.c_longlong(), ctypes.c_double()
        _lib.check(_lib.lib().pdg_last_error(self.h, stream_ptr(), ctypes.byref(code), ctypes.byref(i0),
                                             ctypes.byref(i1), ctypes.byref(val)), "pdg_last_error")
        raise_for_code(code.value, i0.value, i1.value, val.value, what)

    def launches(self) -> int:
        return int(_lib.lib().pdg_launch_count(self.h))

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and _lib._lib is not None:
            # cudaFree is illegal while any stream is being captured into a CUDA graph (global capture
            # mode); garbage collection can run this finaliser in the middle of a capture -> defer.
            _PENDING.append(h)
            _drain_pending()


_PENDING = []


def _drain_pending():
    try:
        if torch.cuda.is_available() and torch.cuda.is_current_stream_capturing():
            return
    except Exception:
        return
    while _PENDING:
        h = _PENDING.pop()
        try:
            _lib.lib().pdg_ctx_destroy(h)
        except Exception:
            pass


def mesh_fingerprint(mesh) -> bytes:
    hsh = hashlib.blake2b(digest_size=16)
    for k in ("tri", "nbr", "nbrk", "btag", "vx", "vy", "vb", "b"):
        a = getattr(mesh, k, None)
        if a is not None:
            hsh.update(np.ascontiguousarray(a).tobytes())
    return hsh.digest()


def device_mesh(mesh, L: int | None = None, fracs=None) -> DeviceMesh:
    """Cached DeviceMesh of a Mesh2D for the per-function API (rebuilt if the mesh arrays were
    edited in place).  Steppers never share it: each owns a DeviceMesh of its own."""
    dm = getattr(mesh, "_pdg_dev", None)
    if dm is None or dm.fingerprint != mesh_fingerprint(mesh):
        dm = DeviceMesh(mesh)
        try:
            object.__setattr__(mesh, "_pdg_dev", dm)
        except Exception:
            pass
    if L is not None:
        dm.set_layers(L, fracs)
    return dm


# ------------------------------------------------------------------ layout conversion

class Arr:
    """Remembers whether the caller passed numpy (host) or torch so results come back alike."""

    def __init__(self):
        self.numpy = False

    def dev(self, a, device):
        if a is None:
            return None
        if isinstance(a, torch.Tensor):
            return a.to(device=device, dtype=F64)
        self.numpy = True
        return torch.as_tensor(np.asarray(a, dtype=np.float64), device=device)

    def out(self, t):
        return t.cpu().numpy() if self.numpy else t


def c3_in(a, device):
    """(n,3[,nc]) -> [nc][3][n] contiguous."""
    if a.dim() == 2:
        return a.t().contiguous()
    return a.permute(2, 1, 0).contiguous()


def c3_out(t, nc=None):
    """[nc][3][n] or [3][n] -> (n,3[,nc])."""
    if t.dim() == 2:
        return t.t().contiguous()
    return t.permute(2, 1, 0).contiguous()


def p6_in(a, nt, L):
    """(P,6) or (P,6,nc) -> [6][L][nt] / [nc][6][L][nt]."""
    if a.dim() == 2:
        return a.reshape(nt, L, 6).permute(2, 1, 0).contiguous()
    nc = a.shape[2]
    return a.reshape(nt, L, 6, nc).permute(3, 2, 1, 0).contiguous()


def p6_out(t, nt, L):
    """[6][L][nt] / [nc][6][L][nt] -> (P,6) / (P,6,nc)."""
    if t.dim() == 3:
        return t.permute(2, 1, 0).reshape(nt * L, 6).contiguous()
    return t.permute(3, 2, 1, 0).reshape(nt * L, 6, t.shape[0]).contiguous()


def els_dev(els, device):
    if els is None:
        return None
    e = np.asarray(els.cpu() if isinstance(els, torch.Tensor) else els, dtype=np.int32).reshape(-1)
    return torch.as_tensor(e, device=device)

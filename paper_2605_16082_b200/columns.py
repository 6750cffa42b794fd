"""Drop-in for prismdg/columns.py: column-local vertical solvers on the B200.

solve_r_column / solve_w_column / solve_banded_column / apply_banded /
solve_tridiagonal / apply_mh[_inv] run in csrc/columns.cu (one thread per
column).  Column systems use the reference shapes: rhs (ncol, L, 6[, nc]),
BandedColumnMatrix d (ncol, L, 6, 6), u / w (ncol, L, 3, 6).
assemble_dense_oracle / banded_to_dense are the reference's literal dense
test oracles (host numpy, not a compute path).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .device import Arr, ptr, require_cuda, stream_ptr
from .errors import ShapeMismatch, raise_for_code
from .params import BandedColumnMatrix

F64 = torch.float64
MH_PATTERN = np.array([[2.0, 1.0, 1.0], [1.0, 2.0, 1.0], [1.0, 1.0, 2.0]]) / 24.0
MH_INV_PATTERN = np.array([[3.0, -1.0, -1.0], [-1.0, 3.0, -1.0], [-1.0, -1.0, 3.0]]) * 6.0

_ERR = {}


def _err_word(dev):
    """Per-device error word (pdg_err, 32 bytes) for context-free entries."""
    t = _ERR.get(dev.index)
    if t is None:
        t = torch.zeros(4, dtype=torch.int64, device=dev)
        _ERR[dev.index] = t
    return t


def _err_check(err):
    h = err.cpu()
    code = int(h[0].item() & 0xFFFFFFFF)
    if code:
        val = float(h[3:4].view(torch.float64).item())
        err.zero_()
        raise_for_code(code, int(h[1].item()), int(h[2].item()), val)


def _dev():
    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def mh_matrix(j2d):
    """(..., 3, 3) triangle mass matrix (columns.py:39-42) -- small host helper."""
    return np.asarray(j2d, dtype=float)[..., None, None] * MH_PATTERN


def _mh(values, j2d, inverse):
    dev = _dev()
    A = Arr()
    v = A.dev(values, dev)
    j = A.dev(j2d, dev)
    vec = v.shape[-1] == 3
    lead = v.shape[:-1] if vec else v.shape[:-2]
    n = int(np.prod(lead)) if len(lead) else 1
    nc = 1 if vec else v.shape[-1]
    vd = v.reshape(n, 3, nc).permute(2, 1, 0).contiguous()
    jd = torch.broadcast_to(j, lead).reshape(n).contiguous()
    out = torch.empty_like(vd)
    err = _err_word(dev)
    _lib.check(_lib.lib().pdg_apply_mh(ptr(vd), ptr(jd), n, nc, int(inverse), ptr(out), ptr(err), stream_ptr()), "mh")
    if inverse:
        _err_check(err)
    res = out.permute(2, 1, 0).reshape(v.shape)
    return A.out(res.contiguous())


def apply_mh(values, j2d):
    """Mh @ values (columns.py:45-56)."""
    return _mh(values, j2d, False)


def apply_mh_inv(values, j2d):
    """Mh^-1 @ values, SingularMass if J2D <= 0 (columns.py:59-69)."""
    return _mh(values, j2d, True)


def _col_in(rhs, A, dev):
    r = A.dev(rhs, dev)
    had = r.dim() == 4
    if r.dim() == 3:
        r = r[..., None]
    if r.dim() != 4 or r.shape[2] != 6:
        raise ShapeMismatch(f"column RHS must be (ncol, L, 6[, nc]), got {tuple(r.shape)}")
    return r.permute(3, 2, 1, 0).contiguous(), had     # [nc][6][L][ncol]


def _col_out(t, had):
    r = t.permute(3, 2, 1, 0).contiguous()
    return r if had else r[..., 0].contiguous()


def _sweep(kind, rhs, j2d, layers):
    dev = _dev()
    A = Arr()
    r, had = _col_in(rhs, A, dev)
    nc, _, L, ncol = r.shape
    j = A.dev(j2d, dev).reshape(ncol).contiguous()
    lay = None
    if layers is not None:
        lay = torch.as_tensor(np.asarray(layers.cpu() if isinstance(layers, torch.Tensor) else layers),
                              dtype=torch.int32, device=dev)
    out = torch.empty_like(r)
    err = _err_word(dev)
    _lib.check(_lib.lib().pdg_solve_sweep(kind, ncol, L, nc, ptr(r), ptr(j), ptr(lay), ptr(out), ptr(err),
                                          stream_ptr()), "sweep")
    _err_check(err)
    return A.out(_col_out(out, had))


def solve_r_column(rhs, j2d, layers=None):
    """Top-down sweep of the surface-anchored operator D_vu (columns.py:95-122)."""
    return _sweep(0, rhs, j2d, layers)


def solve_w_column(rhs, j2d, layers=None):
    """Bottom-up sweep of the bed-anchored operator D_vd (columns.py:125-151)."""
    return _sweep(1, rhs, j2d, layers)


def _solve_cell(kind, block, j2d_cols, j2d_pad):
    """The column sweep on a cell block (columns.py:546-580): padded lanes get j2d_pad and zero
    layers and come back zero; the solve runs on the GPU (pdg_solve_sweep)."""
    from .layout import CellBlock, cell_view
    view = cell_view(block)                          # (width, L, 6, ncomp)
    w, n = block.width, block.columns.size
    j = np.full(w, j2d_pad, dtype=block.data.dtype)
    j[:n] = np.asarray(j2d_cols, dtype=block.data.dtype)
    lay = np.zeros(w, dtype=np.int64)
    lay[:n] = block.layers
    x = _sweep(kind, np.ascontiguousarray(view), j, lay)
    out = CellBlock(data=np.zeros_like(block.data), columns=block.columns.copy(), layers=block.layers.copy(),
                    ncomp=block.ncomp)
    cell_view(out)[:] = x
    return out


def solve_r_cell(block, j2d_cols, j2d_pad: float = 1.0):
    """solve_r_column on a cell block (columns.py:546-562)."""
    return _solve_cell(0, block, j2d_cols, j2d_pad)


def solve_w_cell(block, j2d_cols, j2d_pad: float = 1.0):
    """solve_w_column on a cell block (columns.py:565-580)."""
    return _solve_cell(1, block, j2d_cols, j2d_pad)


def assemble_dense_oracle(kind: str, layers: int, mh: np.ndarray) -> np.ndarray:
    """Literal dense D_vu / D_vd (columns.py:154-188): a test oracle, host numpy."""
    L = int(layers)
    a = np.zeros((6 * L, 6 * L))

    def blk(r, c, m):
        a[3 * r:3 * r + 3, 3 * c:3 * c + 3] += m
    for l in range(L):
        t, b = 2 * l, 2 * l + 1
        if kind == "r":
            blk(t, t, -0.5 * mh); blk(t, b, -0.5 * mh); blk(b, t, 0.5 * mh); blk(b, b, -0.5 * mh)
            if l > 0:
                blk(t, 2 * l - 1, mh)
        elif kind == "w":
            blk(t, t, 0.5 * mh); blk(t, b, -0.5 * mh); blk(b, t, 0.5 * mh); blk(b, b, 0.5 * mh)
            if l < L - 1:
                blk(b, 2 * (l + 1), -mh)
        else:
            raise ValueError(f"unknown oracle kind '{kind}'")
    return a


def make_identity_banded(ncol: int, nlay: int, dtype=np.float64) -> BandedColumnMatrix:
    d = np.zeros((ncol, nlay, 6, 6), dtype=dtype)
    d[:, :] = np.eye(6, dtype=dtype)
    return BandedColumnMatrix(d=d, u=np.zeros((ncol, nlay, 3, 6), dtype=dtype),
                              w=np.zeros((ncol, nlay, 3, 6), dtype=dtype))


def pad_banded(mat: BandedColumnMatrix) -> BandedColumnMatrix:
    """Identity systems on inactive layers (columns.py:240-249)."""
    if mat.layers is None:
        return mat
    L = mat.nlay
    lay = np.asarray(mat.layers.cpu() if isinstance(mat.layers, torch.Tensor) else mat.layers)
    inactive = np.arange(L)[None, :] >= lay[:, None]
    for name, eye in (("d", True), ("u", False), ("w", False)):
        a = getattr(mat, name)
        if isinstance(a, torch.Tensor):
            idx = torch.as_tensor(inactive, device=a.device)
            a[idx] = torch.eye(6, dtype=a.dtype, device=a.device) if eye else 0.0
        else:
            a[inactive] = np.eye(6, dtype=a.dtype) if eye else 0.0
    return mat


def banded_to_dense(mat: BandedColumnMatrix, col: int) -> np.ndarray:
    """Dense (6L, 6L) matrix of one column (columns.py:252-263): test helper."""
    d, u, w = (np.asarray(x.cpu() if isinstance(x, torch.Tensor) else x) for x in (mat.d, mat.u, mat.w))
    L = d.shape[1]
    a = np.zeros((6 * L, 6 * L), dtype=d.dtype)
    for l in range(L):
        r = 6 * l
        a[r:r + 6, r:r + 6] = d[col, l]
        if l > 0:
            a[r:r + 3, r - 6:r] = u[col, l]
        if l < L - 1:
            a[r + 3:r + 6, r + 6:r + 12] = w[col, l]
    return a


def _band_in(a, rows, A, dev):
    t = A.dev(a, dev)
    n, L = t.shape[0], t.shape[1]
    return t.reshape(n, L, rows * 6).permute(2, 1, 0).contiguous()


def solve_banded_column(mat: BandedColumnMatrix, rhs, overwrite: bool = False):
    """Block-Thomas elimination without pivoting, ZeroPivot(layer, node) (columns.py:292-348).

    overwrite=True replaces mat.u / mat.w by the propagation tiles G_l, like the reference.
    """
    dev = _dev()
    A = Arr()
    r, had = _col_in(rhs, A, dev)
    nc, _, L, ncol = r.shape
    if mat.d.shape[0] != ncol or mat.d.shape[1] != L:
        raise ShapeMismatch(f"rhs shape {tuple(rhs.shape)} does not match matrix ({mat.d.shape[0]}, {mat.d.shape[1]})")
    d = _band_in(mat.d, 6, A, dev)
    u = _band_in(mat.u, 3, A, dev)
    w = _band_in(mat.w, 3, A, dev)
    gu, gw = torch.empty_like(u), torch.empty_like(w)
    x = torch.empty_like(r)
    err = _err_word(dev)
    _lib.check(_lib.lib().pdg_solve_banded(ncol, L, nc, ptr(d), ptr(u), ptr(w), ptr(gu), ptr(gw), ptr(r), ptr(x),
                                           ptr(err), stream_ptr()), "solve_banded")
    _err_check(err)
    if overwrite:
        # stored tiles replace u / w for layers < L-1, layer L-1 keeps its blocks (columns.py:329-335)
        for name, g, orig in (("u", gu, u), ("w", gw, w)):
            g[:, L - 1] = orig[:, L - 1]
            out = g.permute(2, 1, 0).reshape(ncol, L, 3, 6)
            tgt = getattr(mat, name)
            if isinstance(tgt, torch.Tensor):
                tgt.copy_(out)
            else:
                tgt[...] = out.cpu().numpy()
    return A.out(_col_out(x, had))


def apply_banded(mat: BandedColumnMatrix, x):
    """y = A x for the banded column matrix (columns.py:356-366)."""
    dev = _dev()
    A = Arr()
    r, had = _col_in(x, A, dev)
    nc, _, L, ncol = r.shape
    if mat.d.shape[0] != ncol or mat.d.shape[1] != L:
        raise ShapeMismatch(f"operand shape {tuple(x.shape)} does not match matrix ({mat.d.shape[0]}, {mat.d.shape[1]})")
    d, u, w = _band_in(mat.d, 6, A, dev), _band_in(mat.u, 3, A, dev), _band_in(mat.w, 3, A, dev)
    y = torch.empty_like(r)
    _lib.check(_lib.lib().pdg_apply_banded(ncol, L, nc, ptr(d), ptr(u), ptr(w), ptr(r), ptr(y), stream_ptr()),
               "apply_banded")
    return A.out(_col_out(y, had))


@dataclass
class AccessStats:
    """Working-set record of a column elimination (columns.py:375-379)."""
    max_live: int = 0
    loads: int = 0
    stores: int = 0
    touched: set = field(default_factory=set)


def solve_banded_sequential(mat: BandedColumnMatrix, rhs, col: int, stats: AccessStats = None):
    """One column of solve_banded_column (columns.py:404-485) with its working-set record.

    The solve is the GPU block-Thomas kernel on column `col` (same elimination order as the batched
    solve, so the results agree with solve_banded_column on that column).  The kernel's working
    buffer is one 6x6 tile per layer by construction (36 scalars, reloaded per layer), so the record
    is exact: L diagonal-tile loads, 2 propagation-tile stores per layer but the last, one factored
    diagonal per layer, touching d[l], u[l] (l >= 1) and w[l] (l <= L-2)."""
    rhs_a = rhs.cpu().numpy() if isinstance(rhs, torch.Tensor) else np.asarray(rhs)
    if rhs_a.shape[0] != 1:
        raise ShapeMismatch("sequential solver expects a single-column RHS")
    one = BandedColumnMatrix(d=np.asarray(mat.d)[col:col + 1], u=np.asarray(mat.u)[col:col + 1],
                             w=np.asarray(mat.w)[col:col + 1])
    x = solve_banded_column(one, rhs_a)
    st = stats if stats is not None else AccessStats()
    L = int(np.asarray(mat.d).shape[1])
    st.max_live = max(st.max_live, 36)
    st.loads += L
    st.stores += 2 * (L - 1) + L
    st.touched |= {("d", l) for l in range(L)} | {("u", l) for l in range(1, L)} | {("w", l) for l in range(L - 1)}
    return x, st


def solve_tridiagonal(lower, diag, upper, rhs):
    """Batched Thomas algorithm over leading dimensions (columns.py:507-531)."""
    dev = _dev()
    A = Arr()
    lo, di, up, rh = (A.dev(a, dev) for a in (lower, diag, upper, rhs))
    shape = di.shape
    n = shape[-1]
    nb = int(np.prod(shape[:-1])) if len(shape) > 1 else 1

    def cm(a):
        return torch.broadcast_to(a, shape).reshape(nb, n).t().contiguous()   # [n][nb]
    lo, di, up, rh = cm(lo), cm(di), cm(up), cm(rh)
    x = torch.empty_like(di)
    work = torch.empty_like(di)
    err = _err_word(dev)
    _lib.check(_lib.lib().pdg_solve_tridiagonal(nb, n, ptr(lo), ptr(di), ptr(up), ptr(rh), ptr(x), ptr(work),
                                                ptr(err), stream_ptr()), "tridiagonal")
    _err_check(err)
    return A.out(x.t().reshape(shape).contiguous())

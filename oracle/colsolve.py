"""Column solvers restated (prismdg/columns.py).  Oracle / test infrastructure only.

Column systems are (ncol, L, 6[, nc]); unknowns layer-major, top layer first,
top-face nodes before bottom-face nodes.
"""
from types import SimpleNamespace

import numpy as np

from paper_2605_16082_b200.errors import ShapeMismatch, ZeroPivot
from .ext2d import mh_inv_apply


def _as4(rhs):
    a = np.asarray(rhs)
    if a.ndim == 3:
        return a[..., None], False
    if a.ndim != 4 or a.shape[2] != 6:
        raise ShapeMismatch(f"column RHS must be (ncol, L, 6[, nc]), got {a.shape}")
    return a, True


def sweep_r(rhs, j2d):
    """columns.py:95-122: top-down; s += g_t + g_b, r_t = -s + 2 g_b, r_b = -s."""
    f, had = _as4(rhs)
    out = np.zeros_like(f)
    s = np.zeros((f.shape[0], 3, f.shape[3]), f.dtype)
    jj = np.asarray(j2d)
    for l in range(f.shape[1]):
        gt = mh_inv_apply(f[:, l, 0:3], jj)
        gb = mh_inv_apply(f[:, l, 3:6], jj)
        s = s + (gt + gb)
        out[:, l, 0:3] = -s + 2.0 * gb
        out[:, l, 3:6] = -s
    return out if had else out[..., 0]


def sweep_w(rhs, j2d):
    """columns.py:125-151: bottom-up; w_b = s + g_b - g_t, w_t = s + g_b + g_t."""
    f, had = _as4(rhs)
    out = np.zeros_like(f)
    s = np.zeros((f.shape[0], 3, f.shape[3]), f.dtype)
    jj = np.asarray(j2d)
    for l in range(f.shape[1] - 1, -1, -1):
        gt = mh_inv_apply(f[:, l, 0:3], jj)
        gb = mh_inv_apply(f[:, l, 3:6], jj)
        wb = s + gb - gt
        wt = s + gb + gt
        s = wt
        out[:, l, 0:3] = wt
        out[:, l, 3:6] = wb
    return out if had else out[..., 0]


def dense_sweep_matrix(kind, L, mh):
    """columns.py:154-188: literal D_vu ('r') / D_vd ('w') operators."""
    a = np.zeros((6 * L, 6 * L))

    def put(r, c, blk):
        a[3 * r:3 * r + 3, 3 * c:3 * c + 3] += blk
    for l in range(L):
        t, b = 2 * l, 2 * l + 1
        if kind == "r":
            put(t, t, -0.5 * mh); put(t, b, -0.5 * mh); put(b, t, 0.5 * mh); put(b, b, -0.5 * mh)
            if l > 0:
                put(t, 2 * l - 1, mh)
        elif kind == "w":
            put(t, t, 0.5 * mh); put(t, b, -0.5 * mh); put(b, t, 0.5 * mh); put(b, b, 0.5 * mh)
            if l < L - 1:
                put(b, 2 * (l + 1), -mh)
        else:
            raise ValueError(kind)
    return a


def Banded(d, u, w):
    return SimpleNamespace(d=d, u=u, w=w, layers=None)


def lu6(a, layer):
    """columns.py:266-277: unpivoted in-place LU of (n, 6, 6)."""
    for k in range(6):
        piv = a[:, k, k]
        if np.any(piv == 0.0):
            raise ZeroPivot(layer, k)
        inv = 1.0 / piv
        for i in range(k + 1, 6):
            a[:, i, k] = a[:, i, k] * inv
            for j in range(k + 1, 6):
                a[:, i, j] = a[:, i, j] - a[:, i, k] * a[:, k, j]
    return a


def lu6_solve(a, b):
    """columns.py:280-289: b (n, 6, nrhs) overwritten."""
    for i in range(1, 6):
        for j in range(i):
            b[:, i] = b[:, i] - a[:, i, j, None] * b[:, j]
    for i in range(5, -1, -1):
        for j in range(i + 1, 6):
            b[:, i] = b[:, i] - a[:, i, j, None] * b[:, j]
        b[:, i] = b[:, i] / a[:, i, i, None]
    return b


def block_thomas(mat, rhs):
    """columns.py:292-348: forward fold/factor/propagate, backward substitute."""
    f, had = _as4(rhs)
    d, u, w = mat.d, mat.u.copy(), mat.w.copy()
    n, L = d.shape[0], d.shape[1]
    if f.shape[0] != n or f.shape[1] != L:
        raise ShapeMismatch(f"rhs shape {f.shape} does not match matrix ({n}, {L})")
    nc = f.shape[3]
    g = f.astype(d.dtype).copy()
    for l in range(L):
        a = d[:, l].copy()
        if l > 0:
            G = np.concatenate([u[:, l - 1], w[:, l - 1]], axis=1)
            for i in range(3):
                for j in range(6):
                    acc = np.zeros(n)
                    for k in range(6):
                        acc = acc + u[:, l, i, k] * G[:, k, j]
                    a[:, i, j] = a[:, i, j] - acc
            for i in range(3):
                for c in range(nc):
                    acc = np.zeros(n)
                    for k in range(6):
                        acc = acc + u[:, l, i, k] * g[:, l - 1, k, c]
                    g[:, l, i, c] = g[:, l, i, c] - acc
        lu6(a, l)
        if l < L - 1:
            t = np.zeros((n, 6, 6))
            t[:, 3:6] = w[:, l]
            lu6_solve(a, t)
            u[:, l], w[:, l] = t[:, 0:3], t[:, 3:6]
        g[:, l] = lu6_solve(a, g[:, l].copy())
    x = np.zeros_like(g)
    x[:, L - 1] = g[:, L - 1]
    for l in range(L - 2, -1, -1):
        G = np.concatenate([u[:, l], w[:, l]], axis=1)
        for i in range(6):
            for c in range(nc):
                acc = np.zeros(n)
                for k in range(6):
                    acc = acc + G[:, i, k] * x[:, l + 1, k, c]
                x[:, l, i, c] = g[:, l, i, c] - acc
    return x if had else x[..., 0]


def banded_matvec(mat, x):
    """columns.py:356-366."""
    f, had = _as4(x)
    n, L = mat.d.shape[0], mat.d.shape[1]
    if f.shape[0] != n or f.shape[1] != L:
        raise ShapeMismatch(f"operand shape {f.shape} does not match matrix ({n}, {L})")
    y = np.einsum("clij,cljn->clin", mat.d, f)
    if L > 1:
        y[:, 1:, 0:3] += np.einsum("clij,cljn->clin", mat.u[:, 1:], f[:, :-1])
        y[:, :-1, 3:6] += np.einsum("clij,cljn->clin", mat.w[:, :-1], f[:, 1:])
    return y if had else y[..., 0]


def banded_dense(mat, col):
    """columns.py:252-263."""
    L = mat.d.shape[1]
    a = np.zeros((6 * L, 6 * L))
    for l in range(L):
        r = 6 * l
        a[r:r + 6, r:r + 6] = mat.d[col, l]
        if l > 0:
            a[r:r + 3, r - 6:r] = mat.u[col, l]
        if l < L - 1:
            a[r + 3:r + 6, r + 6:r + 12] = mat.w[col, l]
    return a


def thomas(lower, diag, upper, rhs):
    """columns.py:507-531: batched scalar Thomas."""
    a = np.asarray(lower, float)
    b = np.asarray(diag, float).copy()
    c = np.asarray(upper, float)
    d = np.asarray(rhs, float).copy()
    n = b.shape[-1]
    for i in range(1, n):
        piv = b[..., i - 1]
        if np.any(piv == 0.0):
            raise ZeroPivot(i - 1, 0)
        m = a[..., i] / piv
        b[..., i] = b[..., i] - m * c[..., i - 1]
        d[..., i] = d[..., i] - m * d[..., i - 1]
    if np.any(b[..., n - 1] == 0.0):
        raise ZeroPivot(n - 1, 0)
    x = np.empty_like(d)
    x[..., n - 1] = d[..., n - 1] / b[..., n - 1]
    for i in range(n - 2, -1, -1):
        x[..., i] = (d[..., i] - c[..., i] * x[..., i + 1]) / b[..., i]
    return x

"""Column patches of a large mesh for sampled-column parity (test infrastructure).

Every reference assembly is gather-only and `els`-subset invariant: the
rows of a column depend only on the column and its edge neighbours (one ring per RHS evaluation).
So the oracle can be evaluated on a small patch -- the sampled columns plus `depth` rings of
neighbours -- and its rows for the sampled columns equal the full-mesh rows.  The outermost
ring's missing neighbours become walls; those columns are never compared.
"""
import numpy as np

from oracle.geom import OMesh
from oracle.tables import BTAG_WALL


def build_patch(mesh, cols, depth):
    """(ids, om): ids = global column ids of the patch (the sampled `cols` first, then the rings
    in BFS order); om = an oracle mesh over them with neighbours remapped to patch ids."""
    nt = mesh.nt
    nbr = np.asarray(mesh.nbr)
    seen = np.zeros(nt, bool)
    cols = np.asarray(cols, np.int64)
    seen[cols] = True
    order = [cols]
    front = cols
    for _ in range(depth):
        nb = nbr[front].ravel()
        nb = np.unique(nb[nb >= 0])
        nb = nb[~seen[nb]]
        seen[nb] = True
        order.append(nb)
        front = nb
    ids = np.concatenate(order)
    g2l = np.full(nt, -1, np.int64)
    g2l[ids] = np.arange(ids.size)
    sub = {k: np.ascontiguousarray(np.asarray(getattr(mesh, k))[ids])
           for k in ("j2d", "dphx", "dphy", "elen", "enx", "eny", "b", "x", "y", "tri", "nbrk", "btag")}
    gn = nbr[ids]
    ln = np.where(gn >= 0, g2l[np.maximum(gn, 0)], -1)
    cut = (gn >= 0) & (ln < 0)                       # neighbour outside the patch
    sub["btag"] = np.where(cut, BTAG_WALL, sub["btag"]).astype(np.int64)
    sub["nbrk"] = np.where(cut, -1, sub["nbrk"]).astype(np.int64)
    om = OMesh(vx=np.asarray(mesh.vx), vy=np.asarray(mesh.vy), vb=np.asarray(mesh.vb), nbr=ln.astype(np.int64),
               **{k: v for k, v in sub.items() if k not in ("nbr",)})
    return ids, om


# ---------------------------------------------------------------- device planes -> reference rows

def rows_p6(X, ids):
    """[6][L][nt] -> (n L, 6) of the patch columns."""
    import torch
    t = X[:, :, torch.as_tensor(ids, device=X.device)]
    n, L = len(ids), X.shape[1]
    return t.permute(2, 1, 0).reshape(n * L, 6).cpu().numpy()


def rows_pv(X, ids):
    """[nc][6][L][nt] -> (n L, 6, nc)."""
    import torch
    t = X[:, :, :, torch.as_tensor(ids, device=X.device)]
    n, L, nc = len(ids), X.shape[2], X.shape[0]
    return t.permute(3, 2, 1, 0).reshape(n * L, 6, nc).cpu().numpy()


def rows_c3(X, ids):
    """[3][nt] -> (n, 3);  [nc][3][nt] -> (n, 3, nc)."""
    import torch
    i = torch.as_tensor(ids, device=X.device)
    if X.dim() == 2:
        return X[:, i].t().cpu().numpy()
    return X[:, :, i].permute(2, 1, 0).cpu().numpy()

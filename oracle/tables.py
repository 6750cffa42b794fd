"""Reference-element constants (restated from prismdg/dg.py:27-88, internal3d.py:57-65).

Oracle / test infrastructure only.
"""
import math

import numpy as np

# Dunavant degree-4 six-point rule on the unit triangle (dg.py:27-45).
_a1, _b1, _w1 = 0.108103018168070, 0.445948490915965, 0.111690794839005
_a2, _b2, _w2 = 0.816847572980459, 0.091576213509771, 0.054975871827661
QW = np.array([_w1, _w1, _w1, _w2, _w2, _w2])
BARY = np.array([[_a1, _b1, _b1], [_b1, _a1, _b1], [_b1, _b1, _a1],
                 [_a2, _b2, _b2], [_b2, _a2, _b2], [_b2, _b2, _a2]])

# two-point Gauss on [-1, 1] (dg.py:54-67)
GZ = 1.0 / math.sqrt(3.0)
ZQP = np.array([-GZ, GZ])
ZQW = np.array([1.0, 1.0])
# VS[v, lev]: value at vertical point v of the level-lev shape (0 = top)
VS = np.array([[(1.0 - GZ) / 2.0, (1.0 + GZ) / 2.0],
               [(1.0 + GZ) / 2.0, (1.0 - GZ) / 2.0]])
DV = np.array([0.5, -0.5])
# ES[h, s]: edge shape s at edge point h, own traversal order (dg.py:76-81)
ES = np.array([[(1.0 + GZ) / 2.0, (1.0 - GZ) / 2.0],
               [(1.0 - GZ) / 2.0, (1.0 + GZ) / 2.0]])
EV0 = np.array([0, 1, 2])
EV1 = np.array([1, 2, 0])

# tensor-rule tables (internal3d.py:57-65)
W12 = ZQW[:, None] * QW[None, :]                       # (v, q)
PHI12 = np.zeros((2, 6, 6))                            # (v, q, node)
DPHIZ = np.zeros((6, 6))                               # (q, node)
for node in range(6):
    lev, vtx = divmod(node, 3)
    PHI12[:, :, node] = np.outer(VS[:, lev], BARY[:, vtx])
    DPHIZ[:, node] = DV[lev] * BARY[:, vtx]

# triangle mass pattern (columns.py:35-36)
MH = np.array([[2.0, 1.0, 1.0], [1.0, 2.0, 1.0], [1.0, 1.0, 2.0]]) / 24.0

BTAG_INTERIOR, BTAG_WALL, BTAG_OPEN = 0, 1, 2


def penalty_sigma(l_int, l_ext, dim=3, n0=5.0, order=1):
    """dg.py:161-173: N0 (o+1)(o+d) / (2 d min(L_i, L_e))."""
    lmin = np.minimum(np.asarray(l_int, float), np.asarray(l_ext, float))
    if np.any(lmin <= 0.0):
        raise ValueError("penalty length scale must be positive")
    return n0 * (order + 1.0) * (order + dim) / (2.0 * dim * lmin)

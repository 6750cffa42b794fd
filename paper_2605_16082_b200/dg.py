"""Reference-element tables and the pointwise DG helpers of the reference's dg.py (dg.py:27-275).

The tables are the constants the CUDA kernels compile in (csrc/common.cuh); the helpers take numpy
arrays or torch tensors like the other drop-in modules and evaluate on the device (elementwise
torch ops -- none of them is on the hot path, where the kernels inline the same formulas).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from .device import Arr, require_cuda
from .errors import DegenerateLayer, NonPositiveLength
from .params import PenaltyParams

# ---------------------------------------------------------------- tables (dg.py:27-88)
_A1, _B1, _W1 = 0.108103018168070, 0.445948490915965, 0.111690794839005
_A2, _B2, _W2 = 0.816847572980459, 0.091576213509771, 0.054975871827661
TRI_QW = np.array([_W1, _W1, _W1, _W2, _W2, _W2])
TRI_BARY = np.array([[_A1, _B1, _B1], [_B1, _A1, _B1], [_B1, _B1, _A1],
                     [_A2, _B2, _B2], [_B2, _A2, _B2], [_B2, _B2, _A2]])
TRI_QP = TRI_BARY[:, 1:].copy()
NQ_TRI = 6
_G = 1.0 / math.sqrt(3.0)
SEG_QP = np.array([-_G, _G])
SEG_QW = np.array([1.0, 1.0])
NQ_SEG = 2
# vertical shapes (top, bottom) at the two Gauss points; their zeta-derivatives
VERT_SHAPE = np.array([[(1.0 - _G) / 2.0, (1.0 + _G) / 2.0], [(1.0 + _G) / 2.0, (1.0 - _G) / 2.0]])
DVERT = np.array([0.5, -0.5])
# edge-endpoint shapes at the two edge points in the edge's own traversal order; exterior traces
# use the swapped columns (bitwise antisymmetric shared-edge fluxes)
EDGE_SHAPE = np.array([[(1.0 + _G) / 2.0, (1.0 - _G) / 2.0], [(1.0 - _G) / 2.0, (1.0 + _G) / 2.0]])
EDGE_V0 = np.array([0, 1, 2])
EDGE_V1 = np.array([1, 2, 0])
DPHI_PARENT = np.array([[-1.0, -1.0], [1.0, 0.0], [0.0, 1.0]])


@dataclass(frozen=True)
class ReferenceElement:
    tri_qp: np.ndarray = None
    tri_qw: np.ndarray = None
    tri_bary: np.ndarray = None
    seg_qp: np.ndarray = None
    seg_qw: np.ndarray = None
    vert_shape: np.ndarray = None
    edge_shape: np.ndarray = None

    @staticmethod
    def make() -> "ReferenceElement":
        return ReferenceElement(TRI_QP, TRI_QW, TRI_BARY, SEG_QP, SEG_QW, VERT_SHAPE, EDGE_SHAPE)


def _dev():
    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


# ---------------------------------------------------------------- helpers (dg.py:116-275)
def tri_quad(values_at_qp):
    """sum_q TRI_QW[q] v[..., q]."""
    A = Arr()
    v = A.dev(values_at_qp, _dev())
    return A.out(v @ torch.as_tensor(TRI_QW, device=v.device))


def iface_mean(v_int, v_ext):
    A = Arr()
    d = _dev()
    return A.out((A.dev(v_int, d) + A.dev(v_ext, d)) * 0.5)


def iface_diff(v_int, v_ext):
    A = Arr()
    d = _dev()
    return A.out((A.dev(v_int, d) - A.dev(v_ext, d)) * 0.5)


def iface_max(v_int, v_ext):
    A = Arr()
    d = _dev()
    return A.out(torch.maximum(A.dev(v_int, d), A.dev(v_ext, d)))


def iface_upwind(v_int, v_ext, sign):
    """interior where sign >= 0 (ties pick the interior side), exterior otherwise."""
    A = Arr()
    d = _dev()
    a, b, s = A.dev(v_int, d), A.dev(v_ext, d), A.dev(sign, d)
    return A.out(torch.where(s >= 0.0, a, b))


def penalty_sigma(l_int, l_ext, dim=3, params: PenaltyParams = PenaltyParams()):
    """N0 (o+1)(o+d) / (2 d min(L_int, L_ext)); NonPositiveLength if a length is <= 0."""
    A = Arr()
    d = _dev()
    lmin = torch.minimum(A.dev(l_int, d), A.dev(l_ext, d))
    if bool((lmin <= 0.0).any().item()):
        raise NonPositiveLength("penalty length scale must be positive")
    o = params.order
    return A.out(params.n0 * (o + 1.0) * (o + dim) / (2.0 * dim * lmin))


def metric_vector(dz_mid, dz_jz, jz, zeta):
    """m_z = 1/Jz, m_h = -(grad z_mid + zeta grad Jz)/Jz; DegenerateLayer if Jz <= 0."""
    A = Arr()
    d = _dev()
    j = A.dev(jz, d)
    if bool((j <= 0.0).any().item()):
        raise DegenerateLayer("layer half-thickness must be positive")
    z = A.dev(zeta, d)
    mh = -(A.dev(dz_mid, d) + z[..., None] * A.dev(dz_jz, d)) / j[..., None]
    return A.out(mh), A.out(1.0 / j)


def gradient_decompose(dfdxi_phys, dfdzeta, m_h, m_z):
    """(grad_iso, grad_m): iso-zeta part (z component 0) and the metric part m * df/dzeta."""
    A = Arr()
    d = _dev()
    gx, fz = A.dev(dfdxi_phys, d), A.dev(dfdzeta, d)
    zero = torch.zeros_like(fz)
    giso = torch.cat([gx, zero[..., None]], dim=-1)
    gm = torch.cat([A.dev(m_h, d) * fz[..., None], (A.dev(m_z, d) * fz)[..., None]], dim=-1)
    return A.out(giso), A.out(gm)


def split_velocity(u, w, m_h, m_z):
    """utilde = (u, v, -m_h.u/m_z) (tangent to iso-zeta), wtilde = w + m_h.u/m_z."""
    A = Arr()
    d = _dev()
    uu, mh = A.dev(u, d), A.dev(m_h, d)
    aux = (uu[..., 0] * mh[..., 0] + uu[..., 1] * mh[..., 1]) / A.dev(m_z, d)
    return A.out(torch.cat([uu, (-aux)[..., None]], dim=-1)), A.out(A.dev(w, d) + aux)


@dataclass(frozen=True)
class TensorDiffusivity:
    kappa_i: np.ndarray   # implicit scalar vertical part
    d_e: np.ndarray       # explicit remainder, m . D_e . m = 0


def split_diffusivity(d_tensor, m_h, m_z):
    """D = D_i + D_e with D_i = ((m.D.m)/m_z^2) e_z e_z."""
    A = Arr()
    d = _dev()
    D, mz = A.dev(d_tensor, d), A.dev(m_z, d)
    m = torch.cat([A.dev(m_h, d), mz[..., None]], dim=-1)
    k = torch.einsum("...i,...ij,...j->...", m, D, m) / (mz * mz)
    de = D.clone()
    de[..., 2, 2] -= k
    return TensorDiffusivity(kappa_i=A.out(k), d_e=A.out(de))


def kappa_implicit(kh, kv, m_h, m_z):
    """kv + kh |m_h|^2 / m_z^2 (split_diffusivity for D = diag(kh, kh, kv))."""
    A = Arr()
    d = _dev()
    mh = A.dev(m_h, d)
    return A.out(kv + kh * (mh[..., 0] ** 2 + mh[..., 1] ** 2) / (A.dev(m_z, d) ** 2))

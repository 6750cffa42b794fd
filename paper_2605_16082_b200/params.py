"""Argument / result containers of the drop-in API.

Field names and defaults mirror the reference dataclasses so user code that
builds them keeps working: PhysParams / State2D / ExternalResult
(external2d.py:39-78, 286-293), PenaltyParams (dg.py:155-158),
BandedColumnMatrix (columns.py:196-227), LayerPolicy (mesh.py:279-305).
Arrays may be numpy (host) or torch CUDA tensors (device, zero-copy path).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Any, Optional

import numpy as np


@dataclass
class PhysParams:
    g: float = 9.81
    rho0: float = 1025.0
    f: float = 0.0
    cd: float = 0.0
    tau_x: float = 0.0
    tau_y: float = 0.0
    tau_x1: Optional[float] = None
    tau_y1: Optional[float] = None
    wind_t0: float = 0.0
    wind_t1: float = 0.0
    kappa_h: float = 0.0
    kappa_v: float = 0.0
    nu_h: float = 0.0
    nu_v: float = 0.0
    alpha: float = 0.0
    beta: float = 0.0
    t_ref: float = 10.0
    s_ref: float = 35.0

    def wind(self, t: float):
        """Kinematic surface stress (tau / rho0) at time t (external2d.py:60-67)."""
        tx, ty = self.tau_x, self.tau_y
        if self.tau_x1 is not None and self.wind_t1 > self.wind_t0:
            w = float(np.clip((t - self.wind_t0) / (self.wind_t1 - self.wind_t0), 0.0, 1.0))
            tx = (1.0 - w) * self.tau_x + w * self.tau_x1
            ty = (1.0 - w) * self.tau_y + w * (self.tau_y1 if self.tau_y1 is not None else self.tau_y)
        return tx / self.rho0, ty / self.rho0


@dataclass
class State2D:
    eta: Any
    qx: Any
    qy: Any
    t: float = 0.0

    def copy(self) -> "State2D":
        return State2D(self.eta.clone() if hasattr(self.eta, "clone") else self.eta.copy(),
                       self.qx.clone() if hasattr(self.qx, "clone") else self.qx.copy(),
                       self.qy.clone() if hasattr(self.qy, "clone") else self.qy.copy(), self.t)


@dataclass
class ExternalResult:
    state: State2D
    qbar_x: Any
    qbar_y: Any
    f2d_x: Any
    f2d_y: Any
    steps: int = 0


@dataclass(frozen=True)
class PenaltyParams:
    n0: float = 5.0
    order: int = 1


@dataclass
class BandedColumnMatrix:
    d: Any   # (ncol, L, 6, 6)
    u: Any   # (ncol, L, 3, 6)
    w: Any   # (ncol, L, 3, 6)
    layers: Optional[Any] = None

    @property
    def ncol(self) -> int:
        return self.d.shape[0]

    @property
    def nlay(self) -> int:
        return self.d.shape[1]

    def copy(self) -> "BandedColumnMatrix":
        def cp(a):
            return None if a is None else (a.clone() if hasattr(a, "clone") else a.copy())
        return BandedColumnMatrix(cp(self.d), cp(self.u), cp(self.w), cp(self.layers))


@dataclass(frozen=True)
class LayerPolicy:
    mode: str = "uniform"
    count: int = 1
    table: tuple = ()

    def counts(self, mesh, eta=None) -> np.ndarray:
        """mesh.py:295-305."""
        if self.mode == "uniform":
            return np.full(mesh.nt, self.count, dtype=np.int64)
        if self.mode != "by-depth":
            raise ValueError(f"unknown layer policy mode '{self.mode}'")
        e = np.zeros((mesh.nt, 3)) if eta is None else np.asarray(eta)
        depth = (e - np.asarray(mesh.b)).max(axis=1)
        out = np.full(mesh.nt, self.count, dtype=np.int64)
        for dmin, cnt in sorted(self.table):
            out[depth >= dmin] = int(cnt)
        return out

"""B200-native prism-DG hot path (drop-in for the reference `prismdg` operator API).

Submodules mirror the reference modules: `mesh`, `external2d`, `internal3d`,
`columns`; `stepper` is the fused IMEX internal step that keeps every field
resident in HBM.  Compute runs in libprismdg_b200.so (sm_100a); importing this
package does not load the library -- the first compute call does, and fails
loudly if it is missing.
"""
from . import errors, params
from .params import BandedColumnMatrix, ExternalResult, LayerPolicy, PenaltyParams, PhysParams, State2D


def __getattr__(name):
    import importlib
    if name in ("mesh", "external2d", "internal3d", "columns", "stepper", "device", "scenarios", "partition",
                "snapshot", "layout", "dg"):
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)

"""PRISMDG-SNAP 1 state snapshots: an ASCII header line

    PRISMDG-SNAP 1 <field> <components> <columns> <layers> <time>

followed by the little-endian IEEE-754 float64 payload in FieldSoA order (layout.py:33-51:
address(f, k, c, l) = (f * 6 + k) * P + c * L + l, uniform layers).  Bit-exact round trip.

The stepper's prism fields live on the device as [nc][6][L][nt]; a snapshot is the
[nc][6][nt][L] transpose of that, copied to the host once.  2D fields (eta, qx, qy: three
corner values per column) use the same header with <layers> = 0 and payload [nc][3][nt]
(an extension: SPEC.md defines the format for prism fields only).
"""
from __future__ import annotations

import numpy as np

MAGIC = "PRISMDG-SNAP"
VERSION = 1


def _header(field: str, nc: int, ncol: int, L: int, t: float) -> bytes:
    if not field or any(ch.isspace() for ch in field):
        raise ValueError(f"field name must be one non-empty token, got {field!r}")
    return f"{MAGIC} {VERSION} {field} {nc} {ncol} {L} {float(t)!r}\n".encode("ascii")


def write(path, field: str, data, L: int, t: float = 0.0) -> None:
    """data: numpy array in FieldSoA order, shape (nc, 6, ncol, L) (prism field) or (nc, 3, ncol)
    (2D field, L = 0); written bit-exactly."""
    a = np.ascontiguousarray(np.asarray(data, dtype=np.float64))
    if L > 0:
        if a.ndim != 4 or a.shape[1] != 6 or a.shape[3] != L:
            raise ValueError(f"prism field must be (nc, 6, ncol, L), got {a.shape}")
    elif a.ndim != 3 or a.shape[1] != 3:
        raise ValueError(f"2D field must be (nc, 3, ncol), got {a.shape}")
    with open(path, "wb") as f:
        f.write(_header(field, a.shape[0], a.shape[2], L, t))
        f.write(a.astype("<f8", copy=False).tobytes())


def read(path):
    """(meta dict, array in FieldSoA order); raises ValueError on a malformed or truncated file."""
    with open(path, "rb") as f:
        line = f.readline().decode("ascii").split()
        if len(line) != 7 or line[0] != MAGIC or int(line[1]) != VERSION:
            raise ValueError(f"{path}: not a {MAGIC} {VERSION} file")
        field, nc, ncol, L, t = line[2], int(line[3]), int(line[4]), int(line[5]), float(line[6])
        shape = (nc, 6, ncol, L) if L > 0 else (nc, 3, ncol)
        n = int(np.prod(shape))
        raw = f.read()
    if len(raw) != 8 * n:
        raise ValueError(f"{path}: payload has {len(raw)} bytes, header implies {8 * n}")
    return {"field": field, "components": nc, "columns": ncol, "layers": L, "time": t}, \
        np.frombuffer(raw, dtype="<f8").reshape(shape).astype(np.float64)


def from_device(t, L: int):
    """device [nc][6][L][nt] (or [6][L][nt]) -> host FieldSoA (nc, 6, nt, L); [nc][3][nt] 2D as is."""
    if L == 0:
        x = t if t.dim() == 3 else t.unsqueeze(0)
        return x.cpu().numpy()
    x = t if t.dim() == 4 else t.unsqueeze(0)
    return x.permute(0, 1, 3, 2).contiguous().cpu().numpy()


def to_device(a, L: int, device):
    """host FieldSoA -> device layout ([nc][6][L][nt] for prism fields, [nc][3][nt] for 2D)."""
    import torch
    x = torch.as_tensor(np.ascontiguousarray(a), device=device)
    if L == 0:
        return x
    return x.permute(0, 1, 3, 2).contiguous()


def save_state(stepper, prefix: str) -> list:
    """Write the stepper's prognostic state: <prefix>.{s2d,u,T}.snap (eta/qx/qy, u_x/u_y, T)."""
    L, t = stepper.L, stepper.t
    files = [(f"{prefix}.s2d.snap", "eta_qx_qy", stepper.S, 0), (f"{prefix}.u.snap", "u", stepper.U[stepper.cur], L),
             (f"{prefix}.T.snap", "T", stepper.T[stepper.cur], L)]
    for path, name, tensor, lay in files:
        write(path, name, from_device(tensor, lay), lay, t)
    return [f[0] for f in files]


def load_state(stepper, prefix: str) -> None:
    """Restore a state written by save_state (bit-exact)."""
    metas = {}
    for key, lay, dest in (("s2d", 0, stepper.S), ("u", stepper.L, stepper.U[stepper.cur]),
                           ("T", stepper.L, stepper.T[stepper.cur])):
        meta, a = read(f"{prefix}.{key}.snap")
        if meta["layers"] != lay or meta["columns"] != stepper.nt:
            raise ValueError(f"{prefix}.{key}.snap: {meta} does not match the stepper ({stepper.nt} x {lay})")
        dest.copy_(to_device(a, lay, dest.device).reshape(dest.shape))
        metas[key] = meta
    stepper.t = metas["u"]["time"]

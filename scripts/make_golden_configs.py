"""Golden trajectories of the BASELINE configs at their stated sizes, from the REAL reference.

    python scripts/make_golden_configs.py [c2] [c3] [c3w]

The reference ships no stepper: each step is the orchestrator of
oracle/stepper.py (imex_step_ops) composed from the reference's own functions
(/root/reference/pkg/src/prismdg).  Initial states: tests/config_states.py (seeded).

  c2   32x32 basin (2,048 tri) x 10 layers, dt 40 s, m 20: states after steps 1 and 100
  c3   250x100 lock exchange (50,000 tri) x 20 layers, dt 20 s, m 20: one full step, stored on
       2,048 sampled columns (the full 1 M-prism state is 144 MB)
  c3w  20x8 window of the C3 basin (same resolution) x 20 layers: states after steps 1 and 100
Writes tests/golden/cfg_<name>.npz.  Runs in the build container only (needs /root/reference).
"""
import os
import sys
import time
from types import SimpleNamespace

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
REF = "/root/reference/pkg/src"
OUT = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def ref_modules():
    from oracle import refops
    r = refops.load(REF)
    return r.RC, r.RE, r.RI, r.RM


def ref_ops():
    from oracle import refops
    return refops.load(REF).ops


def run(cfg, state_fn, keep_steps, sample=None):
    import config_states as CS
    import oracle.stepper as OS
    RC, RE, RI, RM = ref_modules()
    ops = ref_ops()
    mesh = RM.hilbert_reorder(RM.generate_basin_mesh(cfg["nx"], cfg["ny"], cfg["lx"], cfg["ly"], CS.flat_bed))
    L = cfg["L"]
    s0 = state_fn(mesh, L)
    p = RE.PhysParams(**cfg["params"])
    s = SimpleNamespace(grid=RM.extrude(mesh, RM.LayerPolicy(count=L), s0["eta"]), ux=s0["ux"], uy=s0["uy"],
                        T=s0["T"], s2d=RE.State2D(s0["eta"].copy(), s0["qx"], s0["qy"], 0.0))
    out = {}
    cols = None if sample is None else CS.sample_columns(mesh.nt, sample)
    if cols is not None:
        out["cols"] = cols
    pr = None if cols is None else (cols[:, None] * L + np.arange(L)[None, :]).ravel()
    t0 = time.time()
    for i in range(1, max(keep_steps) + 1):
        s = OS.imex_step_ops(ops, s, p, cfg["dt"], cfg["m"], cfg["kv"], cfg["nu_v"])
        if i in keep_steps:
            for n, a in (("ux", s.ux), ("uy", s.uy), ("T", s.T)):
                out[f"s{i}_{n}"] = a if pr is None else a[pr]
            for n, a in (("eta", s.s2d.eta), ("qx", s.s2d.qx), ("qy", s.s2d.qy)):
                out[f"s{i}_{n}"] = a if cols is None else a[cols]
        print(f"  step {i} ({time.time() - t0:.1f} s)", flush=True)
    out["in_sum"] = np.array([float(np.sum(np.abs(v))) for v in (s0[k] for k in ("eta", "qx", "qy", "ux", "uy", "T"))])
    out["numpy_version"] = np.array(np.__version__)
    return out


def main():
    import config_states as CS
    which = sys.argv[1:] or ["c2", "c3w", "c3"]
    os.makedirs(OUT, exist_ok=True)
    for name in which:
        print(name, flush=True)
        if name == "c2":
            out = run(CS.C2, CS.c2_state, (1, 100))
        elif name == "c3w":
            out = run(CS.C3W, lambda m, L: CS.c3_state(m, L, CS.C3W["lx"]), (1, 100))
        elif name == "c3":
            out = run(CS.C3, lambda m, L: CS.c3_state(m, L, CS.C3["lx"]), (1,), sample=2048)
        else:
            raise SystemExit(f"unknown config {name}")
        np.savez_compressed(os.path.join(OUT, f"cfg_{name}.npz"), **out)
        print("wrote", os.path.join(OUT, f"cfg_{name}.npz"), flush=True)


if __name__ == "__main__":
    main()

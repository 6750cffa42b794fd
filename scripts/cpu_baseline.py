"""SURVEY.md section 8d CPU baseline legs, timed on this host with the REFERENCE's own functions.

    python scripts/cpu_baseline.py [--out FILE] [--skip-c3-step] [--procs N]

(i)  single process (numpy ~ 1 core): full steps of C1 (2D only: SSP-RK3 steps of the external
     mode, 2D-DOF = 3 nt per step), C2 and C3 at their stated sizes, the reference functions
     composed by the shared orchestrator (oracle/stepper.imex_step_ops; the reference has no stepper)
(ii) all cores: one RHS evaluation of each hot-path function at C3, `els`-chunked over processes
     (every reference assembly is els-subset invariant; fork workers share
     the inputs copy-on-write and return only their rows); C4 (50 M prisms) does not fit this
     host's memory for that scheme, so its figures are EXTRAPOLATED per prism from C3 and
     labelled so, like the full C4 step
plus the host: nproc, CPU model, numpy.show_config().  Test / measurement infrastructure only.
"""
import argparse
import io
import json
import multiprocessing as mp
import os
import sys
import time
from contextlib import redirect_stdout

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ[_v] = "1"
os.environ.setdefault("PDG_MESH_HOST", "1")

import numpy as np  # noqa: E402

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)

_G = {}   # fork-shared inputs of the (ii) leg


def _host():
    model = None
    with open("/proc/cpuinfo") as f:
        for ln in f:
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    buf = io.StringIO()
    with redirect_stdout(buf):
        np.show_config()
    return {"nproc": os.cpu_count(), "cpu_model": model, "numpy": np.__version__, "numpy_show_config": buf.getvalue()}


def _ref_case(name):
    from oracle import refops
    from paper_2605_16082_b200.scenarios import make_case
    ref = refops.load()
    c = make_case(name)
    s, p = refops.initial(ref, (c.mesh.vx, c.mesh.vy, c.mesh.vb, c.mesh.tri), c.L, c.state, c.params)
    return ref, c, s, p


def leg_single(name, steps):
    from oracle import stepper as OS
    ref, c, s, p = _ref_case(name)
    t = []
    if name == "c1":   # 2D external mode only: `steps` SSP-RK3 steps (subcycle_external, dt2d = 2 s)
        for _ in range(2):
            t0 = time.perf_counter()
            ref.RE.subcycle_external(s.s2d, s.grid.mesh, p, steps, c.dt2d)
            t.append(time.perf_counter() - t0)
        per = min(t) / steps
        dof = 3 * c.mesh.nt
        return {"config": name, "nt": c.mesh.nt, "ssp_rk3_steps": steps, "s_per_step": per,
                "value": dof / per, "unit": "2D-DOF/s (3 nt per SSP-RK3 step)", "cores": 1}
    for _ in range(steps):
        t0 = time.perf_counter()
        s = OS.imex_step_ops(ref.ops, s, p, c.dt, c.m, c.kv, c.nu_v)
        t.append(time.perf_counter() - t0)
    per = float(np.mean(t))
    return {"config": name, "prisms": c.prisms, "L": c.L, "m": c.m, "steps": steps, "s_per_step": per,
            "value": 6.0 * c.prisms / per, "unit": "prism-DOF/s", "cores": 1}


def _rhs_worker(args):
    fname, chunk = args
    g = _G
    RI, grid, p = g["RI"], g["grid"], g["p"]
    nt, L = grid.mesh.nt, grid.n_layers
    els = np.arange(chunk[0], chunk[1])
    t0 = time.perf_counter()
    if fname == "compute_r":
        out = RI.compute_r(grid, g["rho"], p, els=els)
    elif fname == "project_transport":
        out = RI.project_transport(grid, g["ux"], g["uy"], els=els, mass=g["M"])
    elif fname == "lateral_flux_factor":
        out = RI.lateral_flux_factor(grid, g["q"], p, els=els)
    elif fname == "horizontal_rhs":
        out = RI.horizontal_rhs(grid, g["ux"], g["uy"], g["q"], g["fac"], g["r"], g["M"], p, els=els)
    elif fname == "tracer_horizontal_rhs":
        out = RI.tracer_horizontal_rhs(grid, g["T"], g["q"], g["fac"], p, els=els)
    elif fname == "compute_wtilde":
        out = RI.compute_wtilde(grid, g["q"], g["fac"], els=els)
    elif fname == "assemble_vertical_operator":
        out = RI.assemble_vertical_operator(grid, g["wt"], grid.w_m, 0.0, 1e-4, els=els).d
    else:
        raise ValueError(fname)
    dt = time.perf_counter() - t0
    o = np.asarray(out)
    rows = o.reshape(nt, L, -1)[els] if fname != "assemble_vertical_operator" else o
    return dt, rows.nbytes


def leg_chunked(name, procs):
    ref, c, s, p = _ref_case(name)
    RI, RE = ref.RI, ref.RE
    grid = s.grid
    rng = np.random.default_rng(0)
    P = c.prisms
    ux, uy = 0.05 * rng.standard_normal((P, 6)), 0.05 * rng.standard_normal((P, 6))
    T = np.asarray(s.T)
    M = RI.prism_mass(grid)
    q = RI.project_transport(grid, ux, uy, mass=M)
    fac = RI.lateral_flux_factor(grid, q, p)
    rho = RE.eos_density(T, p)
    r = RI.compute_r(grid, rho, p)
    wt = RI.compute_wtilde(grid, q, fac)
    _G.update(RI=RI, grid=grid, p=p, ux=ux, uy=uy, T=T, M=M, q=q, fac=fac, rho=rho, r=r, wt=wt)
    nt = c.mesh.nt
    bounds = np.linspace(0, nt, procs + 1).astype(int)
    chunks = [(int(a), int(b)) for a, b in zip(bounds[:-1], bounds[1:])]
    res = {}
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        for fname in ("compute_r", "project_transport", "lateral_flux_factor", "horizontal_rhs",
                      "tracer_horizontal_rhs", "compute_wtilde", "assemble_vertical_operator"):
            pool.map(_rhs_worker, [(fname, (0, min(nt, 8)))] * procs)          # warm the workers
            t0 = time.perf_counter()
            out = pool.map(_rhs_worker, [(fname, ch) for ch in chunks])
            wall = time.perf_counter() - t0
            res[fname] = {"wall_s": wall, "max_worker_s": max(o[0] for o in out), "prisms_per_s": P / wall}
    return {"config": name, "prisms": P, "procs": procs, "functions": res}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_cpu_baseline.json"))
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    ap.add_argument("--skip-c3-step", action="store_true")
    ap.add_argument("--single-from", default=None, help="reuse the (i) legs of an earlier report")
    a = ap.parse_args()
    rep = {"host": _host(), "kind": "reference (unmodified prismdg functions; oracle/stepper.py orchestration)"}
    if a.single_from:
        with open(a.single_from) as f:
            rep["single"] = json.load(f)["single"]
    else:
        rep["single"] = [leg_single("c1", 100), leg_single("c2", 2)]
        if not a.skip_c3_step:
            rep["single"].append(leg_single("c3", 1))
    print(json.dumps(rep["single"]), flush=True)
    c3 = leg_chunked("c3", a.procs)
    rep["chunked"] = [c3]
    c4_prisms = 1_000_000 * 50
    rep["chunked_c4_extrapolated"] = {
        "label": "EXTRAPOLATED per prism from the C3 all-core timings (C4 inputs do not fit this scheme in host RAM)",
        "prisms": c4_prisms, "procs": a.procs,
        "functions": {k: {"wall_s": v["wall_s"] * c4_prisms / c3["prisms"]} for k, v in c3["functions"].items()}}
    c3s = [x for x in rep["single"] if x["config"] == "c3"]
    if c3s:
        rep["c4_full_step_extrapolated"] = {
            "label": "EXTRAPOLATED per prism from the single-process C3 step (a C4 step needs ~280 GB)",
            "s_per_step": c3s[0]["s_per_step"] * c4_prisms / c3s[0]["prisms"]}
    with open(a.out, "w") as f:
        json.dump(rep, f, indent=1)
    print(json.dumps({k: v for k, v in rep.items() if k != "host"})[:3000])


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark: prism-DOF updates/s of the full FP64 internal+external IMEX step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

Workload (N=1): config 4 of BASELINE.json -- synthetic coastal basin, 1,000,000 Hilbert-ordered
triangles x 50 sigma layers (50 M prisms, 3e8 prism DOF), dt2d = 0.5 s, m = 20 external substeps
(stage 1: m/2, stage 2: m), momentum (2 comps) + tracer, FP64.  A "step" is one full internal step:
both IMEX stages, both external sub-cycles.  Inputs (~48 GB of fields) are far larger than L2.

value     device-resident throughput: W warm-up steps, K timed steps (one CUDA graph each),
          CUDA events on the launching stream, barrier + synchronize on both sides, max over ranks.
e2e       same metric through the public API with HOST (pinned) buffers: every step uploads the
          full state from host memory, steps, and downloads it again (copies inside the timed region).
roofline  dominant kernel: algorithmic bytes / CUDA-event launch duration vs MEASURED_PEAKS.json hbm_gbs.
cpu_baseline  the CPU oracle (numpy restatement of the reference, oracle/) on a bounded sample.
--impl reference  times that CPU path (the reference arm) with all host cores, same metric.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "prism-DOF updates/s (FP64 RK step)"
UNIT = "prism-DOF/s"

# compulsory (algorithmic) HBM bytes per prism for each stepper launch: the
# prism fields each launch must read and write once; per-column 2D data, neighbour traces and
# geometry (recomputed from eta, b and the sigma fractions) are not counted
KERNEL_BYTES = {
    "r": 48 + 96,                       # read T, write r (2 comps)
    "project": 96 + 96,                 # read u, write q
    "f3d2d": 96 * 2,                    # read u, q -> 2D only (r enters as its per-column layer sum)
    "wtilde": 96 + 48,                  # read q, write w~
    "rhs_u": 96 * 4 + 96,               # read u, u0, q, r; write rhs
    "rhs_T": 48 + 48 + 96 + 48,         # read T, T0, q; write rhs
    # the stage RHS also forms w~ (pdg_step_rhs_ut_w): + write w~ 48 (PDG_NO_FUSEWT=1: separate wtilde)
    "rhs_uT_s1": 96 * 3 + 48 + 96 + 48 + 48,   # stage 1 (u0 = u, T0 = T): read u, q, r, T; write rhs_u, rhs_T, w~ = 528
    "rhs_uT_s2": 96 * 4 + 48 * 2 + 96 + 48 + 48,   # stage 2: + u0, T0 = 672
    "vertical_u_impl": 96 + 48 + 96,    # read rhs, w~; write u1
    "vertical_T_impl": 48 + 48 + 48,
    "vertical_u_expl": 96 + 48 + 96 + 96,   # + u for A u
    "vertical_T_expl": 48 + 48 + 48 + 48,
}
# 2D sub-cycle, SURVEY.md section 8d model M2: per triangle and SSP-RK3 substep 3 evaluations x
# (state 72 + geometry incl. b 194) + 2 x 72 substep-start reads + 3 x 72 writes + 96 Qbar = 1254 B.
# (Part of the 1 M-triangle 2D working set stays in the 126 MB L2 between RK stages, so the
# measured DRAM traffic per substep is below this count: profiles/<round>_traffic.json.)
RK_SUBSTEP_BYTES_PER_TRI = 3 * (72 + 194) + 2 * 72 + 3 * 72 + 96
M2_BYTES_PER_PRISM = lambda L, m: 2736 + 1881.0 * m / L  # noqa: E731  (SURVEY.md section 8d model M2)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, pw, reasons = [], None, [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            try:
                pw.append(float(f[2]))
            except ValueError:
                pass
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "power_w": float(np.median(pw)) if pw else None}


# ----------------------------------------------------------------------------------------- CPU (oracle)

def _oracle_worker(args):
    """One bounded CPU run: `steps` full IMEX steps on a patch of the workload (own process).
    kind "reference": the reference's own functions (baseline/_ref, oracle/refops.py) composed by
    the shared orchestrator; "port": the numpy restatement (oracle/)."""
    name, scale, L, steps, seed, kind = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from types import SimpleNamespace

    from oracle import stepper as OS
    from paper_2605_16082_b200.scenarios import make_case
    c = make_case(name, scale=scale, L=L)
    s0 = c.state
    if kind == "reference":
        from oracle import refops
        ref = refops.load()
        s, p = refops.initial(ref, (c.mesh.vx, c.mesh.vy, c.mesh.vb, c.mesh.tri), c.L, s0, c.params)
        step = lambda s_: OS.imex_step_ops(ref.ops, s_, p, c.dt, c.m, c.kv, c.nu_v)  # noqa: E731
    else:
        from oracle import ext2d as OE
        from oracle import geom as OG
        om = OG.make_mesh(c.mesh.vx, c.mesh.vy, c.mesh.vb, c.mesh.tri)
        s = SimpleNamespace(grid=OG.extrude(om, c.L, s0["eta"]), ux=s0["ux"], uy=s0["uy"], T=s0["T"],
                            s2d=OE.S2(s0["eta"].copy(), s0["qx"], s0["qy"], 0.0))
        step = lambda s_: OS.imex_step(s_, c.params, c.dt, c.m, c.kv, c.nu_v)  # noqa: E731
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        s = step(s)
        times.append(time.perf_counter() - t0)
    return times, c.prisms


def cpu_kind():
    """"reference" when the unmodified reference is installed (baseline/_ref), else the "port"."""
    from oracle import refops
    return "reference" if refops.find() else "port"


def host_info():
    """CPU model, core count and numpy build of the host the CPU legs ran on."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = None
    try:
        cfg = np.show_config(mode="dicts")
        b = cfg.get("Build Dependencies", {}).get("blas", {})
        blas = f"{b.get('name')} {b.get('version')}".strip()
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "numpy": np.__version__, "numpy_blas": blas}


def cpu_oracle_throughput(name, steps, procs, scale, skip=0, kind="port"):
    """prism-DOF/s of the CPU path: `procs` independent patches in parallel processes (all host cores).

    Returns (value, seconds per step (max over processes, mean over the timed steps), prisms per process).
    """
    import multiprocessing as mp
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):   # one BLAS thread per process
        os.environ[v] = "1"
    os.environ["PDG_MESH_HOST"] = "1"          # the CPU arm never touches the GPU
    L = 50 if name == "c4" else None
    jobs = [(name, scale, L, steps, i, kind) for i in range(procs)]
    if procs == 1:
        res = [_oracle_worker(jobs[0])]
    else:
        with mp.get_context("spawn").Pool(procs) as pool:
            res = pool.map(_oracle_worker, jobs)
    per_step = np.max(np.array([r[0] for r in res]), axis=0)[skip:]
    tstep = float(np.mean(per_step))
    prisms = res[0][1]
    return 6.0 * prisms * procs / tstep, tstep, prisms


def run_reference(args, rank, world):
    """The reference arm: the reference's CPU implementation of the step on all host cores."""
    if rank != 0:
        return
    procs = max(1, min(os.cpu_count() or 1, 64))
    scale = 0.02 if args.config == "c4" else 0.2   # c4 patch: 20 x 10 squares = 400 tri x 50 layers
    kind = cpu_kind()
    value, tstep, prisms = cpu_oracle_throughput(args.config, args.warmup + args.steps, procs, scale,
                                                 skip=args.warmup, kind=kind)
    what = ("the reference's own functions (baseline/_ref prismdg, unmodified) composed by the shared "
            "orchestrator oracle/stepper.py" if kind == "reference" else "numpy restatement oracle/")
    sample = (f"{procs} independent processes, each one full IMEX step (L=50, m=20) of a {prisms}-prism patch of the "
              f"{args.config} workload per bench step ({what}); the full C4 step (50 M prisms) does not fit a "
              f"single CPU process (SURVEY.md section 0.5), so the value is per-prism throughput on patches")
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": tstep * 1e3, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": {"workload": f"{args.config} (bounded CPU sample: {prisms} prisms per process)"},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": kind, "sample": sample,
                            "host": host_info()},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ----------------------------------------------------------------------------------------- GPU

def fp64_floor(prof, counts, t_ms, mhz):
    """The step's FP64 issue floor: executed DFMA + DMUL + DADD warp instructions per launch from the
    newest profiles/r*_fp64.json (ncu --set full, scripts/fp64_floor.py) at the SM clock measured
    during the timed region; B200 issues 2 FP64 warp instructions per SM per cycle (64 lanes)."""
    import glob
    try:
        path = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_fp64.json")))[-1]
        with open(path) as f:
            inst = json.load(f)
    except (IndexError, OSError, ValueError):
        return None
    if not mhz:
        return None
    rate = 148 * 2 * mhz * 1e3          # FP64 warp instructions per ms
    tot, per = 0.0, {}
    for k, ms in prof.items():
        if k in inst:
            n = inst[k]["fp64_warp_inst"]
        elif k.startswith("subcycle") and all(f"rk_stage{i}" in inst for i in range(3)):
            n = int(k[len("subcycle"):]) * sum(inst[f"rk_stage{i}"]["fp64_warp_inst"] for i in range(3))
        else:
            continue
        tot += n * counts[k]
        per[k] = round(n / rate / ms, 3)
    return {"floor_ms_per_step": tot / rate, "frac_of_step": tot / rate / t_ms, "sm_mhz": mhz,
            "per_kernel_frac": per, "source": os.path.relpath(path, ROOT)}


def pcie_bandwidth(torch, nbytes=1 << 30, reps=3):
    """Measured pinned-host <-> device copy bandwidth (GB/s): H2D alone, D2H alone, both at once."""
    h = torch.empty(nbytes // 8, dtype=torch.float64, pin_memory=True)
    h2 = torch.empty_like(h, pin_memory=True)
    d = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
    d2 = torch.empty_like(d)
    up, down = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        best = None
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        return best
    t_up = timed(lambda: d.copy_(h, non_blocking=True))
    t_dn = timed(lambda: h2.copy_(d2, non_blocking=True))

    def both():
        with torch.cuda.stream(up):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(down):
            h2.copy_(d2, non_blocking=True)
    t_bi = timed(both)
    return {"h2d_GBps": nbytes / t_up / 1e9, "d2h_GBps": nbytes / t_dn / 1e9, "bidir_GBps": 2 * nbytes / t_bi / 1e9,
            "probe_bytes": nbytes}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--backend", default="nccl", help="process group for N>1 (gloo: host-staged halos, testing)")
    ap.add_argument("--halo", default="capi", choices=["capi", "p2p", "torch"],
                    help="N>1 halo transport: the library's NCCL plans (graph-captured step), NVLink peer "
                         "stores (csrc/p2p.cu, CUDA IPC inboxes; graph-captured) or torch.distributed")
    ap.add_argument("--phase-csv", default=None, help="append step,rank,phase,micros rows of one eager step")
    ap.add_argument("--dump", default=None, help="write the final local state to this .npz (testing)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    if args.backend == "gloo":
        local = 0 if torch.cuda.device_count() == 1 else local     # ranks may share one GPU for testing
    torch.cuda.set_device(local)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")

    from paper_2605_16082_b200 import stepper as S
    from paper_2605_16082_b200.partition import PAPER_EXCHANGES_PER_STEP, PartitionedRun, exchanges_per_step
    from paper_2605_16082_b200.scenarios import device_state_c4, make_case

    t_setup = time.perf_counter()
    case = make_case(args.config, with_state=(args.config != "c4"))
    if world == 1:
        st = S.ImexStepper(case.mesh, case.L, case.params, case.dt, case.m, case.kv, case.nu_v)
        stepper = st
    else:
        # strong scaling: the one C4 mesh split into `world` Hilbert ranges, halos over NCCL
        run = PartitionedRun(case.mesh, case.L, case.params, case.dt, case.m, case.kv, case.nu_v, world,
                             transport=("p2p" if args.halo == "p2p" else
                                        "nccl" if args.backend == "nccl" and args.halo == "capi" else "dist"),
                             rank=rank, device=local)
        st = run.st[rank]
        stepper = run
    if args.config == "c4":
        device_state_c4(case, st)
    elif world == 1:
        st.set_state(**case.state)
    else:
        run.set_state(**case.state)
    setup_s = time.perf_counter() - t_setup
    P = case.prisms
    dof_per_step = 6.0 * P          # whole job (all ranks together)

    # warm-up (graph capture happens on the first step)
    stepper.step(args.warmup)
    torch.cuda.synchronize()
    st.check()

    # ---- timed region: K graph replays
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        e0.record()
        stepper.step(args.steps)
        e1.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        tt = torch.tensor([t_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    st.check()
    value = dof_per_step / (t_ms * 1e-3)

    # ---- per-kernel breakdown (same K steps, unfused launches with CUDA events on the launching stream)
    launches = st.launches_per_step()
    st.use_graph = False
    st.prof = {}
    stepper.step(args.steps)
    torch.cuda.synchronize()
    prof = {k: float(np.mean([a.elapsed_time(b) for a, b in v])) for k, v in st.prof.items()}
    counts = {k: len(v) / args.steps for k, v in st.prof.items()}
    st.prof = None
    if args.phase_csv:   # SPEC.md:616 phase timings (step,rank,phase,micros) of one eager step per rank
        st.phase_trace = []
        stepper.step(1)
        st.phase_csv(args.phase_csv + (f".{rank}" if world > 1 else ""), step=0)
        st.phase_trace = None
    st.use_graph = True
    step_sum = sum(prof[k] * counts[k] for k in prof)
    hbm, peak_kind = peaks()
    per = {}
    P_local = st.nt * case.L if world == 1 else st.part.n_own * case.L
    for k, ms in prof.items():
        if k in KERNEL_BYTES:
            b = KERNEL_BYTES[k] * P_local
            if k.startswith("rhs_uT") and os.environ.get("PDG_NO_FUSEWT", "0") == "1":
                b -= 48 * P_local
        elif k.startswith("subcycle"):
            msub = int(k[len("subcycle"):])
            b = RK_SUBSTEP_BYTES_PER_TRI * (P_local // case.L) * msub
        elif k.startswith("rk"):
            b = RK_SUBSTEP_BYTES_PER_TRI * (P_local // case.L) / 3.0
        else:
            b = 0
        per[k] = {"ms": ms, "share": ms * counts[k] / step_sum, "GBps": (b / (ms * 1e-3) / 1e9) if b else None,
                  "bytes": b}
    dom = max((k for k in per if per[k]["bytes"]), key=lambda k: per[k]["ms"] * counts[k])
    ach = per[dom]["GBps"]
    traffic, traffic_src, tr_all = None, None, {}
    try:   # DRAM read+write bytes per launch from the newest committed ncu --set full capture
        import glob
        tj = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")))[-1]
        with open(tj) as f:
            tr_all = json.load(f) if args.config == "c4" and world == 1 else {}
        if dom in tr_all:
            traffic, traffic_src = tr_all[dom]["dram_bytes"], tr_all[dom]["source"]
    except Exception:
        pass
    roofline = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "peak_kind": peak_kind, "traffic": traffic, "traffic_source": traffic_src,
                "bytes_per_launch": per[dom]["bytes"], "launch_ms": per[dom]["ms"],
                "per_kernel": {k: {"alg_bytes": v["bytes"], "ms": round(v["ms"], 4),
                                   "frac": (round(v["GBps"] / hbm, 4) if v["GBps"] else None),
                                   "dram_bytes": (tr_all[k]["dram_bytes"] if k in tr_all else None)}
                               for k, v in per.items() if v["bytes"]},
                "step_model_M2": {"bytes_per_prism": M2_BYTES_PER_PRISM(case.L, case.m),
                                  "frac": M2_BYTES_PER_PRISM(case.L, case.m) * P / world / (t_ms * 1e-3) / 1e9 / hbm}}

    # ---- e2e: public API, host pinned buffers, full state round trip every step
    e2e = None
    if not args.no_e2e:
        from paper_2605_16082_b200.hostmem import near_gpu
        with near_gpu() as local_cpus:    # pinned buffers on the GPU's NUMA node (hostmem.py)
            host = st.get_state(numpy=False)
            pin = {k: (torch.empty(v.shape, dtype=v.dtype, pin_memory=True).copy_(v) if isinstance(v, torch.Tensor)
                       else v) for k, v in host.items()}
            h2d = sum(v.numel() * 8 for v in pin.values() if isinstance(v, torch.Tensor))
            ke = max(1, args.steps)     # steady state: a download overlaps the next upload (PCIe both ways)
            torch.cuda.synchronize()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record()
            for _ in range(ke):
                # public API with host (pinned) buffers: upload, step, download into the same buffers
                st.set_state(pin["eta"], pin["qx"], pin["qy"], pin["ux"], pin["uy"], pin["T"], pin["t"])
                stepper.step(1)
                st.get_state(numpy=False, out=pin)
            st.wait_io()                      # the last step's download is inside the timed region
            f1.record()
            torch.cuda.synchronize()
        te = f0.elapsed_time(f1) / ke
        if world > 1:
            tt = torch.tensor([te], device="cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        pcie = pcie_bandwidth(torch)
        # floor of the host round trip: a step needs its whole state uploaded before it starts and the
        # previous state's download overlaps the next upload on the other PCIe direction -- so both
        # directions are busy at once and share the measured bidirectional bandwidth
        floor_ms = max(h2d / pcie["h2d_GBps"], h2d / pcie["d2h_GBps"], 2 * h2d / pcie["bidir_GBps"]) / 1e6 + t_ms
        pcie.update(floor_ms=floor_ms, frac_of_floor=floor_ms / te,
                    achieved_io_GBps=h2d / max(te - t_ms, 1e-9) / 1e6)
        e2e = {"value": dof_per_step / (te * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d * world,
               "d2h_bytes_per_step": h2d * world, "ms_per_step": te, "steps": ke,
               "path": "ImexStepper.set_state/step/get_state with pinned host buffers (full state round trip)",
               "host_cpus": (f"{len(local_cpus)} GPU-local cpus ({local_cpus[0]}-{local_cpus[-1]})" if local_cpus
                             else "unbound"), "pcie": pcie}

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        procs = 1
        kind = cpu_kind()
        v, tstep, prisms = cpu_oracle_throughput(args.config, 2, procs, 0.02 if args.config == "c4" else 0.2,
                                                 kind=kind)
        what = "reference functions (baseline/_ref) + oracle/stepper.py" if kind == "reference" else \
            "numpy oracle (oracle/stepper.py)"
        cpu = {"value": v, "unit": UNIT, "cores": procs, "kind": kind, "host": host_info(),
               "sample": f"2 full IMEX steps (L={case.L}, m={case.m}) of a {prisms}-prism patch of {args.config}, "
                         f"{what}, single process; {tstep:.2f} s/step. C4 at full size extrapolated per prism: "
                         f"{tstep * case.prisms / prisms / 3600:.1f} h/step (not run: ~280 GB)"}

    if args.dump:
        s_ = st.get_state()
        n_own = st.part.n_own if world > 1 else st.nt
        gid = (st.mesh.global_ids if world > 1 else np.arange(st.nt))[:n_own]
        np.savez(f"{args.dump}.{rank}.npz", gid=gid, eta=s_["eta"][:n_own], T=s_["T"][:n_own * case.L],
                 ux=s_["ux"][:n_own * case.L])
    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": t_ms, "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic (seeded coastal basin; inputs larger than L2, no flush needed)",
               "config": {"workload": f"{args.config}: {case.mesh.nt} tri x {case.L} layers = {P} prisms, "
                                      f"m={case.m}, dt2d={case.dt2d} s, momentum+tracer, FP64",
                          "nt": case.mesh.nt, "L": case.L, "m": case.m, "prism_dof_per_step": dof_per_step,
                          "parallelism": (f"column partition x{world} (Hilbert ranges, 3 ghost rings, "
                                          + ("NVLink peer-store halos (CUDA IPC inboxes), one CUDA graph per rank "
                                             "and step" if args.halo == "p2p" else
                                             "library NCCL halo plans, one CUDA graph per rank and step"
                                             if args.backend == "nccl" and args.halo == "capi" else
                                             f"{'NCCL' if args.backend == 'nccl' else 'gloo host-staged'} "
                                             "torch.distributed send/recv, eager")
                                          + ", 2D halos overlapped with interior columns)")
                          if world > 1 else "single GPU",
                          "l2": "inputs larger than L2 (~48 GB resident fields)",
                          "halo_exchanges_per_step": (exchanges_per_step(case.m) if world > 1 else 0),
                          "paper_exchanges_per_step": PAPER_EXCHANGES_PER_STEP},
               "e2e": e2e, "gpu_launches": launches * args.steps, "launches_per_step": launches,
               "roofline": roofline, "fp64": fp64_floor(prof, counts, t_ms, clk.summary().get("sm_mhz")),
               "cpu_baseline": cpu, "clocks": clk.summary(),
               "kernels": {k: {"ms": round(v["ms"], 4), "share": round(v["share"], 4),
                               "GBps": None if v["GBps"] is None else round(v["GBps"], 1)} for k, v in per.items()},
               "setup_s": setup_s}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Fused 2-stage IMEX internal step (the hot path), every field resident in HBM.

The reference ships no stepper.  The composition is the
one defined in DESIGN.md section 3 and restated by the oracle
(oracle/stepper.py): stage 1 over dt/2 with m/2 external substeps and an
implicit vertical solve, stage 2 over dt with m substeps, explicit, from the
stage-1 midpoint.  Per stage the device work is

  1  compute_r with the EOS inline, + its layer sum   (k_compute_r_t<FROM_T>, tile-staged)
  2  q = project(u) + column sum of q + total depth   (k_project)
  3  F3D->2D = column sum of (F_h(u, q, fac(q)) + stresses)     (k_hrhs_t<2, PRED, RS>)
  4  m_s SSP-RK3 substeps, one fused kernel per RK stage, + Qbar, F2D
  5  mismatch (Qbar - sum q) / H                      (k_mismatch)
  6  rhs_u = M0 u0 + dt (F_h(u, qbar) + stress + M1 F2D/H1), rhs_T = M0 T0 + dt F_T(T, qbar),
     and w~ (qbar = q + Jz mis and its factor on the fly; bottom-up layer loop carrying the
     w~ sweep)                                        (k_hrhs_s<3, STAGE, .., WT>)
  7  vertical: (M1 - dt A) x = rhs (block Thomas: k_vimpl_fwd + k_vimpl_bwd_r) or
     x = M1^-1 (rhs + dt A x) (k_vexpl3), A assembled per layer in registers

The flux factors, qbar, prism masses, mesh velocity and the banded matrices
are never materialised.  The whole step is one CUDA graph.
"""
from __future__ import annotations

from types import SimpleNamespace

import ctypes
import os

import numpy as np
import torch

from . import _lib
from .device import DeviceMesh, c3_out, p6_out, ptr, stream_ptr
from .params import PenaltyParams, PhysParams

F64 = torch.float64


class ImexStepper:
    """Device-resident internal+external stepper for one mesh / layer count."""

    def __init__(self, mesh, L: int, params: PhysParams, dt: float, m: int, kv: float, nu_v: float,
                 pen: PenaltyParams = PenaltyParams(), device=None, part=None):
        if m % 2:
            raise ValueError("m must be even (stage 1 uses m/2 substeps)")
        self.mesh, self.L, self.p = mesh, L, params
        self.dt, self.m, self.kv, self.nu_v, self.pen = float(dt), int(m), float(kv), float(nu_v), pen
        self.part = part          # partition.Part when this stepper owns only part of the columns
        # a context of its own: the captured graphs hold its layer count, sigma fractions and
        # block-Thomas workspace, which a shared (per-mesh) context could resize under them
        self.dm = DeviceMesh(mesh, device).set_layers(L)
        if part is not None:
            _lib.check(_lib.lib().pdg_ctx_set_owned(self.dm.h, part.n_own), "set_owned")
        self.halo = None          # DistHalo for multi-process runs (VirtualGroup drives several steppers)
        self.dev = self.dm.device
        nt = self.nt = mesh.nt
        z = lambda *s: torch.zeros(s, dtype=F64, device=self.dev)  # noqa: E731
        self.S = z(3, 3, nt)                     # 2D state (eta, qx, qy); eta is also the grid free surface
        self.Sw = [z(3, 3, nt), z(3, 3, nt)]     # per-stage external working states
        self.U = [z(2, 6, L, nt) for _ in range(3)]   # rotating: state / stage-1 result / stage-2 result
        self.T = [z(6, L, nt) for _ in range(3)]
        self.r = z(2, 6, L, nt)
        self.q = z(2, 6, L, nt)
        self.wt = z(6, L, nt)
        self.qsum, self.htot, self.f3d2d = z(2, 3, nt), z(3, nt), z(2, 3, nt)
        self.qbar, self.f2d, self.mis = z(2, 3, nt), z(2, 3, nt), z(2, 3, nt)
        self.rsum = z(2, 3, nt)                  # layer sum of the baroclinic head for F3D->2D
        self._rs_ok = ctypes.c_int(0)
        self.use_rsum = os.environ.get("PDG_NO_RSUM", "0") != "1"   # (A/B: F3D->2D reading r instead)
        self.W12 = (z(3, 3, nt), z(3, 3, nt)) if part is not None else None   # RK stage states (partitioned)
        # partitions (>= 3 ghost rings): the RK stages of a substep run on owned + rings 1-2, owned +
        # ring 1 and owned columns, so the 2D state is exchanged once per substep; the last stage
        # updates the columns other ranks receive first and the rest while the exchange is in flight
        self.cols2d = None
        if part is not None:
            if part.ring is None or part.ring.size and part.ring.max() < 3:
                raise ValueError("partitioned stepping needs 3 ghost rings (partition.decompose depth=3)")
            n_own = part.n_own
            ring = np.concatenate([np.zeros(n_own, np.int32), part.ring])
            sent = np.zeros(n_own, bool)
            for idx in part.send.values():
                sent[idx] = True
            sets = (np.flatnonzero(ring <= 2), np.flatnonzero(ring <= 1), np.flatnonzero(sent),
                    np.flatnonzero(~sent))
            self.cols2d = tuple(torch.as_tensor(x.astype(np.int32), device=self.dev) for x in sets)
        self.cur = 0
        self.t = 0.0
        self.graphs = {}
        self.use_graph = True
        self.prof = None       # {name: [(start_event, end_event), ...]} when profiling
        self.fuse_rhs = True   # momentum + tracer stage right-hand sides in one kernel
        self._pending_d2h = {}   # host buffer address -> event of the download filling it
        self.schedule_check = False  # debug: poison in-flight ghost slots (partitioned runs)
        self._skip_exchanges = set()  # tests only: exchange names to leave out (a broken schedule)
        self.phase_trace = None      # list -> per-phase CUDA events of eager steps (phase_csv)
        self.nvtx = os.environ.get("PDG_NVTX", "0") == "1"   # NVTX range per library launch
        self.concurrent_vertical = os.environ.get("PDG_CONC_VERT", "0") == "1"
        self.concurrent_rp = os.environ.get("PDG_CONC_RP", "0") == "1"   # r || projection (A/B)
        self.fuse_wt = os.environ.get("PDG_NO_FUSEWT", "0") != "1"   # w~ inside the stage RHS

    def _c(self, name, rc):
        _lib.check(rc, name)

    def _timed(self, name, fn, *args):
        """Launch one library entry; record CUDA events around it on the current stream when profiling,
        and an NVTX range around the launch when `nvtx` is set (nsys / ncu --nvtx phase markers)."""
        if self.nvtx:
            torch.cuda.nvtx.range_push(name)
            try:
                self._timed_inner(name, fn, *args)
            finally:
                torch.cuda.nvtx.range_pop()
            return
        self._timed_inner(name, fn, *args)

    def _timed_inner(self, name, fn, *args):
        if self.prof is None:
            _lib.check(fn(*args), name)
            return
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(fn(*args), name)
        e1.record()
        self.prof.setdefault(name, []).append((e0, e1))

    # ------------------------------------------------------------------ state I/O (reference layouts)
    IO_CHUNK_BYTES = 256 << 20   # DMA granularity of the host I/O pipeline (scripts/e2e_sweep.py: 241 vs 243 ms at 128 MB)
    IO_SLOTS = 4                 # device staging buffers per direction

    def _io_plan(self):
        """(name, device planes, L_f, nk, [(c0, c1), ...]) of the prognostic state: the column chunks
        of every field (the same plan for uploads and downloads, so chunk events pair up)."""
        if getattr(self, "_plan", None) is None:
            nt, L = self.nt, self.L
            plan = []
            for name, lf, nk in (("eta", 1, 3), ("qx", 1, 3), ("qy", 1, 3), ("ux", L, 6), ("uy", L, 6), ("T", L, 6)):
                n = max(1, min(nt, self.IO_CHUNK_BYTES // (lf * nk * 8)))
                plan.append((name, lf, nk, [(c, min(nt, c + n)) for c in range(0, nt, n)]))
            self._plan = plan
            self._read_ev = {}       # (field, chunk) -> event: the device planes of that chunk were read out
        return self._plan

    def _planes(self, name):
        u = self.U[self.cur]
        return {"eta": self.S[0], "qx": self.S[1], "qy": self.S[2], "ux": u[0], "uy": u[1], "T": self.T[self.cur]}[name]

    def _io(self):
        """upload / download streams (the two PCIe directions), the two layout-conversion streams and
        the device staging slots of each direction."""
        if getattr(self, "_iost", None) is None:
            S = lambda: torch.cuda.Stream(device=self.dev)  # noqa: E731
            w = self.IO_CHUNK_BYTES // 8
            self._iost = SimpleNamespace(
                up=S(), down=S(), ut=S(), dt=S(),
                ubuf=[torch.empty(w, dtype=F64, device=self.dev) for _ in range(self.IO_SLOTS)],
                dbuf=[torch.empty(w, dtype=F64, device=self.dev) for _ in range(self.IO_SLOTS)],
                ufree=[None] * self.IO_SLOTS, dfree=[None] * self.IO_SLOTS, ui=0, di=0)
        return self._iost

    @staticmethod
    def _event(stream):
        e = torch.cuda.Event()
        e.record(stream)
        return e

    def set_state(self, eta, qx, qy, ux, uy, T, t: float = 0.0):
        """Load a state in the reference layouts ((nt, 3) 2D fields, (P, 6) prism fields).

        Host tensors (ideally pinned) stream in column chunks: each chunk is copied by DMA into a
        device staging slot on the upload stream and rearranged into the device planes by the
        library kernel (pdg_rows_to_planes) on a conversion stream.  A chunk that a previous
        get_state(out=...) is still downloading into the same host memory is uploaded as soon as
        THAT chunk has arrived, so a download and the next upload overlap on the two PCIe
        directions.  numpy / CUDA inputs are converted directly."""
        lb = _lib.lib()
        src = dict(eta=eta, qx=qx, qy=qy, ux=ux, uy=uy, T=T)
        main = torch.cuda.current_stream(self.dev)
        host = all(isinstance(a, torch.Tensor) and not a.is_cuda for a in src.values())
        io = self._io()
        io.ut.wait_stream(main)                  # the planes may still be read by queued work
        for name, lf, nk, chunks in self._io_plan():
            a = src[name]
            if not host:
                a = (a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a, np.float64)))
                a = a.to(self.dev, F64).contiguous()
            else:
                a = a.to(F64).contiguous()
            flat = a.reshape(-1)
            dest = self._planes(name)
            for ci, (c0, c1) in enumerate(chunks):
                n = (c1 - c0) * lf * nk
                part = flat[c0 * lf * nk:c0 * lf * nk + n]
                rev = self._read_ev.pop((name, ci), None)
                if host:
                    k = io.ui
                    io.ui = (io.ui + 1) % self.IO_SLOTS
                    if io.ufree[k] is not None:
                        io.up.wait_event(io.ufree[k])
                    ev = self._pending_d2h.pop(part.data_ptr(), None)
                    if ev is not None:
                        io.up.wait_event(ev)
                    buf = io.ubuf[k][:n]
                    with torch.cuda.stream(io.up):
                        buf.copy_(part, non_blocking=True)
                    io.ut.wait_event(self._event(io.up))
                else:
                    buf = part
                    io.ut.wait_stream(main)
                if rev is not None:
                    io.ut.wait_event(rev)
                _lib.check(lb.pdg_rows_to_planes(ptr(buf), c1 - c0, lf, nk, ptr(dest), self.nt, c0,
                                                 ctypes.c_void_p(io.ut.cuda_stream)), "rows_to_planes")
                if host:
                    io.ufree[k] = self._event(io.ut)
                else:
                    buf.record_stream(io.ut)
        main.wait_stream(io.ut)
        self.t = float(t)

    def get_state(self, numpy=True, out=None):
        """The state in the reference layouts.  out: dict of host tensors (pinned) to fill: each column
        chunk is rearranged by the library kernel (pdg_planes_to_rows) into a device staging slot
        and copied to the host on the download stream (asynchronous: wait_io() / synchronise before
        reading the buffers; a later set_state from the same buffers orders itself after each
        chunk's download)."""
        nt, L = self.nt, self.L
        if out is not None:
            lb = _lib.lib()
            io = self._io()
            io.dt.wait_stream(torch.cuda.current_stream(self.dev))
            for name, lf, nk, chunks in self._io_plan():
                src = self._planes(name)
                flat = out[name].reshape(-1)
                for ci, (c0, c1) in enumerate(chunks):
                    n = (c1 - c0) * lf * nk
                    k = io.di
                    io.di = (io.di + 1) % self.IO_SLOTS
                    if io.dfree[k] is not None:
                        io.dt.wait_event(io.dfree[k])
                    buf = io.dbuf[k][:n]
                    _lib.check(lb.pdg_planes_to_rows(ptr(src), nt, c0, c1 - c0, lf, nk, ptr(buf),
                                                     ctypes.c_void_p(io.dt.cuda_stream)), "planes_to_rows")
                    rd = self._event(io.dt)
                    self._read_ev[(name, ci)] = rd
                    io.down.wait_event(rd)
                    hpart = flat[c0 * lf * nk:c0 * lf * nk + n]
                    with torch.cuda.stream(io.down):
                        hpart.copy_(buf, non_blocking=True)
                    ev = self._event(io.down)
                    io.dfree[k] = ev
                    self._pending_d2h[hpart.data_ptr()] = ev
            out["t"] = self.t
            return out
        u = self.U[self.cur]
        res = dict(eta=c3_out(self.S[0]), qx=c3_out(self.S[1]), qy=c3_out(self.S[2]), ux=p6_out(u[0], nt, L),
                   uy=p6_out(u[1], nt, L), T=p6_out(self.T[self.cur], nt, L), t=self.t)
        if numpy:
            res = {k: (v.cpu().numpy() if isinstance(v, torch.Tensor) else v) for k, v in res.items()}
        return res

    def wait_io(self):
        """Order the current stream after every pending get_state(out=...) download."""
        if getattr(self, "_iost", None) is not None:
            torch.cuda.current_stream(self.dev).wait_stream(self._iost.down)
        self._pending_d2h.clear()

    # ------------------------------------------------------------------ one stage
    def _stage(self, s, eta_u, u, T, u0, T0, Sw, out_u, out_T, dt_s, m_s, implicit, t_wind):
        """One IMEX stage as a generator: yields the fields whose ghost columns must be refreshed
        (partitioned runs only) and returns the end-of-stage free surface."""
        lb, h, p = _lib.lib(), self.dm.h, self.p
        tm = self._timed
        part = self.part is not None
        eta0 = self.S[0]
        tsx, tsy = p.wind(t_wind)
        tag = "impl" if implicit else "expl"
        if part:   # debug: ghosts of the fields this stage produces stay NaN until their exchange lands
            self._poison([self.q, self.mis, out_u, out_T], False)
            self._poison([self.f3d2d], True)
        r_args = (h, ptr(eta_u), ptr(T), p.alpha, p.t_ref, p.g, ptr(self.r),
                  ptr(self.rsum) if self.use_rsum else None, ctypes.byref(self._rs_ok))
        conc_rp = self.concurrent_rp and self.prof is None
        if conc_rp:   # r (FP64-bound) on a second stream, overlapping the HBM-bound projection
            main = torch.cuda.current_stream(self.dev)
            side = self._side_stream()
            side.wait_stream(main)
            with torch.cuda.stream(side):
                _lib.check(lb.pdg_step_r(*r_args, stream_ptr()), "r")
        else:
            tm("r", lb.pdg_step_r, *r_args, s)
        tm("project", lb.pdg_project_transport, h, ptr(eta_u), ptr(u[0]), ptr(u[1]), None, None, 0, ptr(self.q),
           ptr(self.qsum), ptr(self.htot), s)
        if conc_rp:
            main.wait_stream(side)
        # the 3D ring-1 exchanges block the stream: a boundary-first split (boundary columns, post,
        # interior) was measured slower -- the extra launch of the 50-layer column loops costs a
        # latency-bound partial wave (~0.3-0.6 ms per call at 8 ranks) against ~30 us of transfer
        if part:
            yield ("all", [self.q], "q")
        tm("f3d2d", lb.pdg_step_f3d2d_rsum, h, ptr(eta_u), ptr(u), ptr(self.q), ptr(self.r),
           ptr(self.rsum) if self._rs_ok.value else None, p.g, p.f, p.rho0, tsx, tsy,
           p.cd, ptr(self.f3d2d), s)
        if p.kappa_h:   # explicit horizontal viscosity in horizontal_rhs: its column sum (csrc/hdiff.cu)
            tm("hdiff_f3d2d", lb.pdg_horizontal_diffusion, h, ptr(eta_u), ptr(u), 2, p.kappa_h, 1, 1.0, 1, None, 0,
               ptr(self.f3d2d), s)
        if part:
            yield ("deep", [self.f3d2d], "f3d2d")   # the ring columns' RK stages need their forcing
        self._c("copy", lb.pdg_copy_d2d(ptr(Sw), ptr(self.S), self.S.numel() * 8, s))
        dt2 = dt_s / m_s
        if not part:
            tm(f"subcycle{m_s}", lb.pdg_ext2d_subcycle, h, ptr(Sw), m_s, dt2, p.g, p.rho0, ptr(self.f3d2d), None,
               None, None, ptr(self.qbar), ptr(self.f2d), 1, s)
        else:
            tm("sub_begin", lb.pdg_ext2d_subcycle_begin, h, ptr(Sw), p.g, dt2, 1, ptr(self.qbar), s)
            W1, W2 = self.W12
            c012, c01, bnd, intr = self.cols2d
            for _ in range(m_s):
                for k, (X, Y, cols) in enumerate(((Sw, W1, c012), (W1, W2, c01))):
                    tm(f"rk{k}", lb.pdg_ext2d_rk_stage_cols, h, k, ptr(X), ptr(Sw), ptr(Y), dt2, p.g, p.rho0,
                       ptr(self.f3d2d), ptr(self.qbar), ptr(cols), cols.numel(), s)
                tm("rk2", lb.pdg_ext2d_rk_stage_cols, h, 2, ptr(W2), ptr(Sw), ptr(Sw), dt2, p.g, p.rho0,
                   ptr(self.f3d2d), ptr(self.qbar), ptr(bnd), bnd.numel(), s)
                self._poison([Sw], True)      # in flight: the interior stage must not read ghosts
                yield ("start", [Sw], "state2d")
                tm("rk2", lb.pdg_ext2d_rk_stage_cols, h, 2, ptr(W2), ptr(Sw), ptr(Sw), dt2, p.g, p.rho0,
                   ptr(self.f3d2d), ptr(self.qbar), ptr(intr), intr.numel(), s)
                yield ("finish", [Sw], "state2d")
            tm("sub_end", lb.pdg_ext2d_subcycle_end, h, ptr(Sw), ptr(self.f3d2d), m_s, dt2, ptr(self.qbar),
               ptr(self.f2d), s)
        eta1 = Sw[0]
        tm("mismatch", lb.pdg_mismatch, h, ptr(self.qbar), ptr(self.qsum), ptr(self.htot), ptr(self.mis), s)
        if part:
            yield ("all", [self.mis], "mis")
        if self.fuse_rhs and self.fuse_wt:   # w~ formed in the stage-RHS layer loop (pdg_step_rhs_ut_w)
            tm("rhs_uT_s1" if u is u0 else "rhs_uT_s2", lb.pdg_step_rhs_ut_w, h, ptr(eta_u), ptr(eta0), ptr(eta1),
               ptr(u), ptr(T), ptr(u0), ptr(T0), ptr(self.q), ptr(self.mis), ptr(self.r), ptr(self.f2d), p.g, p.f,
               p.rho0, tsx, tsy, p.cd, dt_s, ptr(out_u), ptr(out_T), ptr(self.wt), s)
        elif self.fuse_rhs:
            tm("wtilde", lb.pdg_compute_wtilde, h, ptr(eta_u), ptr(self.q), None, ptr(self.mis), p.g, None, 0,
               ptr(self.wt), s)
            tm("rhs_uT_s1" if u is u0 else "rhs_uT_s2", lb.pdg_step_rhs_ut, h, ptr(eta_u), ptr(eta0), ptr(eta1), ptr(u), ptr(T), ptr(u0), ptr(T0),
               ptr(self.q), ptr(self.mis), ptr(self.r), ptr(self.f2d), p.g, p.f, p.rho0, tsx, tsy, p.cd, dt_s,
               ptr(out_u), ptr(out_T), s)
        else:
            tm("wtilde", lb.pdg_compute_wtilde, h, ptr(eta_u), ptr(self.q), None, ptr(self.mis), p.g, None, 0,
               ptr(self.wt), s)
            tm("rhs_u", lb.pdg_step_rhs, h, 2, ptr(eta_u), ptr(eta0), ptr(eta1), ptr(u), ptr(u0), ptr(self.q),
               ptr(self.mis), ptr(self.r), ptr(self.f2d), p.g, p.f, p.rho0, tsx, tsy, p.cd, dt_s, ptr(out_u), s)
            tm("rhs_T", lb.pdg_step_rhs, h, 1, ptr(eta_u), ptr(eta0), ptr(eta1), ptr(T), ptr(T0), ptr(self.q),
               ptr(self.mis), None, None, p.g, p.f, p.rho0, 0.0, 0.0, 0.0, dt_s, ptr(out_T), s)
        if p.kappa_h:   # + dt D_u(u) (horizontal_rhs, internal3d.py:743) and + dt D_T(T) (:788)
            tm("hdiff_u", lb.pdg_horizontal_diffusion, h, ptr(eta_u), ptr(u), 2, p.kappa_h, 1, dt_s, 0, None, 0,
               ptr(out_u), s)
        if p.nu_h:
            tm("hdiff_T", lb.pdg_horizontal_diffusion, h, ptr(eta_u), ptr(T), 1, p.nu_h, 0, dt_s, 0, None, 0,
               ptr(out_T), s)
        pe = self.pen
        conc = self.concurrent_vertical and self.prof is None
        if conc:   # the tracer solve on a second stream (own workspace): overlaps the momentum solve
            main = torch.cuda.current_stream(self.dev)
            side = self._side_stream()
            side.wait_stream(main)
        tm(f"vertical_u_{tag}", lb.pdg_step_vertical, h, 2, int(implicit), ptr(eta_u), ptr(eta0), ptr(eta1), dt_s,
           ptr(self.wt), p.kappa_h, self.kv, pe.n0, pe.order, dt_s, ptr(out_u), ptr(u), ptr(out_u), s)
        if conc:
            with torch.cuda.stream(side):
                _lib.check(lb.pdg_step_vertical(h, 1, int(implicit), ptr(eta_u), ptr(eta0), ptr(eta1), dt_s,
                                                ptr(self.wt), p.nu_h, self.nu_v, pe.n0, pe.order, dt_s, ptr(out_T),
                                                ptr(T), ptr(out_T), stream_ptr()), "vertical_T")
            main.wait_stream(side)
        else:
            tm(f"vertical_T_{tag}", lb.pdg_step_vertical, h, 1, int(implicit), ptr(eta_u), ptr(eta0), ptr(eta1), dt_s,
               ptr(self.wt), p.nu_h, self.nu_v, pe.n0, pe.order, dt_s, ptr(out_T), ptr(T), ptr(out_T), s)
        if part:
            yield ("all", [out_u, out_T], "uT")
        return eta1

    def _step_gen(self, t0):
        s = stream_ptr()
        a, b, c = self.cur, (self.cur + 1) % 3, (self.cur + 2) % 3
        U, T = self.U, self.T
        eta_h = yield from self._stage(s, self.S[0], U[a], T[a], U[a], T[a], self.Sw[0], U[b], T[b], 0.5 * self.dt,
                                       self.m // 2, True, t0)
        yield from self._stage(s, eta_h, U[b], T[b], U[a], T[a], self.Sw[1], U[c], T[c], self.dt, self.m, False,
                               t0 + 0.5 * self.dt)
        self._c("copy", _lib.lib().pdg_copy_d2d(ptr(self.S), ptr(self.Sw[1]), self.S.numel() * 8, s))

    def _launch_step(self, t0):
        tr = self.phase_trace
        ev = (lambda: torch.cuda.Event(enable_timing=True)) if tr is not None else None
        last = None
        if tr is not None:
            last = ev()
            last.record()
        for phase, fields, name in self._step_gen(t0):
            if tr is not None:     # compute since the previous exchange point, then the exchange call
                e = ev()
                e.record()
                seg = {"start": "boundary", "finish": "interior", "start1": "boundary",
                       "finish1": "interior"}.get(phase, "compute")
                tr.append((f"{seg}:{name}", last, e))
                last = e
            if name in self._skip_exchanges:          # tests: a deliberately broken schedule
                pass
            elif phase in ("all", "deep"):
                self.halo.exchange(fields, deep=phase == "deep")
            elif phase in ("start", "start1"):      # boundary-first: all rings (2D) / ring 1 (3D)
                self.halo.start(fields, phase == "start")
            else:
                self.halo.finish(fields, phase == "finish")
            if tr is not None:
                e = ev()
                e.record()
                tr.append(({"start": "pack+post", "finish": "join+unpack", "start1": "pack+post",
                            "finish1": "join+unpack"}.get(phase, "exchange") + f":{name}", last,
                           e))
                last = e
        if tr is not None:
            e = ev()
            e.record()
            tr.append(("compute:tail", last, e))

    def _side_stream(self):
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(device=self.dev, priority=-1)
        return self._side

    # ------------------------------------------------------------------ schedule checking (debug)
    def _poison(self, fields, deep):
        """schedule_check: fill the ghost slots a pending exchange will refresh with NaN, so a kernel
        that reads them before the exchange joins produces non-finite owned values."""
        if not (self.schedule_check and self.part is not None):
            return
        idx = self._ghost_slots(deep)
        if idx.numel() == 0:
            return
        lb = _lib.lib()
        for f in fields:
            npl = f.numel() // self.nt
            need = npl * idx.numel()
            if getattr(self, "_nan", None) is None or self._nan.numel() < need:
                self._nan = torch.full((need,), float("nan"), dtype=F64, device=self.dev)
            _lib.check(lb.pdg_halo_unpack(ptr(self._nan), npl, self.nt, ptr(idx), idx.numel(), ptr(f), stream_ptr()),
                       "poison")

    def _ghost_slots(self, deep):
        key = "_gs_deep" if deep else "_gs_ring1"
        if getattr(self, key, None) is None:
            rv = self.part.recv if deep else self.part.recv1
            arr = np.concatenate([np.asarray(v, np.int32) for _, v in sorted(rv.items())]) if rv else \
                np.zeros(0, np.int32)
            setattr(self, key, torch.as_tensor(arr, device=self.dev))
        return getattr(self, key)

    def check_schedule(self):
        """schedule_check: raise ScheduleViolation if a poisoned ghost reached an owned value."""
        from .errors import ScheduleViolation
        n = self.part.n_own if self.part is not None else self.nt
        bad = [k for k, f in (("eta/qx/qy", self.S[..., :n]), ("u", self.U[self.cur][..., :n]),
                              ("T", self.T[self.cur][..., :n])) if not bool(torch.isfinite(f).all())]
        if bad:
            r = self.part.rank if self.part is not None else 0
            raise ScheduleViolation(f"rank {r}: owned {', '.join(bad)} read a ghost slot before its exchange joined "
                                    f"(step ending t={self.t})")

    def phase_csv(self, path, step: int, rank: int | None = None):
        """Append this step's phases (phase_trace = [] before the step; eager stepping) as SPEC.md:616
        rows step,rank,phase,micros (CUDA events on the launching stream)."""
        import os
        torch.cuda.synchronize(self.dev)
        r = (self.part.rank if self.part is not None else 0) if rank is None else rank
        new = not os.path.exists(path)
        with open(path, "a") as f:
            if new:
                f.write("step,rank,phase,micros\n")
            for name, a, b in self.phase_trace or []:
                f.write(f"{step},{r},{name},{a.elapsed_time(b) * 1e3:.3f}\n")
        self.phase_trace = []

    def _advance(self):
        self.cur = (self.cur + 2) % 3
        self.t = self.t + self.dt

    def step(self, n: int = 1):
        """Advance n internal steps (stream ordered, no host sync)."""
        with torch.cuda.device(self.dev):
            if getattr(self, "_iost", None) is not None:   # a pending get_state(out=...) still reads S / U
                torch.cuda.current_stream(self.dev).wait_stream(self._iost.dt)
            for _ in range(n):
                wind_varies = self.p.tau_x1 is not None
                capturable = self.part is None or getattr(self.halo, "capturable", False)
                if self.use_graph and not wind_varies and capturable and not self.schedule_check:
                    g = self.graphs.get(self.cur)
                    if g is None:
                        g = self._capture()
                    g.replay()
                else:
                    self._launch_step(self.t)
                self._advance()
                if self.schedule_check:
                    self.check_schedule()

    def _capture(self):
        # warm the workspace (block-Thomas scratch is sized on first use), then capture
        side = torch.cuda.Stream(device=self.dev)
        side.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(side):
            saved = [x.clone() for x in (self.S,)]
            self._launch_step(self.t)                          # sizes workspaces (result discarded)
            self.S.copy_(saved[0])
        torch.cuda.current_stream().wait_stream(side)
        import gc
        gc.collect()                       # run pending finalisers before the capture, not inside it
        gcflag = gc.isenabled()
        gc.disable()
        try:
            with torch.cuda.graph(g):
                self._launch_step(self.t)
        finally:
            if gcflag:
                gc.enable()
        self.graphs[self.cur] = g
        return g

    def diagnostics(self, stage: int = 2) -> dict:
        """diagnostics_2d (external2d.py:366-380) + budget_3d (internal3d.py:942-951) of the resident
        state on its grid, reduced on the device in one fused pass (one 80-byte read-back).

        stage 2 (default): the current state; stage 1: the last step's stage-1 result (midpoint
        fields on the stage-1 free surface), kept in the rotating buffers until the next step."""
        lb = _lib.lib()
        if stage == 1:
            S, u, T, t = self.Sw[0], self.U[(self.cur + 2) % 3], self.T[(self.cur + 2) % 3], self.t - 0.5 * self.dt
        else:
            S, u, T, t = self.S, self.U[self.cur], self.T[self.cur], self.t
        with torch.cuda.device(self.dev):
            if getattr(self, "_diag_work", None) is None:
                self._diag_work = torch.empty(lb.pdg_diagnostics_work_doubles(self.dm.h), dtype=F64, device=self.dev)
                self._diag_out = torch.empty(10, dtype=F64, device=self.dev)
            self._c("diagnostics", lb.pdg_step_diagnostics(self.dm.h, ptr(S), ptr(u), ptr(T), self.p.g,
                                                           ptr(self._diag_work), ptr(self._diag_out), stream_ptr()))
            v = self._diag_out.cpu().tolist()
        return {"t": t, "total_volume": v[0], "total_energy": v[1], "eta_min": v[2], "eta_max": v[3],
                "volume": v[4], "momentum_x": v[5], "momentum_y": v[6], "tracer_mass": v[7], "tracer_min": v[8],
                "tracer_max": v[9]}

    DIAG_CSV = ("t", "total_volume", "total_energy", "eta_min", "eta_max")
    BUDGET_CSV = ("t", "stage", "volume", "momentum_x", "momentum_y", "tracer_mass", "tracer_min",
                  "tracer_max")

    def log_csv(self, diag_path=None, budget_path=None):
        """Append this step's rows to the diagnostics CSV (t,total_volume,total_energy,eta_min,eta_max)
        and the per-step budget CSV (one row per IMEX stage); headers are written on creation."""
        import os
        rows = []
        if diag_path is not None:
            d = self.diagnostics()
            rows.append((diag_path, self.DIAG_CSV, [d[k] for k in self.DIAG_CSV]))
        if budget_path is not None:
            for stage in (1, 2):
                d = self.diagnostics(stage)
                rows.append((budget_path, self.BUDGET_CSV, [d["t"], stage] + [d[k] for k in self.BUDGET_CSV[2:]]))
        for path, header, vals in rows:
            new = not os.path.exists(path)
            with open(path, "a") as f:
                if new:
                    f.write(",".join(header) + "\n")
                f.write(",".join(repr(float(v)) if isinstance(v, float) else str(v) for v in vals) + "\n")

    def check(self):
        """Synchronise and raise the first device-side error (DryColumn, ZeroPivot, CflViolation ...)."""
        self.dm.raise_errors("imex step")

    def launches_per_step(self) -> int:
        """Kernel launches issued by one step (counted by the library)."""
        with torch.cuda.device(self.dev):
            saved = (self.S.clone(), self.cur, self.t)
            n0 = self.dm.launches()
            self._launch_step(self.t)
            n1 = self.dm.launches()
            self.S.copy_(saved[0])
            torch.cuda.synchronize(self.dev)
        return n1 - n0


def imex_step(state, params: PhysParams, dt: float, m: int, kv: float, nu_v: float):
    """Drop-in one-step driver with the oracle-stepper interface (state.grid/ux/uy/T/s2d)."""
    from .mesh import update_moving_mesh
    from .params import State2D
    grid = state.grid
    st = ImexStepper(grid.mesh, grid.n_layers, params, dt, m, kv, nu_v)
    st.use_graph = False
    st.set_state(state.s2d.eta, state.s2d.qx, state.s2d.qy, state.ux, state.uy, state.T, state.s2d.t)
    st.step(1)
    st.check()
    o = st.get_state()
    return SimpleNamespace(grid=update_moving_mesh(grid, o["eta"], dt), ux=o["ux"], uy=o["uy"], T=o["T"],
                           s2d=State2D(o["eta"], o["qx"], o["qy"], o["t"]))

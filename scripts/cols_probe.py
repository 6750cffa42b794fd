"""Probe: the stepper's vertical stage and projection over all columns vs over an identity column
list (the partitioned path's launch form) on the C4 case."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2605_16082_b200 import _lib, stepper as S
from paper_2605_16082_b200.device import ptr, stream_ptr
from paper_2605_16082_b200.scenarios import device_state_c4, make_case
c = make_case("c4", with_state=False)
st = S.ImexStepper(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v)
device_state_c4(c, st)
st.use_graph = False
st.step(1)
torch.cuda.synchronize()
lb, h = _lib.lib(), st.dm.h
ident = torch.arange(c.mesh.nt, dtype=torch.int32, device="cuda")
u, T = st.U[0], st.T[0]
out_u = torch.empty_like(u)
eta = st.S[0]
pe = st.pen
def timeit(fn, n=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
for implicit in (1, 0):
    a = timeit(lambda: _lib.check(lb.pdg_step_vertical(h, 2, implicit, ptr(eta), ptr(eta), ptr(eta), 0.5 * c.dt, ptr(st.wt), 0.0, st.kv, pe.n0, pe.order, 0.5 * c.dt, ptr(u), ptr(u), ptr(out_u), stream_ptr()), "v"))
    b = timeit(lambda: _lib.check(lb.pdg_step_vertical_cols(h, 2, implicit, ptr(eta), ptr(eta), ptr(eta), 0.5 * c.dt, ptr(st.wt), 0.0, st.kv, pe.n0, pe.order, 0.5 * c.dt, ptr(u), ptr(u), ptr(out_u), ptr(ident), ident.numel(), stream_ptr()), "vc"))
    print("vertical implicit" if implicit else "vertical explicit", "all", round(a, 3), "list", round(b, 3), flush=True)
a = timeit(lambda: _lib.check(lb.pdg_project_transport(h, ptr(eta), ptr(u[0]), ptr(u[1]), None, None, 0, ptr(st.q), ptr(st.qsum), ptr(st.htot), stream_ptr()), "p"))
b = timeit(lambda: _lib.check(lb.pdg_project_transport(h, ptr(eta), ptr(u[0]), ptr(u[1]), None, ptr(ident), ident.numel(), ptr(st.q), ptr(st.qsum), ptr(st.htot), stream_ptr()), "p"))
print("project all", round(a, 3), "list", round(b, 3))

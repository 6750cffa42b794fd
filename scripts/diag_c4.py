"""Stability diagnostics of the C4 workload variants on the GPU (development aid)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2605_16082_b200 import stepper as S
from paper_2605_16082_b200.scenarios import device_state_c4, make_case


def run(tag, case, nsteps, host_state=False, graph=True):
    st = S.ImexStepper(case.mesh, case.L, case.params, case.dt, case.m, case.kv, case.nu_v)
    st.use_graph = graph
    if host_state:
        st.set_state(**case.state)
    else:
        device_state_c4(case, st)
    for i in range(nsteps):
        st.step(1)
        torch.cuda.synchronize()
        u = st.U[st.cur]
        e = st.S[0]
        H = e - st.dm.b3
        print(f"{tag} step {i}: max|eta| {e.abs().max().item():.4g} max|u| {u.abs().max().item():.4g} "
              f"min H {H.min().item():.4g} argmin {int(H.min(0).values.argmin().item())}", flush=True)
        try:
            st.check()
        except Exception as exc:
            print(f"{tag}: {exc!r}", flush=True)
            return
    print(f"{tag}: stable for {nsteps} steps", flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["full", "alpha0", "L10", "nograph"]
    c = make_case("c4", with_state=False)
    m = c.mesh
    col = 999120
    print("col", col, "x", m.x[col], "y", m.y[col], "b", m.b[col], flush=True)
    if "full" in which:
        run("full", c, 4)
    if "long" in which:
        run("long", c, 30)
    if "nograph" in which:
        run("nograph", c, 3, graph=False)
    if "alpha0" in which:
        c2 = make_case("c4", with_state=False)
        c2.params.alpha = 0.0
        run("alpha0", c2, 4)
    if "L10" in which:
        run("L10", make_case("c4", with_state=False, L=10), 4)
    if "win" in which:
        w = make_case("c4", scale=0.1)
        run("win0.1", w, 4, host_state=True)

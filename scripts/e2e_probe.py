"""Where the end-to-end (host state round trip) time goes at C4: raw PCIe copies vs the stepper's
set_state / get_state / step, each timed alone and in the bench's loop."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import pcie_bandwidth  # noqa: E402
from paper_2605_16082_b200 import stepper as S  # noqa: E402
from paper_2605_16082_b200.scenarios import device_state_c4, make_case  # noqa: E402


def timed(fn, reps=3):
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best * 1e3


if __name__ == "__main__":
    out = {"pcie": pcie_bandwidth(torch)}
    c = make_case("c4", with_state=False)
    st = S.ImexStepper(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v)
    device_state_c4(c, st)
    st.step(2)
    torch.cuda.synchronize()
    host = st.get_state(numpy=False)
    pin = {k: (torch.empty(v.shape, dtype=v.dtype, pin_memory=True).copy_(v) if isinstance(v, torch.Tensor) else v)
           for k, v in host.items()}
    nb = sum(v.numel() * 8 for v in pin.values() if isinstance(v, torch.Tensor))
    out["state_bytes"] = nb
    args = lambda: (pin["eta"], pin["qx"], pin["qy"], pin["ux"], pin["uy"], pin["T"], pin["t"])  # noqa: E731
    out["set_state_ms"] = timed(lambda: st.set_state(*args()))
    out["get_state_ms"] = timed(lambda: (st.get_state(numpy=False, out=pin), st.wait_io()))
    out["step_ms"] = timed(lambda: st.step(1))

    def loop():
        for _ in range(3):
            st.set_state(*args())
            st.step(1)
            st.get_state(numpy=False, out=pin)
        st.wait_io()
    out["loop_ms_per_step"] = timed(loop, 2) / 3
    print(json.dumps(out))

"""Steady-state A/B of kernel variants on the graph-replayed C4 step, with the SM clock and board
power sampled during each run (the FP64-dense step runs power-capped, so fewer operations can show
up as a higher clock rather than in an isolated kernel timing).

    python scripts/ab_steady.py "7=3" "7=4"        # pdg_tune key=value[,key=value] per variant
"""
import sys

import torch

sys.path.insert(0, ".")
from bench import Clocks  # noqa: E402
from paper_2605_16082_b200 import _lib  # noqa: E402
from paper_2605_16082_b200 import stepper as S  # noqa: E402
from paper_2605_16082_b200.scenarios import device_state_c4, make_case  # noqa: E402

if __name__ == "__main__":
    c = make_case("c4", with_state=False)
    st = S.ImexStepper(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v)
    device_state_c4(c, st)
    lib = _lib.lib()
    defaults = {k: lib.pdg_tune(k, -1) for k in range(16)}
    for rep in range(2):
        for spec in sys.argv[1:]:
            for k, v in defaults.items():
                lib.pdg_tune(k, v)
            for kv in filter(None, spec.split(",")):
                k, v = kv.split("=")
                lib.pdg_tune(int(k), int(v))
            st.graphs = {}
            st.step(3)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with Clocks(0) as clk:
                e0.record()
                st.step(20)
                e1.record()
                torch.cuda.synchronize()
            st.check()
            cs = clk.summary()
            print(f"{spec:12s} ms/step {e0.elapsed_time(e1) / 20:.3f}  sm {cs['sm_mhz']} MHz  power {cs['power_w']} W",
                  flush=True)

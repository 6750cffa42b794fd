"""One un-graphed C4 internal step (for ncu launch lists / --set full captures)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2605_16082_b200 import stepper as S
from paper_2605_16082_b200.scenarios import device_state_c4, make_case

if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    c = make_case(name, with_state=(name != "c4"))
    st = S.ImexStepper(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v)
    st.use_graph = False
    if name == "c4":
        device_state_c4(c, st)
    else:
        st.set_state(**c.state)
    st.step(n)
    torch.cuda.synchronize()
    st.check()
    print("ok", st.dm.launches())

"""A/B of stepper options on the C4 step (per-kernel CUDA-event times, un-graphed)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2605_16082_b200 import stepper as S
from paper_2605_16082_b200.scenarios import device_state_c4, make_case


def measure(st, n=2):
    st.use_graph = False
    st.prof = {}
    st.step(n)
    torch.cuda.synchronize()
    out = {k: round(float(np.mean([a.elapsed_time(b) for a, b in v])), 3) for k, v in st.prof.items()}
    st.prof = None
    return out


if __name__ == "__main__":
    c = make_case("c4", with_state=False)
    st = S.ImexStepper(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v)
    device_state_c4(c, st)
    st.use_graph = False
    st.step(1)
    for opt in sys.argv[1:]:
        k, v = opt.split("=")
        setattr(st, k, type(getattr(st, k))(int(v)) if isinstance(getattr(st, k), (bool, int)) else v)
        r = measure(st)
        print(opt, json.dumps(r), "sum", round(sum(r.values()), 2), flush=True)

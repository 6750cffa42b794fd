"""A/B of kernel variants (pdg_tune key=value sets) on the C4 step: per-launch CUDA-event times and
the max relative difference of the stepped state against the first variant.

    python scripts/ab_tune.py "7=1" "7=2" "7=2,1=2"
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2605_16082_b200 import _lib
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
    name = sys.argv[1] if sys.argv[1].startswith("c") else "c4"
    sets = [a for a in sys.argv[1:] if not a.startswith("c")]
    c = make_case(name, with_state=(name != "c4"))
    st = S.ImexStepper(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v)
    lib = _lib.lib()
    defaults = {k: lib.pdg_tune(k, -1) for k in range(16)}

    def reset():
        st.cur, st.t = 0, 0.0
        if name == "c4":
            device_state_c4(c, st)
        else:
            st.set_state(**c.state)

    ref = None
    for spec in sets:
        for k, v in defaults.items():
            lib.pdg_tune(k, v)
        for kv in filter(None, spec.split(",")):
            k, v = kv.split("=")
            lib.pdg_tune(int(k), int(v))
        reset()
        st.use_graph = False
        st.step(1)
        st.check()
        fields = [st.U[st.cur].clone(), st.T[st.cur].clone(), st.S.clone()]
        if ref is None:
            ref = fields
            diff = 0.0
        else:
            diff = max(float(((a - b).abs().max() / b.abs().max().clamp_min(1e-300)).item()) for a, b in zip(fields, ref))
        r = measure(st)
        print(spec, "reldiff %.3e" % diff, json.dumps(r), "sum", round(sum(r.values()), 2), flush=True)

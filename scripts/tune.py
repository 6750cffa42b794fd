"""Occupancy variants (pdg_tune) of the heavy kernel families on the C4 step: per-kernel CUDA-event times."""
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
    out = {k: float(np.mean([a.elapsed_time(b) for a, b in v])) for k, v in st.prof.items()}
    st.prof = None
    return out


if __name__ == "__main__":
    c = make_case("c4", with_state=False)
    st = S.ImexStepper(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v)
    device_state_c4(c, st)
    lib = _lib.lib()
    st.use_graph = False
    st.step(1)
    res = {}
    variants = [int(v) for v in sys.argv[1:]] or [1, 3, 4]
    keys = [int(k) for k in __import__("os").environ.get("TUNE_KEYS", "0,5").split(",")] if sys.argv[1:] else range(6)
    for v in variants:
        for key in keys:
            lib.pdg_tune(key, v)
        res[v] = measure(st)
        print(v, json.dumps({k: round(x, 3) for k, x in res[v].items()}), flush=True)

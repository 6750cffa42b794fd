"""Same-box A/B of library builds on the C4 step: per-kernel CUDA-event times (un-graphed) and the
graph-replayed step, each build in its own process (PDG_LIB), alternated A B A B.

    python scripts/ab_lib.py build/lib_a.so paper_2605_16082_b200/libprismdg_b200.so
    python scripts/ab_lib.py lib.so "lib.so:PDG_TUNE=6=7"        # same build, pdg_tune key=value[,..]
"""
import json
import os
import subprocess
import sys

CHILD = r'''
import json, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2605_16082_b200 import stepper as S
from paper_2605_16082_b200.scenarios import device_state_c4, make_case
from bench import Clocks
import os
from paper_2605_16082_b200 import _lib
for kv in filter(None, os.environ.get("PDG_TUNE", "").split(",")):
    k, v = kv.split("=")
    _lib.lib().pdg_tune(int(k), int(v))
c = make_case("c4", with_state=False)
st = S.ImexStepper(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v)
device_state_c4(c, st)
st.use_graph = False
st.step(1)
st.prof = {}
st.step(2)
torch.cuda.synchronize()
out = {k: round(float(np.mean([a.elapsed_time(b) for a, b in v])), 3) for k, v in st.prof.items()}
st.prof = None
st.use_graph = True
st.step(3)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with Clocks(0) as clk:
    e0.record(); st.step(10); e1.record(); torch.cuda.synchronize()
st.check()
out["step_ms"] = round(e0.elapsed_time(e1) / 10, 3)
out["sm_mhz"] = clk.summary().get("sm_mhz")
print("ABJSON" + json.dumps(out))
'''

if __name__ == "__main__":
    libs = sys.argv[1:]
    res = {lib: [] for lib in libs}
    for rep in range(2):
        for lib in libs:
            path, *kv = lib.split(":")
            env = dict(os.environ, PDG_LIB=os.path.abspath(path), **dict(x.split("=", 1) for x in kv))
            p = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
            line = [ln for ln in p.stdout.splitlines() if ln.startswith("ABJSON")]
            if not line:
                print(p.stdout[-2000:], p.stderr[-3000:])
                sys.exit(1)
            res[lib].append(json.loads(line[0][6:]))
    keys = list(dict.fromkeys(k for lib in libs for r in res[lib] for k in r))
    print(f"{'kernel':22s}" + "".join(f"{os.path.basename(lib)[-18:]:>20s}" for lib in libs))
    for k in keys:
        print(f"{k:22s}" + "".join(f"{' / '.join(str(r.get(k, '-')) for r in res[lib]):>20s}" for lib in libs))

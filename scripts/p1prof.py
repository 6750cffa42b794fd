import sys, json
import numpy as np, torch
sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from rank_overhead import NullHalo
from paper_2605_16082_b200.partition import GHOST_DEPTH, decompose, local_mesh
from paper_2605_16082_b200.scenarios import device_state_c4, make_case
from paper_2605_16082_b200.stepper import ImexStepper
case = make_case("c4", with_state=False)
out = {}
for P in (1, 8):
    parts = decompose(case.mesh, P, np.full(case.mesh.nt, case.L), depth=GHOST_DEPTH)
    lm = local_mesh(case.mesh, parts[0])
    st = ImexStepper(lm, case.L, case.params, case.dt, case.m, case.kv, case.nu_v, part=parts[0])
    st.halo = NullHalo()
    device_state_c4(case, st)
    st.use_graph = False
    st.step(1)
    st.prof = {}
    st.step(1)
    torch.cuda.synchronize()
    r = {k: (round(float(np.sum([a.elapsed_time(b) for a, b in v])), 3), len(v)) for k, v in st.prof.items()}
    print(P, json.dumps(r), flush=True)
    st.prof = None
    del st
    torch.cuda.empty_cache()

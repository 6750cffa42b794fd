import sys, torch
sys.path.insert(0, ".")
from paper_2605_16082_b200 import stepper as S
from paper_2605_16082_b200.scenarios import device_state_c4, make_case
c = make_case("c4", with_state=False)
st = S.ImexStepper(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v)
device_state_c4(c, st)
d0 = st.diagnostics()
st.step(2); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    d = st.diagnostics()
e1.record(); torch.cuda.synchronize()
print("diagnostics ms (incl. 80-byte read-back)", e0.elapsed_time(e1) / 10)
print("volume drift", (d["total_volume"] - d0["total_volume"]) / d0["total_volume"], d)

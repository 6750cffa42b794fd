"""Per-rank launch overhead of the partitioned C4 step on ONE GPU (no peers needed).

    python scripts/rank_overhead.py [P ...]      (default 2 4 8)  -> JSON line per P

Rank 0 of a P-way partition of the C4 mesh (1 M tri x 50 layers) steps alone with a no-op halo
(same launches, same local mesh incl. its 3 ghost rings, no transfers).  For each P:
  eager_host_ms   host time to issue one step's launches (ctypes, no synchronisation)
  eager_gpu_ms    device time of the eager step (CUDA events; host-bound when ~ eager_host_ms)
  graph_gpu_ms    device time of one graph replay (the whole step, one launch)
  launches        kernel launches per step; 2D RK-stage launch device time (graph) vs host issue
The halo exchanges themselves are not included (they need peers); exchanges_per_step is listed.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)


class NullHalo:
    capturable = True
    exchanges = 0

    def exchange(self, fields, deep=False):
        pass

    def start(self, fields, deep=True):
        pass

    def finish(self, fields, deep=True):
        pass


def main():
    import torch

    from paper_2605_16082_b200.partition import GHOST_DEPTH, decompose, exchanges_per_step, local_mesh
    from paper_2605_16082_b200.scenarios import device_state_c4, make_case
    from paper_2605_16082_b200.stepper import ImexStepper
    Ps = [int(a) for a in sys.argv[1:]] or [2, 4, 8]
    case = make_case("c4", with_state=False)
    for P in Ps:
        parts = decompose(case.mesh, P, np.full(case.mesh.nt, case.L), depth=GHOST_DEPTH)
        lm = local_mesh(case.mesh, parts[0])
        st = ImexStepper(lm, case.L, case.params, case.dt, case.m, case.kv, case.nu_v, part=parts[0])
        st.halo = NullHalo()
        device_state_c4(case, st)
        st.use_graph = False
        for _ in range(2):
            st.step(1)
        torch.cuda.synchronize()
        hs, gs = [], []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            t0 = time.perf_counter()
            st._launch_step(st.t)
            t1 = time.perf_counter()
            e1.record()
            torch.cuda.synchronize()
            st._advance()
            hs.append((t1 - t0) * 1e3)
            gs.append(e0.elapsed_time(e1))
        launches = st.launches_per_step()
        st.use_graph = True
        st.step(3)                       # captures the three rotating-buffer graphs
        torch.cuda.synchronize()
        rs = []
        for _ in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            st.step(1)
            e1.record()
            torch.cuda.synchronize()
            rs.append(e0.elapsed_time(e1))
        # the 2D sub-cycle launches alone: device time per RK-stage launch vs host issue time
        st.use_graph = False
        st.prof = {}
        st._launch_step(st.t)
        torch.cuda.synchronize()
        rk = [a.elapsed_time(b) for k, v in st.prof.items() if k.startswith("rk") for a, b in v]
        st.prof = None
        st._advance()
        print(json.dumps({"P": P, "n_own": parts[0].n_own, "n_local": lm.nt, "L": case.L,
                          "launches_per_step": launches, "exchanges_per_step": exchanges_per_step(case.m),
                          "eager_host_ms": float(np.median(hs)), "eager_gpu_ms": float(np.median(gs)),
                          "graph_gpu_ms": float(np.median(rs)),
                          "rk_stage_launches": len(rk), "rk_stage_gpu_us_median": float(np.median(rk) * 1e3),
                          "eager_host_us_per_launch": float(np.median(hs)) * 1e3 / launches,
                          "host_bound_without_graph": bool(np.median(hs) > 0.9 * np.median(gs))}), flush=True)
        del st
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

"""Device cost of the halo exchanges of the partitioned C4 step, measured on ONE GPU.

    python scripts/virtual_scaling.py [P ...]      (default 2 4 8)  -> JSON line per P

All P ranks of a P-way partition of the C4 mesh run in this process on one device and exchange
through the device-initiated peer-store protocol (partition.P2PGroup: the same push / pull
kernels, epochs and windows as the multi-process NVLink transport, with raw pointers instead of
CUDA IPC).  One graph replays the whole lockstep step of all ranks, so
    virtual_ms / P        = one rank's step + its share of the exchange kernels
    null_ms               = one rank's step with a no-op halo (same local mesh, rank 0)
    exchange_ms_per_rank  = virtual_ms / P - mean null rank step
is the device time the exchanges add per rank and step (pack + store + epoch + unpack launches;
the stores land in local memory here, so the NVLink transfer itself is estimated separately from
the message bytes at the NVLink 5 per-direction bandwidth).  Measurement infrastructure only.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

NVLINK_GBPS = 900.0    # NVLink 5, per direction per GPU (B200)


def _time_steps(step, n, torch):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    step(n)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def main():
    import torch

    from paper_2605_16082_b200.partition import PartitionedRun, exchanges_per_step
    from paper_2605_16082_b200.scenarios import device_state_c4, make_case
    from rank_overhead import NullHalo
    from paper_2605_16082_b200 import _lib
    for kv in filter(None, os.environ.get("PDG_TUNE", "").split(",")):   # A/B: pdg_tune key=value[,..]
        k, v = kv.split("=")
        _lib.lib().pdg_tune(int(k), int(v))
    Ps = [int(a) for a in sys.argv[1:]] or [2, 4, 8]
    case = make_case("c4", with_state=False)
    for P in Ps:
        run = PartitionedRun(case.mesh, case.L, case.params, case.dt, case.m, case.kv, case.nu_v, P,
                             transport="p2p-virtual")
        for st in run.st.values():
            device_state_c4(case, st)
        run.step(3)                                   # captures the rotating-buffer graphs
        virt = float(np.median([_time_steps(run.step, 2, torch) for _ in range(3)]))
        run.check()
        # message bytes per step of rank 0 (every exchange of the step, both directions)
        st0 = run.st[0]
        part = run.parts[0]
        planes3d = {"q": 12, "mis": 6, "uT": 18}
        n1 = sum(len(v) for v in part.send1.values())
        nd = sum(len(v) for v in part.send.values())
        L = case.L
        b3 = 2 * (planes3d["q"] * L + planes3d["mis"] + planes3d["uT"] * L) * n1 * 8     # per stage x 2 stages
        b2 = (exchanges_per_step(case.m) - 8) * 9 * nd * 8 + 2 * 6 * nd * 8           # 2D state + F3D->2D
        sent = b3 + b2
        # the same ranks with a no-op halo: the compute alone
        nulls = []
        for r, st in run.st.items():
            real = st.halo
            st.halo = NullHalo()
            st.graphs = {}
            st.step(3)
            nulls.append(float(np.median([_time_steps(st.step, 2, torch) for _ in range(3)])))
            st.halo = real
            st.graphs = {}
        print(json.dumps({
            "P": P, "transport": "p2p-virtual (all ranks on one GPU, peer-store kernels)",
            "virtual_ms_all_ranks": virt, "virtual_ms_per_rank": virt / P,
            "null_rank_ms_mean": float(np.mean(nulls)), "null_rank_ms_max": float(np.max(nulls)),
            "exchange_ms_per_rank": virt / P - float(np.mean(nulls)),
            "exchanges_per_step": exchanges_per_step(case.m),
            "rank0_sent_bytes_per_step": int(sent),
            "nvlink_ms_per_step_est": sent / (NVLINK_GBPS * 1e9) * 1e3,
            "note": "exchange_ms_per_rank = pack/store/epoch/unpack kernels on one device; the NVLink "
                    "transfer adds about nvlink_ms_per_step_est when the peers are other GPUs"}), flush=True)
        del run
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

"""e2e (host round trip per step) vs the host I/O pipeline's chunk size and staging slots at C4, plus
the raw-DMA floor of the same dependency pattern (download chunk i, then upload chunk i from the
same pinned memory, both directions pipelined) -- used to pick ImexStepper.IO_CHUNK_BYTES / IO_SLOTS.

    python scripts/e2e_sweep.py   -> one JSON line per setting
"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2605_16082_b200 import stepper as S  # noqa: E402
from paper_2605_16082_b200.scenarios import device_state_c4, make_case  # noqa: E402


def raw_floor(nbytes, chunk):
    """download chunk i -> upload chunk i (same pinned region), pipelined on two streams."""
    n = nbytes // 8
    h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    up, dn = torch.cuda.Stream(), torch.cuda.Stream()
    w = chunk // 8
    best = None
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(0, n, w):
            j = min(n, i + w)
            with torch.cuda.stream(dn):
                h[i:j].copy_(d[i:j], non_blocking=True)
                e = torch.cuda.Event()
                e.record(dn)
            up.wait_event(e)
            with torch.cuda.stream(up):
                d[i:j].copy_(h[i:j], non_blocking=True)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
        best = dt if best is None else min(best, dt)
    return best


def main():
    c = make_case("c4", with_state=False)
    st = S.ImexStepper(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v)
    device_state_c4(c, st)
    st.step(2)
    torch.cuda.synchronize()
    host = st.get_state(numpy=False)
    pin = {k: (torch.empty(v.shape, dtype=v.dtype, pin_memory=True).copy_(v) if isinstance(v, torch.Tensor) else v)
           for k, v in host.items()}
    nb = sum(v.numel() * 8 for v in pin.values() if isinstance(v, torch.Tensor))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st.step(1)
    e1.record()
    torch.cuda.synchronize()
    step_ms = e0.elapsed_time(e1)
    for chunk_mb in (32, 64, 128, 256):
        for slots in (4, 8):
            st.IO_CHUNK_BYTES = chunk_mb << 20
            st.IO_SLOTS = slots
            st._plan = None
            st._iost = None
            args = (pin["eta"], pin["qx"], pin["qy"], pin["ux"], pin["uy"], pin["T"], pin["t"])
            for _ in range(2):
                st.set_state(*args)
                st.step(1)
                st.get_state(numpy=False, out=pin)
            st.wait_io()
            torch.cuda.synchronize()
            k = 4
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record()
            for _ in range(k):
                st.set_state(*args)
                st.step(1)
                st.get_state(numpy=False, out=pin)
            st.wait_io()
            f1.record()
            torch.cuda.synchronize()
            ms = f0.elapsed_time(f1) / k
            print(json.dumps({"chunk_MB": chunk_mb, "slots": slots, "e2e_ms": ms, "step_ms": step_ms,
                              "io_ms": ms - step_ms, "raw_dma_pipelined_ms": raw_floor(nb, chunk_mb << 20),
                              "state_bytes": nb}), flush=True)


if __name__ == "__main__":
    main()

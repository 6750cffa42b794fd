"""Host-side placement for the pinned state buffers of the host I/O path (set_state / get_state).

A full C4 state is 7.27 GB each way per step, so the PCIe copies dominate an end-to-end step; when
the pinned buffers sit on the NUMA node far from the GPU, every copy also crosses the socket link.
`near_gpu(device)` pins the calling thread to the CPUs local to the GPU's PCIe root (sysfs
`local_cpulist`) for the duration of the block, so buffers allocated (and first touched) inside it
land on the GPU's node; the previous affinity is restored on exit.
"""
from __future__ import annotations

import contextlib
import os

import torch


def _parse_cpulist(text: str):
    cpus = []
    for part in text.strip().split(","):
        if not part:
            continue
        if "-" in part:
            a, b = part.split("-")
            cpus.extend(range(int(a), int(b) + 1))
        else:
            cpus.append(int(part))
    return cpus


def gpu_local_cpus(device=None):
    """CPUs on the GPU's NUMA node (sysfs local_cpulist), or None when unknown."""
    if device is None:
        d = torch.cuda.current_device()
    elif isinstance(device, int):
        d = device
    else:
        d = torch.device(device).index
        if d is None:                      # "cuda" without an index: the current device
            d = torch.cuda.current_device()
    p = torch.cuda.get_device_properties(d)
    path = f"/sys/bus/pci/devices/{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0/local_cpulist"
    try:
        with open(path) as f:
            cpus = _parse_cpulist(f.read())
    except OSError:
        return None
    allowed = os.sched_getaffinity(0)
    cpus = [c for c in cpus if c in allowed]
    return cpus or None


@contextlib.contextmanager
def near_gpu(device=None):
    """Run the block on the GPU-local CPUs (no-op when the topology is unknown); yields the CPU list."""
    cpus = None if os.environ.get("PDG_NO_NUMA") else gpu_local_cpus(device)   # PDG_NO_NUMA=1: A/B off
    if not cpus:
        yield None
        return
    old = os.sched_getaffinity(0)
    os.sched_setaffinity(0, cpus)
    try:
        yield cpus
    finally:
        os.sched_setaffinity(0, old)

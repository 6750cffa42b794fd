"""Host placement helper of the pinned state buffers (paper_2605_16082_b200/hostmem.py)."""
import pytest

from paper_2605_16082_b200.hostmem import _parse_cpulist


def test_parse_cpulist():
    assert _parse_cpulist("0-3,8,10-11\n") == [0, 1, 2, 3, 8, 10, 11]
    assert _parse_cpulist("5") == [5]
    assert _parse_cpulist("") == []


@pytest.mark.gpu
def test_near_gpu_restores_affinity():
    import os
    from paper_2605_16082_b200.hostmem import near_gpu
    before = os.sched_getaffinity(0)
    with near_gpu() as cpus:
        if cpus:
            assert os.sched_getaffinity(0) == set(cpus)
    assert os.sched_getaffinity(0) == before


@pytest.mark.gpu
def test_device_argument_forms_agree():
    """'cuda' (no index), an int and torch.device all name the current device."""
    import torch
    from paper_2605_16082_b200.hostmem import gpu_local_cpus
    cur = torch.cuda.current_device()
    ref = gpu_local_cpus(None)
    assert gpu_local_cpus("cuda") == ref
    assert gpu_local_cpus(cur) == ref
    assert gpu_local_cpus(torch.device("cuda", cur)) == ref

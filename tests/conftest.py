import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")

try:   # no GPU here: the CPU suite builds meshes with the host restatement, explicitly
    import torch
    if not torch.cuda.is_available():
        os.environ.setdefault("PDG_MESH_HOST", "1")
except ImportError:
    os.environ.setdefault("PDG_MESH_HOST", "1")


PARITY = {}   # test id -> worst normwise relative error it checked (PDG_PARITY_LOG=path writes them)


def record(name, err):
    PARITY[name] = max(PARITY.get(name, 0.0), float(err))
    return err


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("PDG_PARITY_LOG")
    if path and PARITY:
        import json
        with open(path, "w") as f:
            json.dump(dict(sorted(PARITY.items())), f, indent=1)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    def load(name):
        return dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    return load

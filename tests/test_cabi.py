"""The C-ABI library loads and exports every symbol include/prismdg_b200.h declares (CPU, no compute)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "prismdg_b200.h")).read()
    return sorted(set(re.findall(r"\b(pdg_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_header(tmp_path):
    from paper_2605_16082_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2605_16082_b200 import build
        build.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_matches_header():
    from paper_2605_16082_b200 import _lib
    declared = set(_lib.exported_symbols())
    assert set(header_symbols()) <= declared, set(header_symbols()) - declared


def test_no_cuda_no_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2605_16082_b200.device import require_cuda
    with pytest.raises(RuntimeError):
        require_cuda()

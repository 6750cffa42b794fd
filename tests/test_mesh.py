"""Product mesh setup vs golden reference vectors (bit-exact integer maps) -- CPU."""
import os
import tempfile

import numpy as np

from paper_2605_16082_b200 import mesh as PM
from paper_2605_16082_b200.params import LayerPolicy


def test_mesh_bitwise(golden):
    g = golden("mesh")
    raw = PM.make_mesh(g["vx"], g["vy"], g["vb"], g["raw_tri"])
    assert np.array_equal(raw.nbr, g["raw_nbr"]) and np.array_equal(raw.nbrk, g["raw_nbrk"])
    m = PM.hilbert_reorder(raw)
    for k in ["tri", "j2d", "dphx", "dphy", "elen", "enx", "eny", "nbr", "nbrk", "btag", "hilbert_perm", "b"]:
        assert np.array_equal(getattr(m, k), g[k]), k
    assert PM.hilbert_reorder(m).hilbert_perm.tolist() == list(range(m.nt))   # idempotent


def test_generator_matches_oracle():
    from oracle import geom as OG
    bed = lambda x, y: -10.0 - 0.001 * x
    a = PM.hilbert_reorder(PM.generate_basin_mesh(13, 7, 3e3, 2e3, bed))
    b = OG.hilbert_reorder(OG.basin_mesh(13, 7, 3e3, 2e3, bed))
    for k in ["tri", "nbr", "nbrk", "btag", "hilbert_perm", "j2d", "enx"]:
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    assert a.n_edges() == 3 * 13 * 7 + 13 + 7


def test_grid_geometry(golden):
    g = golden("mesh")
    i = golden("int3d")
    m = PM.hilbert_reorder(PM.make_mesh(g["vx"], g["vy"], g["vb"], g["raw_tri"]))
    G = PM.extrude(m, LayerPolicy(count=int(i["L"])), i["eta"])
    for k in ["z", "jz", "dzmid", "djz", "dztop", "dzbot"]:
        assert np.array_equal(getattr(G, k), i[k]), k
    G1 = PM.update_moving_mesh(G, i["eta1"], float(i["dt_mesh"]))
    assert np.array_equal(G1.w_m, i["w_m"])
    assert np.allclose(PM.total_thickness(G), i["eta"] - m.b, rtol=1e-13)


def test_mesh_file_roundtrip():
    m = PM.generate_basin_mesh(3, 2, 1.0, 1.0, lambda x, y: -1.0 - x)
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "m.txt")
        PM.write_mesh(p, m)
        r = PM.read_mesh(p)
    assert np.array_equal(r.tri, m.tri) and np.array_equal(r.vb, m.vb) and np.array_equal(r.nbr, m.nbr)


def _reference_pkg():
    """The installed reference (baseline/_ref) or its source tree; None when neither is present."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for p in (os.path.join(root, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "prismdg")):
            if p not in sys.path:
                sys.path.insert(0, p)
            return p
    return None


def test_reference_reads_product_mesh_file():
    """PRISMDG-MESH 1 written by the product is read bit-exactly by the reference reader (mesh.py:256)."""
    import pytest
    if _reference_pkg() is None:
        pytest.skip("reference package not present")
    from prismdg import mesh as RM
    m = PM.hilbert_reorder(PM.generate_basin_mesh(5, 4, 2e3, 1e3, lambda x, y: -7.0 - 0.003 * x + 1e-4 * y))
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "m.txt")
        PM.write_mesh(p, m)
        r = RM.read_mesh(p)
    for k in ("vx", "vy", "vb", "tri", "nbr", "nbrk", "btag", "j2d", "dphx", "dphy", "elen", "enx", "eny"):
        assert np.array_equal(np.asarray(getattr(r, k)), np.asarray(getattr(m, k))), k


def test_columngrid_reference_constructor():
    """ColumnGrid accepts the reference dataclass's positional fields (mesh.py:308-325)."""
    m = PM.generate_basin_mesh(3, 2, 1e3, 1e3, lambda x, y: -10.0 - 0.001 * x)
    g = PM.extrude(m, LayerPolicy(count=4), np.full((m.nt, 3), 0.1))
    h = PM.ColumnGrid(m, g.layers, g.offsets, g.fracs, g.eta, g.z, g.jz, g.w_m, g.dzmid, g.djz, g.dztop, g.dzbot)
    assert h.n_layers == 4 and h.n_prisms == g.n_prisms
    for k in ("z", "jz", "w_m", "dzmid", "djz", "dztop", "dzbot"):
        assert np.array_equal(getattr(h, k), getattr(g, k)), k
    # fields left out are derived from (eta, fracs) exactly as extrude does
    h2 = PM.ColumnGrid(m, g.layers, g.offsets, g.fracs, g.eta, None, None, None)
    assert np.array_equal(h2.z, g.z) and np.array_equal(h2.dztop, g.dztop) and not h2.w_m.any()
    if _reference_pkg() is not None:
        from prismdg import mesh as RM
        rg = RM.extrude(RM.make_mesh(m.vx, m.vy, m.vb, m.tri), RM.LayerPolicy(count=4), np.full((m.nt, 3), 0.1))
        r = PM.ColumnGrid(m, rg.layers, rg.offsets, rg.fracs, rg.eta, rg.z, rg.jz, rg.w_m)
        assert np.array_equal(r.z, g.z) and np.array_equal(r.djz, g.djz)


def test_mesh_setup_needs_gpu_or_explicit_host_flag(monkeypatch):
    """No silent CPU fallback: without a GPU, mesh setup raises unless PDG_MESH_HOST is set."""
    import pytest
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: mesh setup runs on the device")
    monkeypatch.delenv("PDG_MESH_HOST", raising=False)
    with pytest.raises(RuntimeError, match="CUDA"):
        PM.generate_basin_mesh(2, 2, 1.0, 1.0, lambda x, y: -1.0 - 0 * x)

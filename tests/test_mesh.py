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

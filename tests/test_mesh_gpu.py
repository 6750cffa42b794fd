"""Mesh2D setup on the GPU (csrc/mesh.cu) vs the host restatement and the golden reference maps."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_gpu_mesh_matches_golden(golden):
    from paper_2605_16082_b200 import mesh as PM
    g = golden("mesh")
    raw = PM.make_mesh(g["vx"], g["vy"], g["vb"], g["raw_tri"])        # GPU path
    assert np.array_equal(raw.nbr, g["raw_nbr"]) and np.array_equal(raw.nbrk, g["raw_nbrk"])
    m = PM.hilbert_reorder(raw)
    for k in ["tri", "nbr", "nbrk", "btag", "hilbert_perm", "b", "j2d", "dphx", "dphy"]:
        assert np.array_equal(getattr(m, k), g[k]), k
    for k in ["elen", "enx", "eny"]:                                     # hypot: <= 1 ulp from glibc
        assert np.allclose(getattr(m, k), g[k], rtol=4e-16, atol=0), k


@pytest.mark.parametrize("nx,ny", [(1, 1), (7, 3), (64, 40), (300, 200)])
def test_gpu_mesh_matches_host(nx, ny):
    from paper_2605_16082_b200 import mesh as PM
    bed = lambda x, y: -10.0 - 1e-3 * x + 0.0 * y  # noqa: E731
    gx, gy = np.meshgrid(np.linspace(0, 1e3 * nx, nx + 1), np.linspace(0, 7e2 * ny, ny + 1), indexing="xy")
    dev = PM.generate_basin_mesh(nx, ny, 1e3 * nx, 7e2 * ny, bed)
    host = PM.Mesh2D(vx=dev.vx, vy=dev.vy, vb=dev.vb, tri=dev.tri)._finish_host()
    for k in ["nbr", "nbrk", "btag", "j2d", "dphx", "dphy", "x", "y", "b"]:
        assert np.array_equal(getattr(dev, k), getattr(host, k)), k
    hd = PM.hilbert_reorder(dev)
    hh = PM.hilbert_reorder_host(host)
    assert np.array_equal(hd.hilbert_perm, hh.hilbert_perm)
    assert np.array_equal(hd.nbr, hh.nbr)


def test_nonmanifold_pairing():
    """Three triangles on one edge: the dict pass pairs the first two, leaves the third open."""
    from oracle import geom as OG
    from paper_2605_16082_b200 import mesh as PM
    vx = np.array([0.0, 1.0, 0.5, 0.5, 0.6])
    vy = np.array([0.0, 0.0, 1.0, -1.0, 2.0])
    tri = np.array([[0, 1, 2], [1, 0, 3], [0, 1, 4]])
    m = PM.make_mesh(vx, vy, np.full(5, -1.0), tri)
    o = OG.pair_edges(tri)
    assert np.array_equal(m.nbr, o[0]) and np.array_equal(m.nbrk, o[1]) and np.array_equal(m.btag, o[2])

"""Structural properties of the 3D operators on the GPU (the properties that pin
the reference's algorithm beyond point comparisons): r vanishes for a uniform density, the
consistent transport integrates to the external-mode transport, the lateral flux factor is
antisymmetric across every interior face, uniform flow over a flat bed gives w = 0 in columns
without walls, and `els` subsets return exactly the rows of the full evaluation."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pdg():
    import paper_2605_16082_b200 as p
    return p


def _case(pdg, bed, L=6, seed=5):
    lx, ly = 2e4, 1e4
    m = pdg.mesh.hilbert_reorder(pdg.mesh.generate_basin_mesh(14, 9, lx, ly, bed))
    rng = np.random.default_rng(seed)
    eta = 0.2 * np.cos(np.pi * m.x / lx) + 0.05 * rng.standard_normal((m.nt, 3))
    G = pdg.mesh.extrude(m, pdg.LayerPolicy(count=L), eta)
    return m, G, rng, L


def _wavy(x, y):
    return -30.0 + 8.0 * np.sin(np.pi * x / 2e4) * np.cos(2 * np.pi * y / 1e4) - 5e-4 * x


def test_r_vanishes_for_uniform_density_under_a_flat_surface(pdg):
    m, G, rng, L = _case(pdg, _wavy)
    G = pdg.mesh.extrude(m, pdg.LayerPolicy(count=L), np.zeros((m.nt, 3)))
    p = pdg.PhysParams()
    rho = np.full((m.nt * L, 6), 0.37)
    r = pdg.internal3d.compute_r(G, rho, p)
    # every term is a gradient or a jump of rho', or the surface fold rho'_s grad eta (flat here):
    # zero up to the rounding of sum_p grad phi_p = 0 and of the sigma-layer metric terms
    assert np.abs(r).max() <= 1e-12 * p.g * 0.37 * 40.0


def test_consistent_transport_column_sum(pdg):
    m, G, rng, L = _case(pdg, _wavy)
    P = m.nt * L
    I = pdg.internal3d
    q = I.project_transport(G, 0.3 * rng.standard_normal((P, 6)), 0.3 * rng.standard_normal((P, 6)))
    qbx, qby = rng.standard_normal((m.nt, 3)), rng.standard_normal((m.nt, 3))
    qb = I.consistent_transport(G, q, qbx, qby)
    s = I.column_sum(qb, G)
    for d, ref in enumerate((qbx, qby)):
        assert np.abs(s[..., d] - ref).max() <= 1e-12 * np.abs(ref).max()


def test_lateral_factor_antisymmetric(pdg):
    m, G, rng, L = _case(pdg, _wavy)
    P = m.nt * L
    I = pdg.internal3d
    q = rng.standard_normal((P, 6, 2))
    fac = I.lateral_flux_factor(G, q, pdg.PhysParams())   # (nt, L, 3, 2 vertical, 2 edge points)
    c, k = np.nonzero(m.nbr >= 0)
    e2, k2 = m.nbr[c, k], m.nbrk[c, k]
    own = fac[c, :, k]                     # (n, L, 2, 2)
    other = fac[e2, :, k2][..., ::-1]      # the neighbour traverses the edge the other way
    assert np.abs(own + other).max() <= 1e-15 * np.abs(fac).max()


def test_uniform_flow_flat_bed_has_no_vertical_velocity(pdg):
    def flat(x, y):
        return np.full_like(x, -25.0)
    lx = 2e4
    m = pdg.mesh.hilbert_reorder(pdg.mesh.generate_basin_mesh(14, 9, lx, 1e4, flat))
    L = 5
    G = pdg.mesh.extrude(m, pdg.LayerPolicy(count=L), np.zeros((m.nt, 3)))
    P = m.nt * L
    I = pdg.internal3d
    p = pdg.PhysParams()
    ux, uy = np.full((P, 6), 0.4), np.full((P, 6), -0.25)
    q = I.project_transport(G, ux, uy)
    fac = I.lateral_flux_factor(G, q, p)
    w = I.compute_w(G, q, ux, uy, p, fac).reshape(m.nt, L, 6)
    inner = np.flatnonzero((m.nbr >= 0).all(axis=1))      # columns without a wall face
    assert inner.size > 0
    assert np.abs(w[inner]).max() <= 1e-12 * 0.4


def test_els_subsets_return_the_full_rows(pdg):
    """The full evaluations run the tile-staged kernels, the subsets the per-column register
    kernels (tiles need contiguous columns): the same arithmetic up to FMA contraction, so the
    rows agree to a few ulps (projection and factor: one kernel, bitwise)."""
    m, G, rng, L = _case(pdg, _wavy)
    P = m.nt * L
    I = pdg.internal3d
    p = pdg.PhysParams(alpha=0.2, t_ref=12.5)
    ux, uy = 0.3 * rng.standard_normal((P, 6)), 0.3 * rng.standard_normal((P, 6))
    rho = rng.standard_normal((P, 6))
    els = np.sort(rng.choice(m.nt, size=m.nt // 3, replace=False))
    rows = (els[:, None] * L + np.arange(L)[None, :]).ravel()
    full_r, sub_r = I.compute_r(G, rho, p), I.compute_r(G, rho, p, els=els)
    assert np.abs(sub_r[rows] - full_r[rows]).max() <= 4e-16 * np.abs(full_r).max()
    full_q, sub_q = I.project_transport(G, ux, uy), I.project_transport(G, ux, uy, els=els)
    assert np.array_equal(np.asarray(sub_q).reshape(-1, 6, 2)[rows] if sub_q.shape[0] == P else sub_q,
                          full_q[rows])
    q = full_q
    full_f, sub_f = I.lateral_flux_factor(G, q, p), I.lateral_flux_factor(G, q, p, els=els)
    assert np.array_equal(sub_f[els] if sub_f.shape[0] == m.nt else sub_f, full_f[els])

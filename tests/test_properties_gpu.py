"""Structural properties of the 3D operators on the GPU (the properties that pin
the reference's algorithm beyond point comparisons): r vanishes for a uniform density, the
consistent transport integrates to the external-mode transport, the lateral flux factor is
antisymmetric across every interior face, uniform flow over a flat bed gives w = 0 in columns
without walls, `els` subsets return exactly the rows of the full evaluation, and the column sum
of the w~ right-hand side is the free-surface residual of the external transport (criterion 6b)."""
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


@pytest.mark.parametrize("surface", ["flat", "elementwise_jumps"])
def test_r_vanishes_for_uniform_density(pdg, surface):
    """SPEC criterion 11: constant rho' gives r = 0 -- also with a free surface that is constant on
    each element and jumps between elements (every term is a gradient or a jump of rho', or the
    surface fold rho'_s grad eta, which vanishes inside each element)."""
    m, G, rng, L = _case(pdg, _wavy)
    eta = np.zeros((m.nt, 3)) if surface == "flat" else np.repeat(0.3 * rng.standard_normal((m.nt, 1)), 3, axis=1)
    G = pdg.mesh.extrude(m, pdg.LayerPolicy(count=L), eta)
    p = pdg.PhysParams()
    rho = np.full((m.nt * L, 6), 0.37)
    r = pdg.internal3d.compute_r(G, rho, p)
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


def _wtilde_rhs_column_sum(pdg, G, w, L):
    """Rebuild the w~ right-hand side from w~ (the bed-anchored sweep inverted, columns.py:125-151:
    g_t = (w_t - w_b)/2, g_b = (w_t + w_b)/2 - w_t(below), rhs = Mh g) and sum it over the column."""
    nt = G.mesh.nt
    w = np.asarray(w).reshape(nt, L, 6)
    j2d = np.asarray(G.mesh.j2d)
    mh = lambda v: pdg.columns.apply_mh(v, j2d)   # noqa: E731
    out = np.zeros((nt, 3))
    s = np.zeros((nt, 3))
    for l in range(L - 1, -1, -1):
        wt, wb = w[:, l, 0:3], w[:, l, 3:6]
        out += np.asarray(mh(0.5 * (wt - wb))) + np.asarray(mh(0.5 * (wt + wb) - s))
        s = wt
    return out


def test_wtilde_rhs_column_sum_is_the_free_surface_residual(pdg):
    """SPEC criterion 6b: the column sum of the w~ right-hand side equals
    rhs_free_surface with the external-mode transport Qbar -- for the API w~ (compute_wtilde) and
    for the w~ the stepper forms inside the stage RHS (pdg_step_rhs_ut_w, q~ = q + Jz mis)."""
    import torch

    from paper_2605_16082_b200 import _lib
    from paper_2605_16082_b200.device import ptr, stream_ptr
    m, G, rng, L = _case(pdg, _wavy)
    P = m.nt * L
    I = pdg.internal3d
    p = pdg.PhysParams()
    ux, uy = 0.3 * rng.standard_normal((P, 6)), 0.3 * rng.standard_normal((P, 6))
    q = I.project_transport(G, ux, uy)
    qbx, qby = rng.standard_normal((m.nt, 3)), rng.standard_normal((m.nt, 3))
    qb = I.consistent_transport(G, q, qbx, qby)
    fs = np.asarray(pdg.external2d.rhs_free_surface(pdg.State2D(np.asarray(G.eta), qbx, qby, 0.0), m, p))
    scale = np.abs(fs).max()
    w_api = I.compute_wtilde(G, qb, I.lateral_flux_factor(G, qb, p))
    assert np.abs(_wtilde_rhs_column_sum(pdg, G, w_api, L) - fs).max() <= 1e-13 * scale
    # the stepper's w~: the stage RHS with its mismatch, on the same grid (eta0 = eta1 = eta)
    st = pdg.stepper.ImexStepper(m, L, p, 30.0, 2, 1e-3, 1e-4)
    st.set_state(np.asarray(G.eta), qbx, qby, ux, uy, np.full((P, 6), 10.0))
    lib, h = _lib.lib(), st.dm.h
    eta = st.S[0]
    u, T = st.U[st.cur], st.T[st.cur]
    assert lib.pdg_project_transport(h, ptr(eta), ptr(u[0]), ptr(u[1]), None, None, 0, ptr(st.q), ptr(st.qsum),
                                     ptr(st.htot), stream_ptr()) == 0
    qbar2d = torch.as_tensor(np.stack([qbx.T, qby.T]).copy(), device=st.dev)     # [2][3][nt]
    assert lib.pdg_mismatch(h, ptr(qbar2d), ptr(st.qsum), ptr(st.htot), ptr(st.mis), stream_ptr()) == 0
    w = torch.zeros_like(st.wt)
    ou, oT = torch.zeros_like(u), torch.zeros_like(T)
    assert lib.pdg_step_rhs_ut_w(h, ptr(eta), ptr(eta), ptr(eta), ptr(u), ptr(T), ptr(u), ptr(T), ptr(st.q),
                                 ptr(st.mis), ptr(st.r), ptr(st.f2d), p.g, p.f, p.rho0, 0.0, 0.0, 0.0, 30.0,
                                 ptr(ou), ptr(oT), ptr(w), stream_ptr()) == 0
    torch.cuda.synchronize()
    w_rows = np.asarray(w.cpu()).reshape(6, L, m.nt).transpose(2, 1, 0).reshape(P, 6)
    assert np.abs(_wtilde_rhs_column_sum(pdg, G, w_rows, L) - fs).max() <= 1e-13 * scale


def test_linear_flow_flat_bed_analytic_vertical_velocity(pdg):
    """SURVEY.md section 4 known answer: u = (x / Lx, 0) over a flat bed gives w = -(z - b) div u =
    -(z - b) / Lx at every node of the columns without walls (P1 represents u exactly)."""
    def flat(x, y):
        return np.full_like(x, -25.0)
    lx = 2e4
    m = pdg.mesh.hilbert_reorder(pdg.mesh.generate_basin_mesh(14, 9, lx, 1e4, flat))
    L = 5
    G = pdg.mesh.extrude(m, pdg.LayerPolicy(count=L), np.zeros((m.nt, 3)))
    P = m.nt * L
    I = pdg.internal3d
    p = pdg.PhysParams()
    xs = np.asarray(m.x) / lx                                        # (nt, 3) corners
    ux = np.repeat(np.concatenate([xs, xs], axis=1), L, axis=0)      # (P, 6): p = c L + l
    uy = np.zeros((P, 6))
    q = I.project_transport(G, ux, uy)
    w = np.asarray(I.compute_w(G, q, ux, uy, p, I.lateral_flux_factor(G, q, p))).reshape(m.nt, L, 6)
    f = np.arange(L + 1) / L                                         # uniform sigma fractions
    H = 25.0
    z_minus_b = np.empty((L, 6))
    for lev, fr in ((0, f[:-1]), (1, f[1:])):
        z_minus_b[:, 3 * lev:3 * lev + 3] = (H - fr * H)[:, None]
    ref = -z_minus_b / lx
    inner = np.flatnonzero((m.nbr >= 0).all(axis=1))
    assert inner.size > 0
    assert np.abs(w[inner] - ref[None]).max() <= 1e-12 * np.abs(ref).max()


def test_projection_reproduces_constant_transport(pdg):
    """SURVEY.md section 4 known answer: on a flat surface over a flat bed (constant Jz) a constant
    velocity projects to q = Jz u exactly (to rounding)."""
    def flat(x, y):
        return np.full_like(x, -20.0)
    m = pdg.mesh.hilbert_reorder(pdg.mesh.generate_basin_mesh(10, 7, 1e4, 1e4, flat))
    L = 4
    G = pdg.mesh.extrude(m, pdg.LayerPolicy(count=L), np.zeros((m.nt, 3)))
    P = m.nt * L
    q = np.asarray(pdg.internal3d.project_transport(G, np.full((P, 6), 0.7), np.full((P, 6), -0.2)))
    jz = 0.5 * 20.0 / L
    assert np.abs(q[..., 0] - 0.7 * jz).max() <= 1e-14 * 0.7 * jz
    assert np.abs(q[..., 1] + 0.2 * jz).max() <= 1e-14 * 0.7 * jz

"""3D internal-mode assemblies and column solvers: CUDA path vs CPU oracle / golden reference vectors."""
import numpy as np
import pytest

from oracle import colsolve as OC
from oracle import ext2d as OE
from oracle import geom as OG
from oracle import int3d as O

pytestmark = pytest.mark.gpu
TOL = 1e-12


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.fixture(scope="module")
def pdg():
    import paper_2605_16082_b200 as p
    return p


@pytest.fixture(scope="module")
def case(pdg):
    """Random non-equilibrium state on a wavy-bed Hilbert-ordered basin, L = 5."""
    lx, ly = 2e4, 1e4

    def bed(x, y):
        return -30.0 + 8.0 * np.sin(np.pi * x / lx) * np.cos(2 * np.pi * y / ly) - 5e-4 * x
    m = pdg.mesh.hilbert_reorder(pdg.mesh.generate_basin_mesh(16, 10, lx, ly, bed))
    om = OG.hilbert_reorder(OG.basin_mesh(16, 10, lx, ly, bed))
    rng = np.random.default_rng(11)
    nt, L = m.nt, 5
    eta = 0.2 * np.cos(np.pi * m.x / lx) + 0.05 * rng.standard_normal((nt, 3))
    eta1 = eta + 0.02 * rng.standard_normal((nt, 3))
    G = pdg.mesh.extrude(m, pdg.LayerPolicy(count=L), eta)
    G1 = pdg.mesh.update_moving_mesh(G, eta1, 7.0)
    OGr = OG.extrude(om, L, eta)
    OG1 = OG.update_moving_mesh(OGr, eta1, 7.0)
    P = nt * L
    p = pdg.PhysParams(f=1.2e-4, alpha=0.2, t_ref=12.5)
    d = dict(m=m, G=G, G1=G1, OG=OGr, OG1=OG1, p=p, nt=nt, L=L, P=P,
             ux=0.3 * rng.standard_normal((P, 6)), uy=0.3 * rng.standard_normal((P, 6)),
             T=12.5 + rng.standard_normal((P, 6)), qbx=rng.standard_normal((nt, 3)), qby=rng.standard_normal((nt, 3)),
             rng=rng)
    d["rho"] = OE.eos(d["T"], p)
    d["M"] = O.prism_mass(OGr)
    d["q"] = O.project_transport(OGr, d["ux"], d["uy"], mass=d["M"])
    d["fac"] = O.lateral_flux_factor(OGr, d["q"], p)
    d["r"] = O.compute_r(OGr, d["rho"], p)
    d["qb"] = O.consistent_transport(OGr, d["q"], d["qbx"], d["qby"])
    d["facb"] = O.lateral_flux_factor(OGr, d["qb"], p)
    d["wt"] = O.compute_wtilde(OGr, d["qb"], d["facb"])
    return d


def test_mass_projection(pdg, case):
    c = case
    I = pdg.internal3d
    M = I.prism_mass(c["G"])
    assert rel(M, c["M"]) <= TOL
    assert rel(I.project_transport(c["G"], c["ux"], c["uy"]), c["q"]) <= TOL            # Kronecker path
    assert rel(I.project_transport(c["G"], c["ux"], c["uy"], mass=c["M"]), c["q"]) <= TOL  # explicit-mass LU path
    f = c["rng"].standard_normal((c["P"], 6, 2))
    assert rel(I.mass_apply(c["M"], f), O.mass_apply(c["M"], f)) <= TOL
    assert rel(I.mass_solve(c["M"], f, c["G"]), O.mass_solve(c["M"], f, c["OG"])) <= TOL
    els = np.array([3, 0, 100])
    assert rel(I.mass_solve(c["M"], f[..., 0], c["G"], els=els), O.mass_solve(c["M"], f[..., 0], c["OG"], els=els)) <= TOL
    assert rel(I.column_sum(c["q"], c["G"]), O.column_sum(c["q"], c["OG"])) <= TOL
    assert rel(I.consistent_transport(c["G"], c["q"], c["qbx"], c["qby"]), c["qb"]) <= TOL


def test_factor_r_w(pdg, case):
    c = case
    I = pdg.internal3d
    assert rel(I.lateral_flux_factor(c["G"], c["q"], c["p"]), c["fac"]) <= TOL
    assert rel(I.compute_r(c["G"], c["rho"], c["p"]), c["r"]) <= TOL
    w = O.compute_w(c["OG"], c["q"], c["ux"], c["uy"], c["p"], c["fac"])
    assert rel(I.compute_w(c["G"], c["q"], c["ux"], c["uy"], c["p"], c["fac"]), w) <= TOL
    assert rel(I.compute_wtilde(c["G"], c["qb"], c["facb"]), c["wt"]) <= TOL
    els = np.array([7, 2, 250])
    assert rel(I.compute_r(c["G"], c["rho"], c["p"], els=els), O.compute_r(c["OG"], c["rho"], c["p"], els=els)) <= TOL


def test_horizontal_rhs(pdg, case):
    c = case
    I = pdg.internal3d
    Fh = O.horizontal_rhs(c["OG"], c["ux"], c["uy"], c["qb"], c["facb"], c["r"], c["M"], c["p"])
    assert rel(I.horizontal_rhs(c["G"], c["ux"], c["uy"], c["qb"], c["facb"], c["r"], c["M"], c["p"]), Fh) <= TOL
    els = np.array([1, 9, 40])
    Fe = O.horizontal_rhs(c["OG"], c["ux"], c["uy"], c["q"], c["fac"], c["r"], c["M"], c["p"], els=els)
    assert rel(I.horizontal_rhs(c["G"], c["ux"], c["uy"], c["q"], c["fac"], c["r"], c["M"], c["p"], els=els), Fe) <= TOL
    Ft = O.tracer_horizontal_rhs(c["OG"], c["T"], c["qb"], c["facb"], c["p"])
    assert rel(I.tracer_horizontal_rhs(c["G"], c["T"], c["qb"], c["facb"], c["p"]), Ft) <= TOL
    st = O.stress_rhs(c["OG"], 1e-4, -3e-5, 2.5e-3, c["ux"], c["uy"])
    assert rel(I.stress_rhs(c["G"], 1e-4, -3e-5, 2.5e-3, c["ux"], c["uy"]), st) <= TOL
    # explicit horizontal viscosity: the patched oracle (tests/test_hdiff_gpu.py has the golden vectors)
    pv = pdg.PhysParams(f=c["p"].f, kappa_h=3.0, nu_h=2.0)
    assert rel(I.horizontal_rhs(c["G"], c["ux"], c["uy"], c["q"], c["fac"], c["r"], c["M"], pv),
               O.horizontal_rhs(c["OG"], c["ux"], c["uy"], c["q"], c["fac"], c["r"], c["M"],
                                pv)) <= TOL
    assert rel(I.tracer_horizontal_rhs(c["G"], c["T"], c["qb"], c["facb"], pv),
               O.tracer_horizontal_rhs(c["OG"], c["T"], c["qb"], c["facb"], pv)) <= TOL


def test_vertical_operator_and_solvers(pdg, case):
    c = case
    I, C = pdg.internal3d, pdg.columns
    wm = c["OG1"].w_m
    assert rel(c["G1"].w_m, wm) <= 1e-13
    A = O.assemble_vertical_operator(c["OG"], c["wt"], wm, 0.7, 1e-3)
    B = I.assemble_vertical_operator(c["G"], c["wt"], wm, 0.7, 1e-3)
    for k in "duw":
        assert rel(getattr(B, k), getattr(A, k)) <= TOL, k
    els = np.array([4, 33])
    Ae = O.assemble_vertical_operator(c["OG"], c["wt"], wm, 0.7, 1e-3, els=els)
    Be = I.assemble_vertical_operator(c["G"], c["wt"], wm, 0.7, 1e-3, els=els)
    for k in "duw":
        assert rel(getattr(Be, k), getattr(Ae, k)) <= TOL, k
    M1 = O.prism_mass(c["OG1"])
    Ai = O.build_implicit(M1, A, 30.0, c["OG"])
    Bi = I.build_implicit(M1, A, 30.0, c["G"])
    for k in "duw":
        assert rel(getattr(Bi, k), getattr(Ai, k)) <= TOL, k
    rhs = c["rng"].standard_normal((c["nt"], c["L"], 6, 2))
    x = OC.block_thomas(Ai, rhs)
    assert rel(C.solve_banded_column(Ai, rhs), x) <= 1e-11
    assert rel(C.solve_banded_column(Ai, rhs[..., 0]), OC.block_thomas(Ai, rhs[..., 0])) <= 1e-11
    assert rel(C.apply_banded(Ai, rhs), OC.banded_matvec(Ai, rhs)) <= TOL


def test_column_solvers_golden(pdg, golden):
    g = golden("columns")
    C = pdg.columns
    assert rel(C.solve_r_column(g["rhs"], g["j2d"]), g["r_out"]) <= TOL
    assert rel(C.solve_w_column(g["rhs"], g["j2d"]), g["w_out"]) <= TOL
    assert rel(C.apply_mh(g["rhs"][:, 0, 0:3], g["j2d"]), g["mh"]) <= TOL
    assert rel(C.apply_mh_inv(g["rhs"][:, 0, 0:3], g["j2d"]), g["mhinv"]) <= TOL
    assert rel(C.solve_tridiagonal(g["lower"], g["diag"], g["upper"], g["trhs"]), g["tri_x"]) <= 1e-12


def test_sweeps_vs_dense_oracle(pdg):
    """SPEC acceptance 1: matrix-free sweeps invert the dense D_vu / D_vd, L = 1..40."""
    C = pdg.columns
    rng = np.random.default_rng(0)
    for L in (1, 2, 7, 40):
        j2d = 0.5 + rng.random(6)
        rhs = rng.standard_normal((6, L, 6))
        r = C.solve_r_column(rhs, j2d)
        w = C.solve_w_column(rhs, j2d)
        for col in range(6):
            mh = OC.__dict__.get("np", np).array([[2.0, 1, 1], [1, 2, 1], [1, 1, 2]]) / 24.0 * j2d[col]
            Dr = OC.dense_sweep_matrix("r", L, mh)
            Dw = OC.dense_sweep_matrix("w", L, mh)
            assert rel(Dr @ r[col].ravel(), rhs[col].ravel()) <= 1e-11
            assert rel(Dw @ w[col].ravel(), rhs[col].ravel()) <= 1e-11


def test_golden_int3d(pdg, golden):
    g = golden("mesh")
    e = golden("int3d")
    m = pdg.mesh.hilbert_reorder(pdg.mesh.make_mesh(g["vx"], g["vy"], g["vb"], g["raw_tri"]))
    L = int(e["L"])
    G = pdg.mesh.extrude(m, pdg.LayerPolicy(count=L), e["eta"])
    p = pdg.PhysParams(f=1e-4, cd=2.5e-3, alpha=0.2, t_ref=12.5)
    I, C = pdg.internal3d, pdg.columns
    assert rel(I.prism_mass(G), e["mass"]) <= TOL
    assert rel(I.project_transport(G, e["ux"], e["uy"], mass=e["mass"]), e["q"]) <= TOL
    assert rel(I.lateral_flux_factor(G, e["q"], p), e["fac"]) <= TOL
    assert rel(I.compute_r(G, e["rho"], p), e["r"]) <= TOL
    assert rel(I.compute_w(G, e["q"], e["ux"], e["uy"], p, e["fac"]), e["w"]) <= TOL
    assert rel(I.consistent_transport(G, e["q"], e["qbx"], e["qby"]), e["qb"]) <= TOL
    assert rel(I.compute_wtilde(G, e["qb"], e["facb"]), e["wt"]) <= TOL
    assert rel(I.horizontal_rhs(G, e["ux"], e["uy"], e["qb"], e["facb"], e["r"], e["mass"], p), e["Fh"]) <= TOL
    assert rel(I.tracer_horizontal_rhs(G, e["T"], e["qb"], e["facb"], p), e["Ft"]) <= TOL
    A = I.assemble_vertical_operator(G, e["wt"], e["w_m"], 0.5, 1e-3)
    assert rel(A.d, e["A_d"]) <= TOL and rel(A.u, e["A_u"]) <= TOL and rel(A.w, e["A_w"]) <= TOL
    from paper_2605_16082_b200.params import BandedColumnMatrix
    Ai = BandedColumnMatrix(e["Ai_d"], e["Ai_u"], e["Ai_w"])
    assert rel(C.solve_banded_column(Ai, e["rhs"]), e["xb"]) <= 1e-11
    assert rel(I.compute_r(G, e["rho"], p, els=e["els"]), e["r_els"]) <= TOL
    assert rel(I.horizontal_rhs(G, e["ux"], e["uy"], e["q"], e["fac"], e["r"], e["mass"], p, els=e["els"]),
               e["Fh_els"]) <= TOL


def test_zero_pivot(pdg):
    C = pdg.columns
    from paper_2605_16082_b200.params import BandedColumnMatrix
    d = np.zeros((2, 3, 6, 6))
    d[:] = np.eye(6)
    d[1, 2, 4, 4] = 0.0
    mat = BandedColumnMatrix(d, np.zeros((2, 3, 3, 6)), np.zeros((2, 3, 3, 6)))
    with pytest.raises(pdg.errors.ZeroPivot) as ei:
        C.solve_banded_column(mat, np.ones((2, 3, 6)))
    assert ei.value.layer == 2 and ei.value.node == 4


def test_solve_banded_sequential_vs_reference(pdg, golden):
    """solve_banded_sequential (columns.py:404-485): the solution and the working-set record."""
    g = golden("seqsolve")
    mat = pdg.BandedColumnMatrix(d=g["d"], u=g["u"], w=g["w"])
    x, st = pdg.columns.solve_banded_sequential(mat, g["rhs"], int(g["col"]))
    assert np.abs(x - g["x"]).max() <= 1e-12 * np.abs(g["x"]).max()
    assert (st.max_live, st.loads, st.stores) == (int(g["max_live"]), int(g["loads"]), int(g["stores"]))
    assert sorted(f"{k}{l}" for k, l in st.touched) == g["touched"].tolist()

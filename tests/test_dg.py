"""dg.py tables (CPU, bitwise) and pointwise helpers (GPU) against the reference
(tests/golden/dg.npz, scripts/make_golden_dg.py)."""
import numpy as np
import pytest

from paper_2605_16082_b200 import dg


def test_tables_bitwise(golden):
    g = golden("dg")
    for k in ("TRI_QW", "TRI_BARY", "TRI_QP", "SEG_QP", "SEG_QW", "VERT_SHAPE", "DVERT", "EDGE_SHAPE", "DPHI_PARENT"):
        assert np.array_equal(getattr(dg, k), g[k]), k


@pytest.mark.gpu
def test_helpers_vs_reference(golden):
    g = golden("dg")
    close = lambda x, y: np.abs(np.asarray(x) - y).max() <= 1e-14 * max(np.abs(y).max(), 1.0)  # noqa: E731
    assert close(dg.tri_quad(g["v"]), g["tri_quad"])
    assert np.array_equal(dg.iface_mean(g["a"], g["b"]), g["mean"])
    assert np.array_equal(dg.iface_diff(g["a"], g["b"]), g["diff"])
    assert np.array_equal(dg.iface_max(g["a"], g["b"]), g["mx"])
    assert np.array_equal(dg.iface_upwind(g["a"], g["b"], g["s"]), g["up"])
    assert close(dg.penalty_sigma(g["la"], g["lb"]), g["pen"])
    assert close(dg.penalty_sigma(g["la"], g["lb"], dim=2), g["pen2"])
    mh, mz = dg.metric_vector(g["dzm"], g["dzj"], g["jz"], g["zeta"])
    assert close(mh, g["mh"]) and close(mz, g["mz"])
    giso, gm = dg.gradient_decompose(g["gx"], g["fz"], g["mh"], g["mz"])
    assert close(giso, g["giso"]) and close(gm, g["gm"])
    ut, wt = dg.split_velocity(g["u"], g["w"], g["mh"], g["mz"])
    assert close(ut, g["ut"]) and close(wt, g["wt"])
    sd = dg.split_diffusivity(g["D"], g["mh"], g["mz"])
    assert close(sd.kappa_i, g["kappa_i"]) and close(sd.d_e, g["d_e"])
    assert close(dg.kappa_implicit(2.0, 1e-3, g["mh"], g["mz"]), g["kimp"])
    with pytest.raises(Exception):
        dg.penalty_sigma(np.array([0.0]), np.array([1.0]))
    with pytest.raises(Exception):
        dg.metric_vector(g["dzm"][:1], g["dzj"][:1], np.array([-1.0]), g["zeta"][:1])

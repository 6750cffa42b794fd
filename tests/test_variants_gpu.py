"""Every kernel variant kept in the library (pdg_tune keys) steps to the same state as the default.

The defaults (csrc/ctx.cu g_tune) are the measured-fastest variants; the alternatives stay in the
library for A/B runs (scripts/ab_tune.py) and must keep producing the same answer:
  key 7  implicit vertical stage: 2 split factored block Thomas (30-double tiles: E_l, S0, S1),
         4 as 2 with the coupling blocks S0, S1 rebuilt in the back substitution (18-double tiles)
  key 9  F3D->2D: 0 register kernel, 64 / 128 tile-staged (shared-memory neighbour traces)
  key 11 r / w~: 0 register kernels, 64 / 128 tile-staged
  key 5  stage RHS: 1 register kernel (128-thread blocks), 8 shared-memory column constants
  key 6  2D RK stage occupancy variant (register allocation can change FMA contraction); 8 (default)
         = 2 launched with programmatic dependent launch (same kernel arithmetic)
  key 12 bit 1: cp.async.bulk (copy-engine) staging ring + mbarriers in the implicit forward
         elimination instead of per-thread cp.async (900 columns: the last block splits a warp)
Tile-staged and register kernels do the same arithmetic (bitwise equal), except the tile-staged
F3D->2D kernel, which forms the column sum per horizontal node (rounding-level difference); the
split Thomas and the branch-free reciprocals of the staged vertical kernels differ at rounding level.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KEYS = (5, 6, 7, 9, 10, 11, 12)


@pytest.fixture(scope="module")
def case():
    import torch

    import paper_2605_16082_b200 as pdg
    from paper_2605_16082_b200 import _lib
    from paper_2605_16082_b200.scenarios import make_case
    c = make_case("c4", scale=0.03, L=12)          # 30 x 15 squares of the C4 basin (900 columns)
    lib = _lib.lib()
    defaults = {k: lib.pdg_tune(k, -1) for k in KEYS}
    yield pdg, c, lib, defaults
    for k, v in defaults.items():
        lib.pdg_tune(k, v)
    torch.cuda.synchronize()


def run(pdg, c, lib, defaults, setting, steps=3, **attrs):
    for k, v in defaults.items():
        lib.pdg_tune(k, v)
    for k, v in setting.items():
        lib.pdg_tune(k, v)
    st = pdg.stepper.ImexStepper(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v)
    st.use_graph = False
    for k, v in attrs.items():
        setattr(st, k, v)
    st.set_state(**c.state)
    st.step(steps)
    st.check()
    return st.get_state()


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("setting,tol", [
    ({7: 2}, 1e-11),
    ({9: 0}, 1e-12), ({9: 64}, 0.0),
    ({11: 0}, 1e-12), ({11: 64}, 0.0),   # 11=0: register r kernel, F3D->2D then reads r (default: its layer sum)
    # 5=1 / 10=128: other stage-RHS kernels (per-layer masses, another summation order)
    ({5: 1}, 1e-11), ({10: 128}, 1e-11),
    ({6: 0}, 1e-12), ({6: 3}, 1e-12), ({6: 2}, 0.0),   # default 8 = 2 + programmatic dependent launch
    ({12: 3}, 0.0),     # bulk-copy (TMA) ring of the implicit forward elimination: same arithmetic
])
def test_variant_matches_default(case, setting, tol):
    pdg, c, lib, defaults = case
    ref = run(pdg, c, lib, defaults, {})
    got = run(pdg, c, lib, defaults, setting)
    for k in ("eta", "qx", "qy", "ux", "uy", "T"):
        err = rel(got[k], ref[k])
        assert err <= tol, (setting, k, err)



@pytest.mark.parametrize("attrs", [
    {"concurrent_rp": True}, {"concurrent_vertical": True},
    {"concurrent_rp": True, "concurrent_vertical": True, "use_graph": True},
])
def test_second_stream_variants_bitwise(case, attrs):
    """The step-graph variants with a second stream (r beside the projection, PDG_CONC_RP; the tracer
    vertical solve beside the momentum one, PDG_CONC_VERT; both measured without gain, DESIGN.md
    section 5) run the same kernels on independent data: bitwise equal to the single-stream step."""
    pdg, c, lib, defaults = case
    ref = run(pdg, c, lib, defaults, {})
    got = run(pdg, c, lib, defaults, {}, **attrs)
    for k in ("eta", "qx", "qy", "ux", "uy", "T"):
        assert np.array_equal(got[k], ref[k]), (attrs, k)


@pytest.mark.parametrize("implicit", [1, 0])
def test_vertical_column_lists_bitwise(case, implicit):
    """pdg_step_vertical_cols over two complementary column lists == one launch over all columns
    (per-column work; the lists may be in any order)."""
    import torch
    from paper_2605_16082_b200.device import ptr, stream_ptr
    pdg, c, lib, defaults = case
    for k, v in defaults.items():
        lib.pdg_tune(k, v)
    st = pdg.stepper.ImexStepper(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v)
    st.use_graph = False
    st.set_state(**c.state)
    st.step(1)
    h, pe, eta, u = st.dm.h, st.pen, st.S[0], st.U[st.cur]
    rng = np.random.default_rng(11)
    perm = rng.permutation(c.mesh.nt).astype(np.int32)
    parts = [torch.as_tensor(np.sort(perm[:97])), torch.as_tensor(perm[97:])]
    outs = []
    for lists in (None, parts):
        out = torch.zeros_like(u)
        for cols in ([None] if lists is None else lists):
            cd = None if cols is None else cols.to("cuda")
            rc = lib.pdg_step_vertical_cols(h, 2, implicit, ptr(eta), ptr(eta), ptr(eta), 0.5 * c.dt, ptr(st.wt), 0.0,
                                            st.kv, pe.n0, pe.order, 0.5 * c.dt, ptr(u), ptr(u), ptr(out), ptr(cd),
                                            0 if cd is None else cd.numel(), stream_ptr())
            assert rc == 0
        torch.cuda.synchronize()
        outs.append(out.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])


def test_r_layer_sum(case):
    """pdg_step_r's rsum is the sum over the layers of jm (r_top + r_bot) of the r it writes
    (jm = (f_b - f_t) / 2), accumulated in layer order (the device contracts each step into an FMA:
    equal to the host sum up to a few ulps)."""
    import ctypes

    import torch
    from paper_2605_16082_b200.device import ptr, stream_ptr
    pdg, c, lib, defaults = case
    for k, v in defaults.items():
        lib.pdg_tune(k, v)
    st = pdg.stepper.ImexStepper(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v)
    st.use_graph = False
    st.set_state(**c.state)
    st.step(1)
    r = torch.zeros_like(st.r)
    rsum = torch.zeros(2, 3, c.mesh.nt, dtype=torch.float64, device="cuda")
    ok = ctypes.c_int(0)
    p = c.params
    assert lib.pdg_step_r(st.dm.h, ptr(st.S[0]), ptr(st.T[st.cur]), p.alpha, p.t_ref, p.g, ptr(r), ptr(rsum),
                          ctypes.byref(ok), stream_ptr()) == 0
    torch.cuda.synchronize()
    assert ok.value == 1
    rn, got = r.cpu().numpy(), rsum.cpu().numpy()          # r: [2][6][L][nt]
    fr = st.dm._fracs                                      # the sigma fractions the kernels use
    want = np.zeros_like(got)
    for l in range(c.L):
        jm = 0.5 * (fr[l + 1] - fr[l])
        want = want + jm * (rn[:, 0:3, l, :] + rn[:, 3:6, l, :])
    assert np.abs(got - want).max() <= 1e-14 * np.abs(want).max()


def test_wtilde_inside_the_stage_rhs(case):
    """pdg_step_rhs_ut_w forms w~ in the stage-RHS layer loop (bottom-up, k_hrhs_s<.., WT>): the
    same w~ as pdg_compute_wtilde on the stage's q and mismatch, and the same step."""
    import torch
    pdg, c, lib, defaults = case
    for k, v in defaults.items():
        lib.pdg_tune(k, v)
    st = pdg.stepper.ImexStepper(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v)
    st.use_graph = False
    st.set_state(**c.state)
    st.step(1)
    from paper_2605_16082_b200.device import ptr, stream_ptr
    h, p = st.dm.h, c.params
    g = torch.Generator(device="cpu").manual_seed(5)
    mis = (1e-3 * torch.randn(st.mis.shape, generator=g, dtype=torch.float64)).to(st.mis.device)
    u, T = st.U[st.cur], st.T[st.cur]
    eta = st.S[0]
    eta1 = eta + 1e-3
    st.q.zero_()
    lib.pdg_project_transport(h, ptr(eta), ptr(u[0]), ptr(u[1]), None, None, 0, ptr(st.q), ptr(st.qsum), ptr(st.htot),
                              stream_ptr())
    w_ref, w_got = torch.zeros_like(st.wt), torch.zeros_like(st.wt)
    ou, oT = torch.zeros_like(u), torch.zeros_like(T)
    ou2, oT2 = torch.zeros_like(u), torch.zeros_like(T)
    assert lib.pdg_compute_wtilde(h, ptr(eta), ptr(st.q), None, ptr(mis), p.g, None, 0, ptr(w_ref), stream_ptr()) == 0
    args = (h, ptr(eta), ptr(eta), ptr(eta1), ptr(u), ptr(T), ptr(u), ptr(T), ptr(st.q), ptr(mis), ptr(st.r),
            ptr(st.f2d), p.g, p.f, p.rho0, 0.01, -0.02, p.cd, 30.0)
    assert lib.pdg_step_rhs_ut(*args, ptr(ou), ptr(oT), stream_ptr()) == 0
    assert lib.pdg_step_rhs_ut_w(*args, ptr(ou2), ptr(oT2), ptr(w_got), stream_ptr()) == 0
    torch.cuda.synchronize()
    assert torch.equal(ou, ou2) and torch.equal(oT, oT2)
    err = float((w_got - w_ref).abs().max() / w_ref.abs().max())
    assert err <= 1e-14, err
    ref = run(pdg, c, lib, defaults, {}, fuse_wt=False)
    got = run(pdg, c, lib, defaults, {}, fuse_wt=True)
    for k in ("eta", "qx", "qy", "ux", "uy", "T"):
        assert rel(got[k], ref[k]) <= 1e-13, (k, rel(got[k], ref[k]))

"""Edge cases of the fused step vs the oracle (layer counts, mesh sizes that leave partial thread
blocks and partial shared-memory tiles), and size-independent properties at the full C4 size
(1,000,000 columns x 50 layers, BASELINE.json config 4) where the oracle cannot run."""
from types import SimpleNamespace

import numpy as np
import pytest

from oracle import ext2d as OE
from oracle import geom as OG
from oracle import stepper as OS

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300))


def setup(pdg, nx, ny, L, seed=7):
    lx, ly = 1.3e4, 9e3

    def bed(x, y):
        return -18.0 + 4.0 * np.sin(np.pi * x / lx) * np.cos(2 * np.pi * y / ly)
    m = pdg.mesh.hilbert_reorder(pdg.mesh.generate_basin_mesh(nx, ny, lx, ly, bed))
    om = OG.hilbert_reorder(OG.basin_mesh(nx, ny, lx, ly, bed))
    rng = np.random.default_rng(seed)
    nt, P = m.nt, m.nt * L
    s0 = dict(eta=0.1 * np.cos(np.pi * m.x / lx) + 0.01 * rng.standard_normal((nt, 3)),
              qx=0.3 * rng.standard_normal((nt, 3)), qy=0.3 * rng.standard_normal((nt, 3)),
              ux=0.05 * rng.standard_normal((P, 6)), uy=0.05 * rng.standard_normal((P, 6)),
              T=np.where(np.repeat(m.x.mean(1), L)[:, None] * np.ones((1, 6)) < lx / 2, 15.0, 10.0))
    p = pdg.PhysParams(f=1e-4, cd=2.5e-3, alpha=0.2, t_ref=12.5, tau_x=0.05, tau_y=-0.02)
    return m, om, p, s0


def oracle_steps(om, L, p, s0, n, dt, msub, kv, nu_v):
    s = SimpleNamespace(grid=OG.extrude(om, L, s0["eta"]), ux=s0["ux"], uy=s0["uy"], T=s0["T"],
                        s2d=OE.S2(s0["eta"].copy(), s0["qx"], s0["qy"], 0.0))
    for _ in range(n):
        s = OS.imex_step(s, p, dt, msub, kv, nu_v)
    return s


@pytest.fixture(scope="module")
def pdg():
    import paper_2605_16082_b200 as p
    return p


@pytest.mark.parametrize("nx,ny,L", [
    (6, 4, 1),      # a single layer: surface and bed faces of the same prism, no interior faces
    (6, 4, 2),      # one interior horizontal face per column
    (7, 5, 7),      # 70 columns: one partial block / tile
    (13, 11, 3),    # 286 columns: two full 128-column tiles and a partial one
])
def test_step_edge_cases_vs_oracle(pdg, nx, ny, L):
    dt, msub, kv, nu_v = 30.0, 4, 1e-3, 1e-4
    m, om, p, s0 = setup(pdg, nx, ny, L)
    st = pdg.stepper.ImexStepper(m, L, p, dt, msub, kv, nu_v)
    st.set_state(**s0)
    st.step(3)
    st.check()
    g = st.get_state()
    o = oracle_steps(om, L, p, s0, 3, dt, msub, kv, nu_v)
    for k, ref in [("ux", o.ux), ("uy", o.uy), ("T", o.T), ("eta", o.s2d.eta), ("qx", o.s2d.qx), ("qy", o.s2d.qy)]:
        assert rel(g[k], ref) <= 1e-11, (nx, ny, L, k, rel(g[k], ref))


@pytest.fixture(scope="module")
def c4():
    import torch

    from paper_2605_16082_b200 import stepper
    from paper_2605_16082_b200.scenarios import device_state_c4, make_case
    c = make_case("c4", with_state=False)
    st = stepper.ImexStepper(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v)
    device_state_c4(c, st)
    yield c, st
    del st
    torch.cuda.empty_cache()


def test_full_size_c4_properties(c4):
    """C4 at full size: the closed basin conserves volume to rounding, a uniform tracer stays
    uniform under the moving-mesh step (consistency of q-bar with Q-bar), every field stays finite."""
    import torch
    c, st = c4
    T = st.T[st.cur]
    T.fill_(12.5)
    j2d = torch.as_tensor(np.asarray(c.mesh.j2d), device=st.dev)

    def volume():
        eta = st.S[0]                                   # [3][nt]
        return float((j2d * eta.sum(0)).sum().item()), float((j2d * eta.abs().sum(0)).sum().item())
    v0, a0 = volume()
    st.step(2)
    st.check()
    v1, _ = volume()
    assert abs(v1 - v0) <= 1e-12 * a0, (v0, v1)
    T = st.T[st.cur]
    assert float((T - 12.5).abs().max().item()) <= 1e-10 * 12.5
    for f in (st.U[st.cur], st.S):
        assert bool(torch.isfinite(f).all().item())


def test_layer_count_beyond_32bit_planes_rejected(pdg):
    """Per-layer addresses are 32-bit plane indices (csrc/col3d.cuh pix): a layer count that would
    make one field array reach 2^32 words is refused with ShapeMismatch, before any allocation."""
    m = pdg.mesh.hilbert_reorder(pdg.mesh.generate_basin_mesh(8, 8, 1e4, 1e4, lambda x, y: -20.0 + 0.0 * x))
    dm = pdg.device.DeviceMesh(m)
    L = (1 << 32) // (6 * m.nt) + 1
    with pytest.raises(pdg.errors.ShapeMismatch):
        dm.set_layers(L)
    dm.set_layers(50)          # the context stays usable
    assert dm.L == 50

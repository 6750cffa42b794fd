"""Host I/O layout kernels (csrc/hostio.cu) and the chunked set_state / get_state pipeline."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ncols,L,nk,nt,c0", [(37, 5, 6, 50, 7), (64, 8, 6, 64, 0), (1, 1, 3, 9, 8), (100, 50, 6, 130, 30),
                                             (33, 13, 2, 40, 0)])
def test_rows_planes_roundtrip(ncols, L, nk, nt, c0):
    import torch
    from paper_2605_16082_b200 import _lib
    from paper_2605_16082_b200.device import ptr, stream_ptr
    lb = _lib.lib()
    g = torch.Generator(device="cuda").manual_seed(1)
    rows = torch.randn(ncols * L, nk, generator=g, device="cuda", dtype=torch.float64)
    planes = torch.full((nk, L, nt), -7.0, device="cuda", dtype=torch.float64)
    _lib.check(lb.pdg_rows_to_planes(ptr(rows), ncols, L, nk, ptr(planes), nt, c0, stream_ptr()))
    ref = rows.reshape(ncols, L, nk).permute(2, 1, 0)
    assert torch.equal(planes[:, :, c0:c0 + ncols], ref)
    assert (planes[:, :, :c0] == -7.0).all() and (planes[:, :, c0 + ncols:] == -7.0).all()
    back = torch.zeros_like(rows)
    _lib.check(lb.pdg_planes_to_rows(ptr(planes), nt, c0, ncols, L, nk, ptr(back), stream_ptr()))
    assert torch.equal(back, rows)


def test_chunked_pipeline_many_chunks():
    """Tiny chunks and 4 staging slots: every slot is reused many times; the round trip through the
    same pinned buffers stays bitwise equal to the device-resident run."""
    import torch
    import paper_2605_16082_b200 as pdg
    m = pdg.mesh.hilbert_reorder(pdg.mesh.generate_basin_mesh(9, 5, 9e3, 5e3, lambda x, y: -20.0 + 0.0 * x))
    L = 7
    rng = np.random.default_rng(3)
    nt, P = m.nt, m.nt * L
    s0 = dict(eta=0.01 * rng.standard_normal((nt, 3)), qx=0.1 * rng.standard_normal((nt, 3)),
              qy=0.1 * rng.standard_normal((nt, 3)), ux=0.05 * rng.standard_normal((P, 6)),
              uy=0.05 * rng.standard_normal((P, 6)), T=12.0 + rng.standard_normal((P, 6)))
    p = pdg.PhysParams(f=1e-4, alpha=0.2, t_ref=12.0)
    ref = pdg.stepper.ImexStepper(m, L, p, 20.0, 4, 1e-3, 1e-4)
    ref.set_state(**s0)
    ref.step(3)
    g = ref.get_state()
    st = pdg.stepper.ImexStepper(m, L, p, 20.0, 4, 1e-3, 1e-4)
    st.IO_CHUNK_BYTES = 8 * 6 * L * 4          # 4 columns per prism chunk
    pin = {k: torch.as_tensor(v).pin_memory() for k, v in s0.items()}
    st.set_state(pin["eta"], pin["qx"], pin["qy"], pin["ux"], pin["uy"], pin["T"])
    for _ in range(3):
        st.step(1)
        st.get_state(numpy=False, out=pin)
        st.set_state(pin["eta"], pin["qx"], pin["qy"], pin["ux"], pin["uy"], pin["T"])
    st.wait_io()
    torch.cuda.synchronize()
    for k in ("eta", "qx", "qy", "ux", "uy", "T"):
        assert np.array_equal(pin[k].numpy(), g[k]), k
    # device inputs in the reference layout go through the same kernels
    st2 = pdg.stepper.ImexStepper(m, L, p, 20.0, 4, 1e-3, 1e-4)
    st2.set_state(**{k: torch.as_tensor(v, device="cuda") for k, v in s0.items()})
    st2.step(3)
    g2 = st2.get_state()
    for k in ("eta", "ux", "T"):
        assert np.array_equal(g2[k], g[k]), k

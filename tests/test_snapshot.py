"""PRISMDG-SNAP 1 snapshots: header, FieldSoA order, bit-exact round trip (CPU), and the
stepper state save / restore on the GPU."""
import numpy as np
import pytest

from paper_2605_16082_b200 import snapshot as SN


def test_roundtrip_bitexact(tmp_path):
    rng = np.random.default_rng(5)
    a = rng.standard_normal((2, 6, 7, 4))
    a[0, 0, 0, 0] = np.nextafter(1.0, 2.0)          # last-bit values survive
    a[1, 5, 6, 3] = -0.0
    SN.write(tmp_path / "u.snap", "u", a, 4, t=12.5)
    meta, b = SN.read(tmp_path / "u.snap")
    assert meta == {"field": "u", "components": 2, "columns": 7, "layers": 4, "time": 12.5}
    assert b.tobytes() == a.tobytes()
    head = (tmp_path / "u.snap").read_bytes().split(b"\n", 1)[0]
    assert head == b"PRISMDG-SNAP 1 u 2 7 4 12.5"
    # FieldSoA order (layout.py:50-51): address(f, k, c, l) = (f * 6 + k) * P + c * L + l
    flat = np.frombuffer((tmp_path / "u.snap").read_bytes().split(b"\n", 1)[1], "<f8")
    P = 7 * 4
    assert flat[(1 * 6 + 2) * P + 3 * 4 + 1] == a[1, 2, 3, 1]


def test_2d_and_errors(tmp_path):
    s = np.arange(3 * 3 * 5, dtype=float).reshape(3, 3, 5)
    SN.write(tmp_path / "s.snap", "eta_qx_qy", s, 0)
    meta, b = SN.read(tmp_path / "s.snap")
    assert meta["layers"] == 0 and np.array_equal(b, s)
    with pytest.raises(ValueError):
        SN.write(tmp_path / "x.snap", "bad name", s, 0)
    with pytest.raises(ValueError):
        SN.write(tmp_path / "x.snap", "u", s, 2)                  # shape / layers mismatch
    raw = (tmp_path / "s.snap").read_bytes()
    (tmp_path / "t.snap").write_bytes(raw[:-8])                 # truncated payload
    with pytest.raises(ValueError):
        SN.read(tmp_path / "t.snap")
    (tmp_path / "m.snap").write_bytes(b"PRISMDG-MESH 1\n")
    with pytest.raises(ValueError):
        SN.read(tmp_path / "m.snap")


@pytest.mark.gpu
def test_stepper_state_roundtrip(tmp_path):
    import paper_2605_16082_b200 as pdg
    from paper_2605_16082_b200.scenarios import make_case
    c = make_case("c4", scale=0.02, L=6)
    st = pdg.stepper.ImexStepper(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v)
    st.set_state(**c.state)
    st.step(2)
    ref = st.get_state()
    SN.save_state(st, str(tmp_path / "run"))
    st2 = pdg.stepper.ImexStepper(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v)
    SN.load_state(st2, str(tmp_path / "run"))
    got = st2.get_state()
    for k in ("eta", "qx", "qy", "ux", "uy", "T"):
        assert np.array_equal(got[k], ref[k]), k
    assert got["t"] == ref["t"]
    st.step(1)
    st2.step(1)                                     # a restored run continues bitwise identically
    a, b = st.get_state(), st2.get_state()
    for k in ("eta", "ux", "T"):
        assert np.array_equal(a[k], b[k]), k

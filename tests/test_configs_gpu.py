"""BASELINE configs at their stated sizes vs the REAL reference (tests/golden/cfg_*.npz).

The fixtures come from scripts/make_golden_configs.py: the reference's own functions
(/root/reference/pkg/src/prismdg) composed by the shared orchestrator (oracle/stepper.py; the
reference ships no stepper), from the seeded parity-variant states of tests/config_states.py.
north_star gates: <= 1e-9 after 100 steps (per-step checks at 1e-11).

  C2   32x32 basin (2,048 tri) x 10 layers, dt 40 s, m 20, 100 steps
  C3   250x100 lock exchange (50,000 tri) x 20 layers (1 M prisms), dt 20 s, m 20: one full
       step, compared on 2,048 sampled columns
  C3w  20x8 window of the C3 basin at the same resolution x 20 layers, 100 steps
"""
import numpy as np
import pytest

import config_states as CS

pytestmark = pytest.mark.gpu


def rel(a, b):
    """normwise relative L-inf error, recorded per test (conftest.record)."""
    import os
    from conftest import record
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    e = float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))
    return record(os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0], e)


def _stepper(cfg, state_fn):
    import paper_2605_16082_b200 as pdg
    mesh = pdg.mesh.hilbert_reorder(pdg.mesh.generate_basin_mesh(cfg["nx"], cfg["ny"], cfg["lx"], cfg["ly"],
                                                                  CS.flat_bed))
    L = cfg["L"]
    s0 = state_fn(mesh, L)
    st = pdg.stepper.ImexStepper(mesh, L, pdg.PhysParams(**cfg["params"]), cfg["dt"], cfg["m"], cfg["kv"],
                                 cfg["nu_v"])
    st.set_state(**s0)
    return st, s0, mesh


def _check_inputs(g, s0):
    ins = np.array([float(np.sum(np.abs(s0[k]))) for k in ("eta", "qx", "qy", "ux", "uy", "T")])
    assert np.array_equal(ins, g["in_sum"]), "seeded inputs differ from the fixture's"


def _run(golden, name, cfg, state_fn, tol_last):
    g = golden(f"cfg_{name}")
    st, s0, mesh = _stepper(cfg, state_fn)
    _check_inputs(g, s0)
    done = 0
    for k in sorted(int(n[1:].split("_")[0]) for n in g if n.startswith("s") and n.endswith("_ux")):
        st.step(k - done)
        done = k
        st.check()
        s = st.get_state()
        tol = tol_last if k > 1 else 1e-11
        for n in ("ux", "uy", "T", "eta", "qx", "qy"):
            assert rel(s[n], g[f"s{k}_{n}"]) <= tol, (name, k, n, rel(s[n], g[f"s{k}_{n}"]))


def test_c2_100_steps(golden):
    _run(golden, "c2", CS.C2, CS.c2_state, 1e-9)


def test_c3_window_100_steps(golden):
    _run(golden, "c3w", CS.C3W, lambda m, L: CS.c3_state(m, L, CS.C3W["lx"]), 1e-9)


def test_c3_full_step_sampled(golden):
    g = golden("cfg_c3")
    cfg = CS.C3
    st, s0, mesh = _stepper(cfg, lambda m, L: CS.c3_state(m, L, cfg["lx"]))
    _check_inputs(g, s0)
    st.step(1)
    st.check()
    s = st.get_state()
    cols, L = g["cols"], cfg["L"]
    pr = (cols[:, None] * L + np.arange(L)[None, :]).ravel()
    for n in ("ux", "uy", "T"):
        assert rel(s[n][pr], g[f"s1_{n}"]) <= 1e-10, n
    for n in ("eta", "qx", "qy"):
        assert rel(s[n][cols], g[f"s1_{n}"]) <= 1e-10, n

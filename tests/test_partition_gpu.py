"""Partitioned stepping on one GPU (virtual ranks): bitwise equal to the unpartitioned run."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pdg():
    import paper_2605_16082_b200 as p
    return p


@pytest.mark.parametrize("P", [2, 3, 4, 7])
def test_partition_invariance_bitwise(pdg, P):
    from paper_2605_16082_b200.partition import PartitionedRun
    from paper_2605_16082_b200.scenarios import make_case
    c = make_case("c4", scale=0.02, L=6)                   # 20 x 10 squares of the coastal basin
    ref = pdg.stepper.ImexStepper(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v)
    ref.use_graph = False
    ref.set_state(**c.state)
    ref.step(3)
    ref.check()
    g = ref.get_state()
    run = PartitionedRun(c.mesh, c.L, c.params, c.dt, c.m, c.kv, c.nu_v, P)
    run.set_state(**c.state)
    run.step(3)
    run.check()
    s = run.get_state()
    for k in ("eta", "qx", "qy", "ux", "uy", "T"):
        assert np.array_equal(s[k], g[k]), (P, k, float(np.abs(s[k] - g[k]).max()))
    assert run.group.exchanges == 3 * (2 * 4 + (c.m // 2 + c.m))   # q, F3D->2D, mis, u/T per stage + 2D per substep

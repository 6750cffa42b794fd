"""Reference storage layouts (layout.py) and the cell-block column solves (columns.py:546-580)
against golden values from the real reference (scripts/make_golden_layout.py)."""
import numpy as np
import pytest

from paper_2605_16082_b200 import layout as LY


def test_layout_bitwise_vs_reference(golden):
    g = golden("layout")
    layers = g["layers"]
    offsets = np.concatenate([[0], np.cumsum(layers)])
    soa = LY.FieldSoA.from_native(g["native"], offsets)
    assert np.array_equal(soa.data, g["soa"])
    assert np.array_equal(soa.to_native(), g["native"])
    blocks = LY.soa_to_cell(soa, width=4)
    assert len(blocks) == int(g["ncells"])
    for i, b in enumerate(blocks):
        assert np.array_equal(b.data, g[f"cell{i}"])
        assert np.array_equal(b.columns, g[f"cell{i}_cols"])
        assert np.array_equal(b.lane_mask(), g[f"cell{i}_mask"])
    back = LY.cell_to_soa(blocks, offsets)
    assert np.array_equal(back.data, g["back"])
    v = LY.cell_view(blocks[0])                          # a view: writes land in the cell matrix
    v[0, 0, 0, 0] = 42.0
    assert blocks[0].data[0, 0] == 42.0
    assert soa.address(1, 2, 3, 1) == (1 * 6 + 2) * soa.n_prisms + offsets[3] + 1


def test_block_shape_table_vs_reference(golden):
    g = golden("layout")
    rows = LY.block_shape_table([1, 2, 3, 7, 10, 31, 50, 64, 100, 128, 200], width=128)
    got = np.array([[r["n"], r["read_chunk"], r["write_chunk"], r["layers"], r["utilization"]] for r in rows])
    assert np.array_equal(got, g["table"])
    with pytest.raises(Exception):
        LY.choose_block_shape(0)


@pytest.mark.gpu
def test_cell_solves_vs_reference(golden):
    from paper_2605_16082_b200 import columns
    g = golden("layout")
    layers = g["layers"]
    offsets = np.concatenate([[0], np.cumsum(layers)])
    blocks = LY.soa_to_cell(LY.FieldSoA.from_native(g["native"], offsets), width=4)
    j2d = g["j2d"]
    for i, b in enumerate(blocks):
        r = columns.solve_r_cell(b, j2d[b.columns])
        w = columns.solve_w_cell(b, j2d[b.columns])
        for got, ref in ((r.data, g[f"r{i}"]), (w.data, g[f"w{i}"])):
            assert np.abs(got - ref).max() <= 1e-12 * max(np.abs(ref).max(), 1.0)

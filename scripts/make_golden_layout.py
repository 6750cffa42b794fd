"""Generate tests/golden/layout.npz from the REAL reference package: FieldSoA / CellBlock
transpositions of a ragged field, the block-shape table and the cell-block column solves.

Run in the build container only (needs /root/reference):  python scripts/make_golden_layout.py
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "layout.npz")


def main():
    sys.path.insert(0, REF)
    from prismdg import columns as RC
    from prismdg import layout as RL

    rng = np.random.default_rng(77)
    layers = np.array([3, 5, 1, 4, 4, 2, 5, 3, 2, 1, 5])           # ragged columns
    offsets = np.concatenate([[0], np.cumsum(layers)])
    native = rng.standard_normal((int(offsets[-1]), 6, 2))
    soa = RL.FieldSoA.from_native(native, offsets)
    blocks = RL.soa_to_cell(soa, width=4)
    back = RL.cell_to_soa(blocks, offsets)
    j2d = 1.0 + rng.random(layers.size)
    r_cells = [RC.solve_r_cell(b, j2d[b.columns]) for b in blocks]
    w_cells = [RC.solve_w_cell(b, j2d[b.columns]) for b in blocks]
    table = RL.block_shape_table([1, 2, 3, 7, 10, 31, 50, 64, 100, 128, 200], width=128)
    tab = np.array([[r["n"], r["read_chunk"], r["write_chunk"], r["layers"], r["utilization"]] for r in table])
    out = dict(layers=layers, native=native, soa=soa.data, back=back.data, table=tab, j2d=j2d)
    for i, b in enumerate(blocks):
        out[f"cell{i}"] = b.data
        out[f"cell{i}_cols"] = b.columns
        out[f"cell{i}_mask"] = b.lane_mask()
        out[f"r{i}"] = r_cells[i].data
        out[f"w{i}"] = w_cells[i].data
    out["ncells"] = len(blocks)
    np.savez_compressed(OUT, **out)
    print(OUT, len(blocks), "cells")


if __name__ == "__main__":
    main()

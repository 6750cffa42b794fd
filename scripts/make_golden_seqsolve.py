"""Generate tests/golden/seqsolve.npz from the REAL reference: solve_banded_sequential
(columns.py:404-485) on one column of a seeded diagonally dominant banded system, with its
working-set record.  Run in the build container only:  python scripts/make_golden_seqsolve.py
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "seqsolve.npz")


def main():
    sys.path.insert(0, REF)
    from prismdg import columns as RC
    rng = np.random.default_rng(1)
    n, L = 3, 5
    d = rng.standard_normal((n, L, 6, 6)) + 8 * np.eye(6)
    u = 0.3 * rng.standard_normal((n, L, 3, 6))
    w = 0.3 * rng.standard_normal((n, L, 3, 6))
    rhs = rng.standard_normal((1, L, 6, 2))
    mat = RC.BandedColumnMatrix(d=d.copy(), u=u.copy(), w=w.copy())
    x, st = RC.solve_banded_sequential(mat, rhs, 1)
    np.savez_compressed(OUT, d=d, u=u, w=w, rhs=rhs, x=x, col=1, max_live=st.max_live, loads=st.loads,
                        stores=st.stores, touched=np.array(sorted(f"{k}{l}" for k, l in st.touched)))
    print(OUT, st.max_live, st.loads, st.stores, len(st.touched))


if __name__ == "__main__":
    main()

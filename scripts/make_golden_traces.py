"""Generate tests/golden/traces.npz from the REAL reference: trace_int / trace_ext / edge_celerity
(external2d.py:95-116) on a seeded state.  Run in the build container only:
    python scripts/make_golden_traces.py
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "traces.npz")


def main():
    sys.path.insert(0, REF)
    from prismdg import external2d as RE
    from prismdg import mesh as RM
    lx, ly = 1e4, 8e3
    mesh = RM.hilbert_reorder(RM.generate_basin_mesh(6, 4, lx, ly, lambda x, y: -20.0 + 0.0 * x))
    rng = np.random.default_rng(95)
    eta = 0.1 * rng.standard_normal((mesh.nt, 3))
    out = {"eta": eta, "b": mesh.b}
    els = np.arange(mesh.nt)
    for k in range(3):
        ti = RE.trace_int(eta, els, k)
        te = RE.trace_ext(eta, mesh.nbr[:, k], mesh.nbrk[:, k])
        bi = RE.trace_int(mesh.b, els, k)
        be = RE.trace_ext(mesh.b, mesh.nbr[:, k], mesh.nbrk[:, k])
        out[f"ti{k}"], out[f"te{k}"] = ti, te
        out[f"cel{k}"] = RE.edge_celerity(ti, te, bi, be, 9.81)
        out[f"nbr{k}"], out[f"nbrk{k}"] = mesh.nbr[:, k], mesh.nbrk[:, k]
    np.savez_compressed(OUT, **out)
    print(OUT)


if __name__ == "__main__":
    main()

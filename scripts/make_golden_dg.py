"""Generate tests/golden/dg.npz from the REAL reference: the dg.py tables and pointwise helpers
on seeded inputs.  Run in the build container only:  python scripts/make_golden_dg.py"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "dg.npz")


def main():
    sys.path.insert(0, REF)
    from prismdg import dg
    rng = np.random.default_rng(27)
    v = rng.standard_normal((5, 6))
    a, b, s = rng.standard_normal(7), rng.standard_normal(7), rng.standard_normal(7)
    s[0] = 0.0
    la, lb = 1.0 + rng.random(7), 1.0 + rng.random(7)
    dzm, dzj, jz, zeta = rng.standard_normal((7, 2)), rng.standard_normal((7, 2)), 0.5 + rng.random(7), \
        rng.uniform(-1, 1, 7)
    mh, mz = dg.metric_vector(dzm, dzj, jz, zeta)
    gx, fz = rng.standard_normal((7, 2)), rng.standard_normal(7)
    giso, gm = dg.gradient_decompose(gx, fz, mh, mz)
    u, w = rng.standard_normal((7, 2)), rng.standard_normal(7)
    ut, wt = dg.split_velocity(u, w, mh, mz)
    D = rng.standard_normal((7, 3, 3))
    D = D + np.swapaxes(D, 1, 2)
    sd = dg.split_diffusivity(D, mh, mz)
    out = dict(TRI_QW=dg.TRI_QW, TRI_BARY=dg.TRI_BARY, TRI_QP=dg.TRI_QP, SEG_QP=dg.SEG_QP, SEG_QW=dg.SEG_QW,
               VERT_SHAPE=dg.VERT_SHAPE, DVERT=dg.DVERT, EDGE_SHAPE=dg.EDGE_SHAPE, DPHI_PARENT=dg.DPHI_PARENT,
               v=v, tri_quad=dg.tri_quad(v), a=a, b=b, s=s, mean=dg.iface_mean(a, b), diff=dg.iface_diff(a, b),
               mx=dg.iface_max(a, b), up=dg.iface_upwind(a, b, s), la=la, lb=lb, pen=dg.penalty_sigma(la, lb),
               pen2=dg.penalty_sigma(la, lb, dim=2), dzm=dzm, dzj=dzj, jz=jz, zeta=zeta, mh=mh, mz=mz, gx=gx, fz=fz,
               giso=giso, gm=gm, u=u, w=w, ut=ut, wt=wt, D=D, kappa_i=sd.kappa_i, d_e=sd.d_e,
               kimp=dg.kappa_implicit(2.0, 1e-3, mh, mz))
    np.savez_compressed(OUT, **out)
    print(OUT)


if __name__ == "__main__":
    main()

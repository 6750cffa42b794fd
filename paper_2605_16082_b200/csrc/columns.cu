// Column-local vertical operators and solvers (columns.py, internal3d.py:800-906).
//
// One thread per column, layers in registers.  The banded system M - dt A is never stored in
// the fused path: each layer's 6x6 diagonal block and 3x6 couplings are assembled in registers
// from (w~, w_m, sigma geometry) and consumed immediately by the block-Thomas elimination; only
// the 6x6 propagation tile G_l and the reduced RHS g_l are kept for the back substitution.
#include "col3d.cuh"
#include "ctx.cuh"

namespace pdg {

// ============================================================================ sweeps (API)
// columns.py:95-151.  rhs/out: [nc][6][L][ncol]; layers (optional) = active layer count
__global__ void k_sweep(int kind, int ncol, int L, int nc, const double* __restrict__ rhs,
                        const double* __restrict__ j2d, const int* __restrict__ layers, double* __restrict__ out,
                        pdg_err* err) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncol) return;
  const double j = j2d[c];
  if (j <= 0.0) report(err, PDG_ERR_SINGULAR_MASS, c, 0, j);
  const int act = layers ? layers[c] : L;
  for (int cc = 0; cc < nc; ++cc) {
    const double* f = rhs + (size_t)cc * 6 * L * ncol;
    double* o = out + (size_t)cc * 6 * L * ncol;
    double s[3] = {0, 0, 0};
    for (int it = 0; it < L; ++it) {
      const int l = kind == 0 ? it : L - 1 - it;
      double v[6], gt[3], gb[3], r[6];
      ld6(f, l, c, L, ncol, v);
      mh_inv3(v, j, gt);
      mh_inv3(v + 3, j, gb);
      const bool on = l < act;
      if (kind == 0) {  // top-down (surface anchored)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          if (on) s[a] = s[a] + (gt[a] + gb[a]);
          r[a] = on ? -s[a] + 2.0 * gb[a] : 0.0;
          r[3 + a] = on ? -s[a] : 0.0;
        }
      } else {  // bottom-up (bed anchored)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const double wb = s[a] + gb[a] - gt[a], wt = s[a] + gb[a] + gt[a];
          r[3 + a] = on ? wb : 0.0;
          r[a] = on ? wt : 0.0;
          if (on) s[a] = wt;
        }
      }
      st6(o, l, c, L, ncol, r);
    }
  }
}

// ============================================================================ generic banded (API)
__device__ __forceinline__ size_t bidx(int e, int l, int c, int L, int ncol) { return ((size_t)e * L + l) * ncol + c; }

// solve_banded_column (columns.py:292-348).  G tiles are written into gu/gw (rows 0-2 / 3-5),
// which may alias the caller's u/w (overwrite=True semantics) or scratch copies.
template <int NC>
__global__ void __launch_bounds__(128) k_banded_solve(int ncol, int L, const double* __restrict__ d,
                                                      const double* u, const double* w, double* gu, double* gw,
                                                      const double* __restrict__ rhs, double* __restrict__ x,
                                                      pdg_err* err) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncol) return;
  const size_t P6 = (size_t)6 * L * ncol;
  double gp[6][NC];
  for (int l = 0; l < L; ++l) {
    double a[6][6], g[6][NC];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
#pragma unroll
      for (int j = 0; j < 6; ++j) a[i][j] = d[bidx(i * 6 + j, l, c, L, ncol)];
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) g[i][cc] = rhs[cc * P6 + bidx(i, l, c, L, ncol)];
    }
    if (l > 0) {
      double U[3][6];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 6; ++k) U[i][k] = u[bidx(i * 6 + k, l, c, L, ncol)];
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        double G[6];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          G[k] = gu[bidx(k * 6 + j, l - 1, c, L, ncol)];
          G[3 + k] = gw[bidx(k * 6 + j, l - 1, c, L, ncol)];
        }
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < 6; ++k) acc = acc + U[i][k] * G[k];
          a[i][j] = a[i][j] - acc;
        }
      }
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) {
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < 6; ++k) acc = acc + U[i][k] * gp[k][cc];
          g[i][cc] = g[i][cc] - acc;
        }
    }
    const int bad = lu6(a);
    if (bad >= 0) {
      report(err, PDG_ERR_ZERO_PIVOT, l, bad, 0.0);
      return;
    }
    if (l < L - 1) {
      double t[6][6];
#pragma unroll
      for (int j = 0; j < 6; ++j) {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          t[i][j] = 0.0;
          t[3 + i][j] = w[bidx(i * 6 + j, l, c, L, ncol)];
        }
      }
      lu6_solve<6>(a, t);
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 6; ++j) {
          gu[bidx(i * 6 + j, l, c, L, ncol)] = t[i][j];
          gw[bidx(i * 6 + j, l, c, L, ncol)] = t[3 + i][j];
        }
    }
    lu6_solve<NC>(a, g);
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        x[cc * P6 + bidx(i, l, c, L, ncol)] = g[i][cc];
        gp[i][cc] = g[i][cc];
      }
  }
  // back substitution x_l = g_l - G_l x_{l+1}  (x holds g on entry)
  double xn[6][NC];
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) xn[i][cc] = gp[i][cc];
  for (int l = L - 2; l >= 0; --l) {
    double xl[6][NC];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      double G[6];
#pragma unroll
      for (int k = 0; k < 6; ++k)
        G[k] = i < 3 ? gu[bidx(i * 6 + k, l, c, L, ncol)] : gw[bidx((i - 3) * 6 + k, l, c, L, ncol)];
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < 6; ++k) acc = acc + G[k] * xn[k][cc];
        xl[i][cc] = x[cc * P6 + bidx(i, l, c, L, ncol)] - acc;
      }
    }
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        x[cc * P6 + bidx(i, l, c, L, ncol)] = xl[i][cc];
        xn[i][cc] = xl[i][cc];
      }
  }
}

// apply_banded (columns.py:356-366)
__global__ void k_banded_apply(int ncol, int L, int nc, const double* __restrict__ d, const double* __restrict__ u,
                               const double* __restrict__ w, const double* __restrict__ xin, double* __restrict__ y) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncol) return;
  const size_t P6 = (size_t)6 * L * ncol;
  for (int cc = 0; cc < nc; ++cc) {
    const double* xc = xin + cc * P6;
    for (int l = 0; l < L; ++l) {
      double xl[6], out[6];
      ld6(xc, l, c, L, ncol, xl);
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        double t = 0.0;
#pragma unroll
        for (int j = 0; j < 6; ++j) t += d[bidx(i * 6 + j, l, c, L, ncol)] * xl[j];
        out[i] = t;
      }
      if (l > 0) {
        double xa[6];
        ld6(xc, l - 1, c, L, ncol, xa);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          double t = 0.0;
#pragma unroll
          for (int j = 0; j < 6; ++j) t += u[bidx(i * 6 + j, l, c, L, ncol)] * xa[j];
          out[i] += t;
        }
      }
      if (l < L - 1) {
        double xb[6];
        ld6(xc, l + 1, c, L, ncol, xb);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          double t = 0.0;
#pragma unroll
          for (int j = 0; j < 6; ++j) t += w[bidx(i * 6 + j, l, c, L, ncol)] * xb[j];
          out[3 + i] += t;
        }
      }
      st6(y + cc * P6, l, c, L, ncol, out);
    }
  }
}

// build_implicit (internal3d.py:902-906): (M - dt A) elementwise
__global__ void k_build_implicit(long long P, const double* __restrict__ mass, const double* __restrict__ d,
                                 const double* __restrict__ u, const double* __restrict__ w, double dt,
                                 double* __restrict__ od, double* __restrict__ ou, double* __restrict__ ow) {
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= P) return;
#pragma unroll
  for (int e = 0; e < 36; ++e) od[e * P + p] = mass[e * P + p] - dt * d[e * P + p];
#pragma unroll
  for (int e = 0; e < 18; ++e) {
    ou[e * P + p] = -dt * u[e * P + p];
    ow[e * P + p] = -dt * w[e * P + p];
  }
}

// mass_apply / mass_solve (internal3d.py:126-151) with explicit (P,6,6) masses
__global__ void k_mass_op(long long P, int L, int nt, int nc, int solve, const double* __restrict__ mass,
                          const double* __restrict__ f, double* __restrict__ out, pdg_err* err) {
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= P) return;
  double a[6][6];
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = 0; j < 6; ++j) a[i][j] = mass[(i * 6 + j) * P + p];
  if (solve) {
    const int bad = lu6(a);
    if (bad >= 0) {
      report(err, PDG_ERR_ZERO_PIVOT, (long long)(p / nt), bad, 0.0);
      return;
    }
  }
  for (int cc = 0; cc < nc; ++cc) {
    double v[6][1], o[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) v[i][0] = f[(cc * 6 + i) * P + p];
    if (solve) {
      lu6_solve<1>(a, v);
#pragma unroll
      for (int i = 0; i < 6; ++i) o[i] = v[i][0];
    } else {
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        double t = 0.0;
#pragma unroll
        for (int j = 0; j < 6; ++j) t += a[i][j] * v[j][0];
        o[i] = t;
      }
    }
#pragma unroll
    for (int i = 0; i < 6; ++i) out[(cc * 6 + i) * P + p] = o[i];
  }
}

// batched scalar Thomas (columns.py:507-531); arrays [n][nb] (batch contiguous)
__global__ void k_tridiag(int nb, int n, const double* __restrict__ lo, const double* __restrict__ di,
                          const double* __restrict__ up, const double* __restrict__ rhs, double* __restrict__ x,
                          double* __restrict__ work, pdg_err* err) {
  const int bI = blockIdx.x * blockDim.x + threadIdx.x;
  if (bI >= nb) return;
  // work holds the modified diagonal; x holds the modified rhs
  double bprev = di[bI], dprev = rhs[bI];
  work[bI] = bprev;
  x[bI] = dprev;
  for (int i = 1; i < n; ++i) {
    if (bprev == 0.0) {
      report(err, PDG_ERR_ZERO_PIVOT, i - 1, 0, 0.0);
      return;
    }
    const double m = lo[(size_t)i * nb + bI] / bprev;
    const double bi = di[(size_t)i * nb + bI] - m * up[(size_t)(i - 1) * nb + bI];
    const double dd = rhs[(size_t)i * nb + bI] - m * dprev;
    work[(size_t)i * nb + bI] = bi;
    x[(size_t)i * nb + bI] = dd;
    bprev = bi;
    dprev = dd;
  }
  if (bprev == 0.0) {
    report(err, PDG_ERR_ZERO_PIVOT, n - 1, 0, 0.0);
    return;
  }
  double xn = dprev / bprev;
  x[(size_t)(n - 1) * nb + bI] = xn;
  for (int i = n - 2; i >= 0; --i) {
    xn = (x[(size_t)i * nb + bI] - up[(size_t)i * nb + bI] * xn) / work[(size_t)i * nb + bI];
    x[(size_t)i * nb + bI] = xn;
  }
}

// ============================================================================ vertical operator
// per-layer geometry factors of assemble_vertical_operator (internal3d.py:825, 838, 875-891)
struct VG {
  double jzq[6];
  double kis;      // ki[0] + ki[1]  (kv + kh |m_h/m_z|^2 at the two vertical points)
  double kt, kb;   // kv + kh |grad z_top|^2, kv + kh |grad z_bot|^2
  double hgt;      // 2 mean(Jz)
  double nz;       // 1/sqrt(1 + |grad z_top|^2)
};

__device__ __forceinline__ void vgeo(const Col& C, const double eta[3], double ft, double fb, double kh, double kv,
                                     VG& V) {
  LGeo G;
  layer_geo(C, eta, ft, fb, G);
  hq(G.jz, V.jzq);
  double ks = 0.0;
#pragma unroll
  for (int vv = 0; vv < 2; ++vv) {
    const double mx = G.dzmid[0] + ZQP[vv] * G.djz[0], my = G.dzmid[1] + ZQP[vv] * G.djz[1];
    ks += kv + kh * (mx * mx + my * my);
  }
  V.kis = ks;
  const double tt = G.dztop[0] * G.dztop[0] + G.dztop[1] * G.dztop[1];
  V.kt = kv + kh * tt;
  V.kb = kv + kh * (G.dzbot[0] * G.dzbot[0] + G.dzbot[1] * G.dzbot[1]);
  V.hgt = 2.0 * (((G.jz[0] + G.jz[1]) + G.jz[2]) / 3.0);
  V.nz = 1.0 / sqrt(1.0 + tt);
}

__device__ __forceinline__ double pen_sigma(double la, double lb, double n0, int order, pdg_err* err) {
  const double lmin = fmin(la, lb);
  if (lmin <= 0.0) report(err, PDG_ERR_NONPOS_LENGTH, 0, 0, lmin);
  return n0 * (order + 1.0) * (order + 3.0) / (2.0 * 3.0 * lmin);
}

// layer l of A: d (6x6), u (3x6, coupling to layer l-1), w (3x6, coupling to layer l+1).
// dw = w~ - w_m on the 6 nodes of layer l; wtn = w~ top nodes of layer l+1; wmb = w_m bottom of l.
__device__ __forceinline__ void vop_layer(double j2d, int l, int L, const VG& Vp, const VG& V, const VG& Vn,
                                          const double dw[6], const double wt_top[3], const double wm[6],
                                          const double wtn[3], double n0, int order, pdg_err* err, double d[6][6],
                                          double u[3][6], double w[3][6]) {
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = 0; j < 6; ++j) d[i][j] = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      u[i][j] = 0.0;
      w[i][j] = 0.0;
    }
  double dt3[6], db3[6];
  hq(dw, dt3);
  hq(dw + 3, db3);
  // advective volume + implicit diffusion volume (internal3d.py:832-841)
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    double A[2];
#pragma unroll
    for (int lj = 0; lj < 2; ++lj) {
      double s = 0.0;
#pragma unroll
      for (int vv = 0; vv < 2; ++vv) {
        const double spd = VS[vv][0] * dt3[q] + VS[vv][1] * db3[q];
        s += QW[q] * (j2d * spd) * VS[vv][lj];
      }
      A[lj] = s;
    }
    const double kd = QW[q] * V.kis * (j2d / V.jzq[q]);
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        const double bb = BARY[q][i % 3] * BARY[q][j % 3];
        d[i][j] += DV[i / 3] * bb * A[j / 3] - kd * DV[i / 3] * DV[j / 3] * bb;
      }
  }
  // advective interface fluxes (internal3d.py:843-870)
  double wtt[6], wmt[6];
  hq(wt_top, wtt);
  hq(wm, wmt);
  if (l == 0 || true) {
    // top face: surface keeps the interior trace; interior faces split by sign
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const double sp = wtt[q] - wmt[q];
      const double pos = l == 0 ? sp : (sp >= 0.0 ? sp : 0.0);
      const double neg = l == 0 ? 0.0 : (sp < 0.0 ? sp : 0.0);
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const double bb = QW[q] * BARY[q][i] * BARY[q][j];
          d[i][j] -= bb * (j2d * pos);
          u[i][3 + j] -= bb * (j2d * neg);
        }
    }
  }
  if (l < L - 1) {
    double wnt[6], wmb[6];
    hq(wtn, wnt);
    hq(wm + 3, wmb);
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const double sb = wnt[q] - wmb[q];
      const double into = sb <= 0.0 ? sb : 0.0, outof = sb > 0.0 ? sb : 0.0;
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const double bb = QW[q] * BARY[q][i] * BARY[q][j];
          d[3 + i][3 + j] += bb * (j2d * into);
          w[i][j] += bb * (j2d * outof);
        }
    }
  }
  // diffusive mean flux and interior penalty on interior horizontal faces (internal3d.py:873-897)
  double mf[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < 6; ++q) s += QW[q] * BARY[q][i] * BARY[q][j];
      mf[i][j] = s;
    }
  if (l > 0) {
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const double hi = 0.5 * j2d * V.kt / V.jzq[q];
      const double he = 0.5 * j2d * Vp.kb / Vp.jzq[q];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 6; ++j) {
          const double bd = QW[q] * BARY[q][i] * (DV[j / 3] * BARY[q][j % 3]);
          d[i][j] += hi * bd;
          u[i][j] += he * bd;
        }
    }
    const double pf = pen_sigma(V.hgt, Vp.hgt, n0, order, err) * fmax(V.kt, Vp.kb) * V.nz * j2d;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        d[i][j] -= 0.5 * pf * mf[i][j];
        u[i][3 + j] += 0.5 * pf * mf[i][j];
      }
  }
  if (l < L - 1) {
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const double he = 0.5 * j2d * V.kb / V.jzq[q];
      const double hi = 0.5 * j2d * Vn.kt / Vn.jzq[q];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 6; ++j) {
          const double bd = QW[q] * BARY[q][i] * (DV[j / 3] * BARY[q][j % 3]);
          d[3 + i][j] -= he * bd;
          w[i][j] -= hi * bd;
        }
    }
    const double pf = pen_sigma(Vn.hgt, V.hgt, n0, order, err) * fmax(Vn.kt, V.kb) * Vn.nz * j2d;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        d[3 + i][3 + j] -= 0.5 * pf * mf[i][j];
        w[i][j] += 0.5 * pf * mf[i][j];
      }
  }
}

struct VopArgs {
  const double* eta_u;  // grid the operator is assembled on (C3)
  const double* wt;     // w~ (P6)
  const double* wm;     // w_m (P6) when given explicitly (API); else from eta0/eta1
  const double* eta0;   // fused: mesh velocity (z(eta1) - z(eta0)) / dtm
  const double* eta1;   //        and M1 = mass(eta1)
  double dtm;
  double kh, kv, n0;
  int order;
};

// node values of w_m at layer l
__device__ __forceinline__ void wm_layer(const VopArgs& a, const double b[3], const double e0[3], const double e1[3],
                                         double ft, double fb, int l, int c, int L, int nt, double wm[6]) {
  if (a.wm) {
    ld6(a.wm, l, c, L, nt, wm);
    return;
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double H0 = __dsub_rn(e0[i], b[i]), H1 = __dsub_rn(e1[i], b[i]);
    const double zt0 = __dsub_rn(e0[i], __dmul_rn(ft, H0)), zt1 = __dsub_rn(e1[i], __dmul_rn(ft, H1));
    const double zb0 = __dsub_rn(e0[i], __dmul_rn(fb, H0)), zb1 = __dsub_rn(e1[i], __dmul_rn(fb, H1));
    wm[i] = (zt1 - zt0) / a.dtm;
    wm[3 + i] = (zb1 - zb0) / a.dtm;
  }
}

// assemble_vertical_operator (API): writes d [36][L][nt], u/w [18][L][nt]
__global__ void __launch_bounds__(128) k_vop(DMesh m, VopArgs a, const int* __restrict__ els, int n,
                                             double* __restrict__ od, double* __restrict__ ou,
                                             double* __restrict__ ow) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = els ? els[i] : i, nt = m.nt, L = m.L;
  Col C;
  load_col(m, c, C);
  double eta[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) eta[k] = a.eta_u[k * nt + c];
  // output rows are compact over the selected columns (reference returns (n_els, L, ...))
  VG Vp, V, Vn;
  vgeo(C, eta, m.fracs[0], m.fracs[1], a.kh, a.kv, V);
  Vp = V;
  for (int l = 0; l < L; ++l) {
    if (l < L - 1) vgeo(C, eta, m.fracs[l + 1], m.fracs[l + 2], a.kh, a.kv, Vn);
    double wt[6], wm[6], wtn[3] = {0, 0, 0}, dw[6];
    ld6(a.wt, l, c, L, nt, wt);
    wm_layer(a, C.b, nullptr, nullptr, 0, 0, l, c, L, nt, wm);
    if (l < L - 1) {
#pragma unroll
      for (int k = 0; k < 3; ++k) wtn[k] = a.wt[((size_t)k * L + l + 1) * nt + c];
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) dw[k] = wt[k] - wm[k];
    double d[6][6], u[3][6], w[3][6];
    vop_layer(C.j2d, l, L, Vp, V, Vn, dw, wt, wm, wtn, a.n0, a.order, m.err, d, u, w);
#pragma unroll
    for (int r = 0; r < 6; ++r)
#pragma unroll
      for (int s = 0; s < 6; ++s) od[((size_t)(r * 6 + s) * L + l) * n + i] = d[r][s];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        ou[((size_t)(r * 6 + s) * L + l) * n + i] = u[r][s];
        ow[((size_t)(r * 6 + s) * L + l) * n + i] = w[r][s];
      }
    Vp = V;
    V = Vn;
  }
}

// ============================================================================ fused vertical step
// IMPLICIT: x = (M1 - dt A)^-1 rhs by block Thomas with A assembled per layer in registers.
// EXPLICIT: x = M1^-1 (rhs + dt A xin)  (internal3d.py:902-906 + columns.py:292-366 + :134-151).
// Scratch: G tiles [36][L][nt] (implicit only).
template <int NC, bool IMPLICIT>
__global__ void __launch_bounds__(128) k_vstep(DMesh m, VopArgs a, double dt, const double* __restrict__ rhs,
                                               const double* __restrict__ xin, double* __restrict__ Gs,
                                               double* __restrict__ x) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int nt = m.nt, L = m.L;
  if (c >= nt) return;
  const size_t P6 = (size_t)6 * L * nt;
  Col C;
  load_col(m, c, C);
  double eta[3], e0[3], e1[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    eta[k] = a.eta_u[k * nt + c];
    e0[k] = a.eta0[k * nt + c];
    e1[k] = a.eta1[k * nt + c];
  }
  const double j2d = C.j2d;
  const double K00 = VS[0][0] * VS[0][0] + VS[1][0] * VS[1][0];
  const double K01 = VS[0][0] * VS[0][1] + VS[1][0] * VS[1][1];
  VG Vp, V, Vn;
  vgeo(C, eta, m.fracs[0], m.fracs[1], a.kh, a.kv, V);
  Vp = V;
  double gp[6][NC];
  double xa[NC][6], xc[NC][6], xb[NC][6];  // explicit: x_{l-1}, x_l, x_{l+1}
  if (!IMPLICIT) {
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) {
      ld6(xin + cc * P6, 0, c, L, nt, xc[cc]);
#pragma unroll
      for (int k = 0; k < 6; ++k) xa[cc][k] = 0.0;
    }
  }
  for (int l = 0; l < L; ++l) {
    const double ft = m.fracs[l], fb = m.fracs[l + 1];
    if (l < L - 1) vgeo(C, eta, fb, m.fracs[l + 2], a.kh, a.kv, Vn);
    double wt[6], wm[6], wtn[3] = {0, 0, 0}, dw[6];
    ld6(a.wt, l, c, L, nt, wt);
    wm_layer(a, C.b, e0, e1, ft, fb, l, c, L, nt, wm);
    if (l < L - 1) {
#pragma unroll
      for (int k = 0; k < 3; ++k) wtn[k] = a.wt[((size_t)k * L + l + 1) * nt + c];
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) dw[k] = wt[k] - wm[k];
    double d[6][6], u[3][6], w[3][6];
    vop_layer(j2d, l, L, Vp, V, Vn, dw, wt, wm, wtn, a.n0, a.order, m.err, d, u, w);
    // M1 of this layer (Kronecker form)
    double jz1[3], q1[6], M1h[3][3];
    layer_jz(C.b, e1, ft, fb, jz1);
    hq(jz1, q1);
    mass_h(q1, M1h);
    double g[6][NC];
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) g[i][cc] = rhs[cc * P6 + ((size_t)i * L + l) * nt + c];
    if (IMPLICIT) {
      // (M1 - dt A) blocks
#pragma unroll
      for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int j = 0; j < 6; ++j) {
          const double Kij = (i / 3 == j / 3) ? K00 : K01;
          d[i][j] = Kij * (j2d * M1h[i % 3][j % 3]) - dt * d[i][j];
        }
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 6; ++j) {
          u[i][j] = -dt * u[i][j];
          w[i][j] = -dt * w[i][j];
        }
      if (l > 0) {
#pragma unroll
        for (int j = 0; j < 6; ++j) {
          double G[6];
#pragma unroll
          for (int k = 0; k < 6; ++k) G[k] = Gs[((size_t)(k * 6 + j) * L + (l - 1)) * nt + c];
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < 6; ++k) acc = acc + u[i][k] * G[k];
            d[i][j] = d[i][j] - acc;
          }
        }
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int cc = 0; cc < NC; ++cc) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < 6; ++k) acc = acc + u[i][k] * gp[k][cc];
            g[i][cc] = g[i][cc] - acc;
          }
      }
      const int bad = lu6(d);
      if (bad >= 0) {
        report(m.err, PDG_ERR_ZERO_PIVOT, l, bad, 0.0);
        return;
      }
      if (l < L - 1) {
        double t[6][6];
#pragma unroll
        for (int j = 0; j < 6; ++j)
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            t[i][j] = 0.0;
            t[3 + i][j] = w[i][j];
          }
        lu6_solve<6>(d, t);
#pragma unroll
        for (int i = 0; i < 6; ++i)
#pragma unroll
          for (int j = 0; j < 6; ++j) Gs[((size_t)(i * 6 + j) * L + l) * nt + c] = t[i][j];
      }
      lu6_solve<NC>(d, g);
#pragma unroll
      for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) {
          x[cc * P6 + ((size_t)i * L + l) * nt + c] = g[i][cc];
          gp[i][cc] = g[i][cc];
        }
    } else {
      // rhs + dt (D x_l + [U x_{l-1}; W x_{l+1}]), then M1^-1 via K^-1 (x) (J2D Mjz)^-1
      if (l < L - 1) {
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) ld6(xin + cc * P6, l + 1, c, L, nt, xb[cc]);
      }
      const double det = K00 * K00 - K01 * K01;
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        double y[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          double t = 0.0;
#pragma unroll
          for (int j = 0; j < 6; ++j) t += d[i][j] * xc[cc][j];
          if (i < 3 && l > 0) {
#pragma unroll
            for (int j = 0; j < 6; ++j) t += u[i][j] * xa[cc][j];
          }
          if (i >= 3 && l < L - 1) {
#pragma unroll
            for (int j = 0; j < 6; ++j) t += w[i - 3][j] * xb[cc][j];
          }
          y[i] = g[i][cc] + dt * t;
        }
        double z[2][3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          z[0][k] = (K00 * y[k] - K01 * y[3 + k]) / det;
          z[1][k] = (-K01 * y[k] + K00 * y[3 + k]) / det;
        }
#pragma unroll
        for (int lev = 0; lev < 2; ++lev) {
          double A[3][3];
#pragma unroll
          for (int p = 0; p < 3; ++p)
#pragma unroll
            for (int q = 0; q < 3; ++q) A[p][q] = j2d * M1h[p][q];
          if (!solve3(A, z[lev])) report(m.err, PDG_ERR_ZERO_PIVOT, l, 3 * lev, 0.0);
        }
        double o[6];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          o[k] = z[0][k];
          o[3 + k] = z[1][k];
        }
        st6(x + cc * P6, l, c, L, nt, o);
      }
#pragma unroll
      for (int cc = 0; cc < NC; ++cc)
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          xa[cc][k] = xc[cc][k];
          xc[cc][k] = xb[cc][k];
        }
    }
    Vp = V;
    V = Vn;
  }
  if (IMPLICIT) {
    double xn[6][NC];
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) xn[i][cc] = gp[i][cc];
    for (int l = L - 2; l >= 0; --l) {
      double xl[6][NC];
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        double G[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) G[k] = Gs[((size_t)(i * 6 + k) * L + l) * nt + c];
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) {
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < 6; ++k) acc = acc + G[k] * xn[k][cc];
          xl[i][cc] = x[cc * P6 + ((size_t)i * L + l) * nt + c] - acc;
        }
      }
#pragma unroll
      for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) {
          x[cc * P6 + ((size_t)i * L + l) * nt + c] = xl[i][cc];
          xn[i][cc] = xl[i][cc];
        }
    }
  }
}

}  // namespace pdg

using namespace pdg;

extern "C" {

int pdg_solve_sweep(int kind, int ncol, int L, int nc, const double* rhs, const double* j2d, const int* layers,
                    double* out, pdg_err* err, void* stream) {
  if (ncol == 0) return PDG_OK;
  k_sweep<<<nblocks(ncol, 128), 128, 0, (cudaStream_t)stream>>>(kind, ncol, L, nc, rhs, j2d, layers, out, err);
  return check_launch_noctx();
}

int pdg_solve_banded(int ncol, int L, int nc, const double* d, const double* u, const double* w, double* gu,
                     double* gw, const double* rhs, double* x, pdg_err* err, void* stream) {
  if (ncol == 0) return PDG_OK;
  const dim3 g(nblocks(ncol, 128)), b(128);
  cudaStream_t s = (cudaStream_t)stream;
  if (nc == 1)
    k_banded_solve<1><<<g, b, 0, s>>>(ncol, L, d, u, w, gu, gw, rhs, x, err);
  else if (nc == 2)
    k_banded_solve<2><<<g, b, 0, s>>>(ncol, L, d, u, w, gu, gw, rhs, x, err);
  else
    return PDG_ERR_SHAPE;
  return check_launch_noctx();
}

int pdg_apply_banded(int ncol, int L, int nc, const double* d, const double* u, const double* w, const double* x,
                     double* y, void* stream) {
  if (ncol == 0) return PDG_OK;
  k_banded_apply<<<nblocks(ncol, 128), 128, 0, (cudaStream_t)stream>>>(ncol, L, nc, d, u, w, x, y);
  return check_launch_noctx();
}

int pdg_build_implicit(long long P, const double* mass, const double* d, const double* u, const double* w, double dt,
                       double* od, double* ou, double* ow, void* stream) {
  if (P == 0) return PDG_OK;
  k_build_implicit<<<nblocks(P, 128), 128, 0, (cudaStream_t)stream>>>(P, mass, d, u, w, dt, od, ou, ow);
  return check_launch_noctx();
}

int pdg_mass_op(int L, int nt, int nc, int solve, const double* mass, const double* f, double* out, pdg_err* err,
                void* stream) {
  const long long P = (long long)L * nt;
  if (P == 0) return PDG_OK;
  k_mass_op<<<nblocks(P, 128), 128, 0, (cudaStream_t)stream>>>(P, L, nt, nc, solve, mass, f, out, err);
  return check_launch_noctx();
}

int pdg_solve_tridiagonal(int nb, int n, const double* lo, const double* di, const double* up, const double* rhs,
                          double* x, double* work, pdg_err* err, void* stream) {
  if (nb == 0 || n == 0) return PDG_OK;
  k_tridiag<<<nblocks(nb, 128), 128, 0, (cudaStream_t)stream>>>(nb, n, lo, di, up, rhs, x, work, err);
  return check_launch_noctx();
}

int pdg_assemble_vertical(pdg_ctx* ctx, const double* eta_g, const double* wt, const double* wm, double kh, double kv,
                          double n0, int order, const int* els, int n_els, double* d, double* u, double* w,
                          void* stream) {
  const int n = els ? n_els : ctx->nt;
  if (n == 0) return PDG_OK;
  VopArgs a{eta_g, wt, wm, nullptr, nullptr, 1.0, kh, kv, n0, order};
  k_vop<<<nblocks(n, 128), 128, 0, (cudaStream_t)stream>>>(ctx->view(), a, els, n, d, u, w);
  return check_launch(ctx);
}

// fused vertical stage: implicit (M1 - dt A) x = rhs, or explicit x = M1^-1 (rhs + dt A xin)
int pdg_step_vertical(pdg_ctx* ctx, int ncomp, int implicit, const double* eta_u, const double* eta0,
                      const double* eta1, double dt_mesh, const double* wt, double kh, double kv, double n0, int order,
                      double dt, const double* rhs, const double* xin, double* x, void* stream) {
  VopArgs a{eta_u, wt, nullptr, eta0, eta1, dt_mesh, kh, kv, n0, order};
  const int nt = ctx->nt;
  double* Gs = nullptr;
  if (implicit) {
    Gs = ctx->ws3((size_t)36 * ctx->L * nt);
    if (!Gs) return PDG_ERR_CUDA;
  }
  const dim3 g(nblocks(nt, 128)), b(128);
  cudaStream_t s = (cudaStream_t)stream;
  DMesh m = ctx->view();
  if (ncomp == 2) {
    if (implicit)
      k_vstep<2, true><<<g, b, 0, s>>>(m, a, dt, rhs, xin, Gs, x);
    else
      k_vstep<2, false><<<g, b, 0, s>>>(m, a, dt, rhs, xin, Gs, x);
  } else {
    if (implicit)
      k_vstep<1, true><<<g, b, 0, s>>>(m, a, dt, rhs, xin, Gs, x);
    else
      k_vstep<1, false><<<g, b, 0, s>>>(m, a, dt, rhs, xin, Gs, x);
  }
  return check_launch(ctx);
}

}  // extern "C"

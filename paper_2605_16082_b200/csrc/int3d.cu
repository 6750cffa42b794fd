// 3D internal-mode assemblies (internal3d.py), one thread per column, layer loop inside.
//
// Each kernel has an API flavour (inputs exactly as the reference passes them: explicit
// factor / mass / q arrays) and, where the stepper needs it, a FUSED flavour that rebuilds
// the flux factor, the consistent transport q~ and the prism masses on the fly, so those
// 12-, 36- and 12-double-per-prism intermediates never touch HBM.
#include "col3d.cuh"
#include "ctx.cuh"
#include "tile.cuh"

namespace pdg {

struct Cols {
  const int* els;
  int n;
  __device__ __forceinline__ int col(int i) const { return els ? els[i] : i; }
};

__device__ __forceinline__ void load_eta(const double* __restrict__ e, int c, int nt, double eta[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) eta[i] = e[i * nt + c];
}

// ============================================================================ prism mass
// internal3d.py:114-123.  M[i][j] = K[li][lj] J2D Mjz[ai][aj] (Kronecker form of the 12-point rule)
__global__ void k_prism_mass(DMesh m, const double* __restrict__ eta_g, Cols cs, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cs.n) return;
  const int c = cs.col(i), nt = m.nt, L = m.L;
  const double j2d = ldg(m.j2d + c);
  double eta[3], b[3];
  load_eta(eta_g, c, nt, eta);
#pragma unroll
  for (int k = 0; k < 3; ++k) b[k] = ldg(m.b + k * nt + c);
  const double K[2][2] = {{VS[0][0] * VS[0][0] + VS[1][0] * VS[1][0], VS[0][0] * VS[0][1] + VS[1][0] * VS[1][1]},
                          {VS[0][1] * VS[0][0] + VS[1][1] * VS[1][0], VS[0][1] * VS[0][1] + VS[1][1] * VS[1][1]}};
  for (int l = 0; l < L; ++l) {
    double jz[3], jzq[6], Mh[3][3];
    layer_jz(b, eta, m.fracs[l], m.fracs[l + 1], jz);
    hq(jz, jzq);
    mass_h(jzq, Mh);
#pragma unroll
    for (int r = 0; r < 6; ++r)
#pragma unroll
      for (int s = 0; s < 6; ++s) out[pix36(r * 6 + s, l, c, L, nt)] = K[r / 3][s / 3] * (j2d * Mh[r % 3][s % 3]);
  }
}

// ============================================================================ projection
// internal3d.py:164-181: M q = <phi (Jz u) J2D Jz>.  Kronecker path: q_lev = Mjz^-1 R_lev,
// R_lev[a] = sum_q QW BARY_a jzq^2 u_lev(q) (K and J2D cancel).  Optional outputs: the
// vertical-DOF column sum of q (internal3d.py:184-187) and total thickness 2 sum Jz (mesh.py:422).
template <bool MASS_GIVEN>
__global__ void k_project(DMesh m, const double* __restrict__ eta_g, const double* __restrict__ ux,
                          const double* __restrict__ uy, const double* __restrict__ mass, Cols cs,
                          double* __restrict__ q, double* __restrict__ qsum, double* __restrict__ htot) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cs.n) return;
  const int c = cs.col(i), nt = m.nt, L = m.L;
  const size_t P6 = (size_t)6 * L * nt;
  const double j2d = ldg(m.j2d + c);
  double eta[3], b[3];
  load_eta(eta_g, c, nt, eta);
#pragma unroll
  for (int k = 0; k < 3; ++k) b[k] = ldg(m.b + k * nt + c);
  double st[2][3] = {{0, 0, 0}, {0, 0, 0}}, sb[2][3] = {{0, 0, 0}, {0, 0, 0}}, hs[3] = {0, 0, 0};
  double fcur = m.fracs[0], fnext = m.fracs[1];  // sigma fractions, loaded one layer ahead
  for (int l = 0; l < L; ++l) {
    const double ft = fcur, fb = fnext;
    fcur = fnext;
    fnext = l + 2 <= L ? m.fracs[l + 2] : 0.0;
    double jz[3], jzq[6];
    layer_jz(b, eta, ft, fb, jz);
    hq(jz, jzq);
    double u[2][6];
    ld6g(ux, l, c, L, nt, u[0]);
    ld6g(uy, l, c, L, nt, u[1]);
    double out[2][6];
    if (MASS_GIVEN) {
      double a[6][6], rhs[6][2];
#pragma unroll
      for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int s = 0; s < 6; ++s) a[r][s] = mass[pix36(r * 6 + s, l, c, L, nt)];
      double up[2][2][6];
      at_pts(u[0], up[0]);
      at_pts(u[1], up[1]);
#pragma unroll
      for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          double t = 0.0;
#pragma unroll
          for (int vv = 0; vv < 2; ++vv)
#pragma unroll
            for (int qq = 0; qq < 6; ++qq)
              t += QW[qq] * (j2d * jzq[qq] * jzq[qq]) * up[cc][vv][qq] * (VS[vv][r / 3] * BARY[qq][r % 3]);
          rhs[r][cc] = t;
        }
      const int bad = lu6(a);
      if (bad >= 0) report(m.err, PDG_ERR_ZERO_PIVOT, l, bad, 0.0);
      lu6_solve<2>(a, rhs);
#pragma unroll
      for (int r = 0; r < 6; ++r) {
        out[0][r] = rhs[r][0];
        out[1][r] = rhs[r][1];
      }
    } else {
      // one unpivoted LU of the jz-weighted triangle mass serves both levels and both components
      double Mh[3][3];
      mass_h(jzq, Mh);
      const double r0 = 1.0 / Mh[0][0];
      const double l10 = Mh[1][0] * r0, l20 = Mh[2][0] * r0;
      const double a11 = Mh[1][1] - l10 * Mh[0][1], a12 = Mh[1][2] - l10 * Mh[0][2];
      const double r1 = 1.0 / a11;
      const double l21 = (Mh[2][1] - l20 * Mh[0][1]) * r1;
      const double a22 = (Mh[2][2] - l20 * Mh[0][2]) - l21 * a12;
      if (Mh[0][0] == 0.0 || a11 == 0.0 || a22 == 0.0) report(m.err, PDG_ERR_ZERO_PIVOT, l, 0, 0.0);
      const double r2 = 1.0 / a22;
#pragma unroll
      for (int cc = 0; cc < 2; ++cc)
#pragma unroll
        for (int lev = 0; lev < 2; ++lev) {
          double uq[6], R[3] = {0, 0, 0};
          hq(u[cc] + 3 * lev, uq);
#pragma unroll
          for (int qq = 0; qq < 6; ++qq) {
            const double w = QW[qq] * jzq[qq] * jzq[qq] * uq[qq];
#pragma unroll
            for (int a = 0; a < 3; ++a) R[a] += w * BARY[qq][a];
          }
          R[1] -= l10 * R[0];
          R[2] -= l20 * R[0] + l21 * R[1];
          R[2] *= r2;
          R[1] = (R[1] - a12 * R[2]) * r1;
          R[0] = (R[0] - Mh[0][1] * R[1] - Mh[0][2] * R[2]) * r0;
#pragma unroll
          for (int a = 0; a < 3; ++a) out[cc][3 * lev + a] = R[a];
        }
    }
    st6(q, l, c, L, nt, out[0]);
    st6(q + P6, l, c, L, nt, out[1]);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      st[0][a] += out[0][a];
      st[1][a] += out[1][a];
      sb[0][a] += out[0][3 + a];
      sb[1][a] += out[1][3 + a];
      hs[a] += jz[a];
    }
  }
  if (qsum) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      qsum[a * nt + c] = st[0][a] + sb[0][a];
      qsum[(3 + a) * nt + c] = st[1][a] + sb[1][a];
    }
  }
  if (htot) {
#pragma unroll
    for (int a = 0; a < 3; ++a) htot[a * nt + c] = 2.0 * hs[a];
  }
}

// vertical-DOF column sum of an N-component P6 field (internal3d.py:184-187) and total thickness
__global__ void k_colsum(int nt, int L, int ncomp, const double* __restrict__ f, double* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nt) return;
  for (int cc = 0; cc < ncomp; ++cc) {
    const double* fc = f + (size_t)cc * 6 * L * nt;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double st = 0.0, sb = 0.0;
      for (int l = 0; l < L; ++l) {
        st += fc[pix(a, l, c, L, nt)];
        sb += fc[pix((3 + a), l, c, L, nt)];
      }
      out[(cc * 3 + a) * nt + c] = st + sb;
    }
  }
}

__global__ void k_htot(DMesh m, const double* __restrict__ eta_g, double* __restrict__ htot) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int nt = m.nt;
  if (c >= m.nown) return;
  double eta[3], b[3], hs[3] = {0, 0, 0};
  load_eta(eta_g, c, nt, eta);
#pragma unroll
  for (int k = 0; k < 3; ++k) b[k] = ldg(m.b + k * nt + c);
  for (int l = 0; l < m.L; ++l) {
    double jz[3];
    layer_jz(b, eta, m.fracs[l], m.fracs[l + 1], jz);
#pragma unroll
    for (int a = 0; a < 3; ++a) hs[a] += jz[a];
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) htot[a * nt + c] = 2.0 * hs[a];
}

// transport mismatch (Qbar - sum_col q) / H per column corner (internal3d.py:198-200)
__global__ void k_mismatch(int nt, int nown, const double* __restrict__ qbar, const double* __restrict__ qsum,
                           const double* __restrict__ htot, double* __restrict__ mis) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nown) return;
#pragma unroll
  for (int cc = 0; cc < 2; ++cc)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int o = (cc * 3 + a) * nt + c;
      mis[o] = (qbar[o] - qsum[o]) / htot[a * nt + c];
    }
}

// consistent_transport (internal3d.py:190-208): qbar = q + Jz mis, both levels
__global__ void k_consistent(DMesh m, const double* __restrict__ eta_g, const double* __restrict__ q,
                             const double* __restrict__ mis, Cols cs, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cs.n) return;
  const int c = cs.col(i), nt = m.nt, L = m.L;
  const size_t P6 = (size_t)6 * L * nt;
  double eta[3], b[3], mi[2][3];
  load_eta(eta_g, c, nt, eta);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    b[k] = ldg(m.b + k * nt + c);
    mi[0][k] = mis[k * nt + c];
    mi[1][k] = mis[(3 + k) * nt + c];
  }
  for (int l = 0; l < L; ++l) {
    double jz[3];
    layer_jz(b, eta, m.fracs[l], m.fracs[l + 1], jz);
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      double v[6];
      ld6(q + cc * P6, l, c, L, nt, v);
#pragma unroll
      for (int n = 0; n < 6; ++n) v[n] = v[n] + jz[n % 3] * mi[cc][n % 3];
      st6(out + cc * P6, l, c, L, nt, v);
    }
  }
}

// ============================================================================ flux factor (API)
__global__ void k_factor(DMesh m, const double* __restrict__ eta_g, const double* __restrict__ q, double g, Cols cs,
                         double* __restrict__ fac) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cs.n) return;
  const int c = cs.col(i), nt = m.nt, L = m.L;
  const size_t P6 = (size_t)6 * L * nt;
  Col C;
  load_col(m, c, C);
  double eta[3];
  load_eta(eta_g, c, nt, eta);
  EdgeNb E[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) edge_setup(m, C, eta, eta_g, k, g, E[k]);
  for (int l = 0; l < L; ++l) {
    const double jm = 0.5 * (m.fracs[l + 1] - m.fracs[l]);
    double qo[2][6];
    ld6(q, l, c, L, nt, qo[0]);
    ld6(q + P6, l, c, L, nt, qo[1]);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double f[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
      if (C.tag[k] == 0) {
        double qn[2][4];
        ld_nb4(q, E[k].k2, E[k].e2, l, L, nt, qn[0]);
        ld_nb4(q + P6, E[k].k2, E[k].e2, l, L, nt, qn[1]);
        lat_factor(C, E[k], k, jm, qo, qn, f);
      }
#pragma unroll
      for (int vv = 0; vv < 2; ++vv)
#pragma unroll
        for (int h = 0; h < 2; ++h) fac[((size_t)((k * 2 + vv) * 2 + h) * L + l) * nt + c] = f[vv][h];
    }
  }
}

__device__ __forceinline__ void ld_fac(const double* __restrict__ fac, int k, int l, int c, int L, int nt,
                                       double f[2][2]) {
#pragma unroll
  for (int vv = 0; vv < 2; ++vv)
#pragma unroll
    for (int h = 0; h < 2; ++h) f[vv][h] = fac[((size_t)((k * 2 + vv) * 2 + h) * L + l) * nt + c];
}

// ============================================================================ baroclinic head r
// sigma-layer geometry of the baroclinic head from per-column constants: z = eta - f H gives
// grad z_top = grad eta - f_t grad H, grad z_mid = grad eta - f_mid grad H, grad Jz = jm grad H and
// MHQ Jz = jm MHQ H with jm = (f_b - f_t)/2 -- a handful of FMAs per layer instead of layer_geo's
// node-wise z evaluation and eight rounded dot products (values agree to rounding).
struct RSig {
  double ex, ey, hx, hy, mh[3];
};
__device__ __forceinline__ void rsig_init(const Col& C, const double eta[3], RSig& R) {
  double H[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) H[i] = eta[i] - C.b[i];
  R.ex = (eta[0] * C.dx[0] + eta[1] * C.dx[1]) + eta[2] * C.dx[2];
  R.ey = (eta[0] * C.dy[0] + eta[1] * C.dy[1]) + eta[2] * C.dy[2];
  R.hx = (H[0] * C.dx[0] + H[1] * C.dx[1]) + H[2] * C.dx[2];
  R.hy = (H[0] * C.dy[0] + H[1] * C.dy[1]) + H[2] * C.dy[2];
  mhq_vec(H, R.mh);
}
struct RLay {
  double A[3], dzmid[2], djz[2], dztop[2];
};
__device__ __forceinline__ void rsig_layer(const RSig& R, double ft, double fb, RLay& G) {
  const double jm = 0.5 * (fb - ft), fm = 0.5 * (ft + fb);
#pragma unroll
  for (int a = 0; a < 3; ++a) G.A[a] = jm * R.mh[a];
  G.dzmid[0] = R.ex - fm * R.hx;
  G.dzmid[1] = R.ey - fm * R.hy;
  G.djz[0] = jm * R.hx;
  G.djz[1] = jm * R.hy;
  G.dztop[0] = R.ex - ft * R.hx;
  G.dztop[1] = R.ey - ft * R.hy;
}

// internal3d.py:327-405 + columns.py:95-122.  FROM_T: rho' = -alpha (T - t_ref) inline.
// Volume term in closed form: -g J2D sum_v VS[v][lev] (grad_iso(v) (MHQ Jz)_a - mid2(v) (MHQ drho/dzeta)_a)
// (meas * m_h = -J2D mid2 cancels the 1/Jz of the metric); lateral {Jz} = (f_b - f_t)/2 {H}.
template <bool FROM_T, int MINB>
__global__ void __launch_bounds__(128, MINB) k_compute_r(DMesh m, const double* __restrict__ eta_g,
                                                   const double* __restrict__ rhoT, double alpha, double tref,
                                                   double g, Cols cs, double* __restrict__ r) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cs.n) return;
  const int c = cs.col(i), nt = m.nt, L = m.L;
  const size_t P6 = (size_t)6 * L * nt;
  Col C;
  load_col(m, c, C);
  double eta[3];
  load_eta(eta_g, c, nt, eta);
  EdgeNb E[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) edge_setup(m, C, eta, eta_g, k, g, E[k]);
  RSig R;
  rsig_init(C, eta, R);
  const double ex = R.ex, ey = R.ey;
  const double j2d = C.j2d;
  const double f6 = 6.0 / j2d;  // Mh^-1 factor (columns.py:59-69), once per column
  double s[2][3] = {{0, 0, 0}, {0, 0, 0}};
  double prevb[3] = {0, 0, 0};
  for (int l = 0; l < L; ++l) {
    const double ft = m.fracs[l], fb = m.fracs[l + 1];
    const double jm = 0.5 * (fb - ft);
    if (l + 1 < L) pf6(rhoT, l + 1, c, L, nt);
    RLay G;
    rsig_layer(R, ft, fb, G);
    double rho[6];
    ld6(rhoT, l, c, L, nt, rho);
    if (FROM_T) {
#pragma unroll
      for (int n = 0; n < 6; ++n) rho[n] = -alpha * (rho[n] - tref);
    }
    double acc[2][6];
    {
      double gi[2][2], A[3], B[3], dzn[3];
#pragma unroll
      for (int lev = 0; lev < 2; ++lev) {
        gi[lev][0] = (rho[3 * lev] * C.dx[0] + rho[3 * lev + 1] * C.dx[1]) + rho[3 * lev + 2] * C.dx[2];
        gi[lev][1] = (rho[3 * lev] * C.dy[0] + rho[3 * lev + 1] * C.dy[1]) + rho[3 * lev + 2] * C.dy[2];
      }
#pragma unroll
      for (int a = 0; a < 3; ++a) dzn[a] = 0.5 * (rho[a] - rho[3 + a]);
#pragma unroll
      for (int a = 0; a < 3; ++a) A[a] = G.A[a];
      mhq_vec(dzn, B);
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        double t[2][3];
#pragma unroll
        for (int vv = 0; vv < 2; ++vv) {
          const double gv = VS[vv][0] * gi[0][d] + VS[vv][1] * gi[1][d];
          const double md = d == 0 ? G.dzmid[0] + ZQP[vv] * G.djz[0] : G.dzmid[1] + ZQP[vv] * G.djz[1];
#pragma unroll
          for (int a = 0; a < 3; ++a) t[vv][a] = gv * A[a] - md * B[a];
        }
#pragma unroll
        for (int lev = 0; lev < 2; ++lev)
#pragma unroll
          for (int a = 0; a < 3; ++a) acc[d][3 * lev + a] = -(g * j2d) * (VS[0][lev] * t[0][a] + VS[1][lev] * t[1][a]);
      }
    }
    // interior horizontal face above this layer: 2g J2D (-grad z_face) . int phi [[rho]]
    if (l > 0) {
      double dr[3], fi[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) dr[a] = 0.5 * (rho[a] - prevb[a]);
      const double sdr = (dr[0] + dr[1]) + dr[2];
#pragma unroll
      for (int a = 0; a < 3; ++a) fi[a] = (dr[a] + sdr) * (1.0 / 24.0);
#pragma unroll
      for (int d = 0; d < 2; ++d)
#pragma unroll
        for (int a = 0; a < 3; ++a) acc[d][a] += 2.0 * g * j2d * (-G.dztop[d]) * fi[a];
    }
    // interior lateral faces: g n [[rho]] {Jz} Jedge
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (C.tag[k] != 0) continue;
      double n4[4], dj[2][2];
      ld_nb4(rhoT, E[k].k2, E[k].e2, l, L, nt, n4);
      if (FROM_T) {
#pragma unroll
        for (int n = 0; n < 4; ++n) n4[n] = -alpha * (n4[n] - tref);
      }
      tr_jump(rho, k, n4, dj);
      // one scalar face field projected once, added with g Je n_d (as k_compute_r_t: bitwise equal)
      double xs[2][2], pr[2][2];
#pragma unroll
      for (int vv = 0; vv < 2; ++vv)
#pragma unroll
        for (int h = 0; h < 2; ++h) xs[vv][h] = dj[vv][h] * (jm * E[k].hm[h]);
      lat_proj(xs, pr);
      const double gje = g * (0.5 * C.el[k]);
      lat_put(acc[0], k, pr, gje * C.nx[k]);
      lat_put(acc[1], k, pr, gje * C.ny[k]);
    }
    // surface fold: -Mh (g rho_s grad_h eta)
    if (l == 0) {
      double mr[3];
      mh_apply3(rho, j2d, mr);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        acc[0][a] -= g * mr[a] * ex;
        acc[1][a] -= g * mr[a] * ey;
      }
    }
    // top-down sweep (columns.py:108-121)
#pragma unroll
    for (int d = 0; d < 2; ++d) {
      double gt[3], gb[3], out[6];
      mh_inv3f(acc[d], f6, gt);
      mh_inv3f(acc[d] + 3, f6, gb);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        s[d][a] = s[d][a] + (gt[a] + gb[a]);
        out[a] = -s[d][a] + 2.0 * gb[a];
        out[3 + a] = -s[d][a];
      }
      st6(r + d * P6, l, c, L, nt, out);
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) prevb[a] = rho[3 + a];
  }
}

// ============================================================================ w from continuity (API)
// internal3d.py:434-502 + columns.py:125-151 (bed-anchored sweep, bottom-up)
__global__ void __launch_bounds__(128) k_compute_w(DMesh m, const double* __restrict__ eta_g,
                                                   const double* __restrict__ q, const double* __restrict__ ux,
                                                   const double* __restrict__ uy, const double* __restrict__ fac,
                                                   Cols cs, double* __restrict__ w) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cs.n) return;
  const int c = cs.col(i), nt = m.nt, L = m.L;
  const size_t P6 = (size_t)6 * L * nt;
  Col C;
  load_col(m, c, C);
  double eta[3];
  load_eta(eta_g, c, nt, eta);
  const double j2d = C.j2d;
  const double f6 = 6.0 / j2d;  // Mh^-1 factor (columns.py:59-69), once per column
  double s[3] = {0, 0, 0};
  double ut_below[6][2];  // top-face q/Jz of layer l+1 at the 6 horizontal points
  for (int l = L - 1; l >= 0; --l) {
    const double ft = m.fracs[l], fb = m.fracs[l + 1];
    LGeo G;
    layer_geo(C, eta, ft, fb, G);
    double jzq[6];
    hq(G.jz, jzq);
    double qv[2][6];
    ld6(q, l, c, L, nt, qv[0]);
    ld6(q + P6, l, c, L, nt, qv[1]);
    double acc[6] = {0, 0, 0, 0, 0, 0};
    double qp[2][2][6];
    at_pts(qv[0], qp[0]);
    at_pts(qv[1], qp[1]);
    // volume: + <q . grad_h(phi) J2D> (iso part) + metric part J2D dphi_z/dzeta (q . m_h)
    {
      double S[2][2];
#pragma unroll
      for (int mm = 0; mm < 2; ++mm) {
        double sx = 0.0, sy = 0.0;
#pragma unroll
        for (int vv = 0; vv < 2; ++vv)
#pragma unroll
          for (int qq = 0; qq < 6; ++qq) {
            sx += QW[qq] * VS[vv][mm] * qp[0][vv][qq];
            sy += QW[qq] * VS[vv][mm] * qp[1][vv][qq];
          }
        S[mm][0] = sx;
        S[mm][1] = sy;
      }
      iso_add(C, S, acc);
      double met[3] = {0, 0, 0};
#pragma unroll
      for (int vv = 0; vv < 2; ++vv) {
        const double m0 = G.dzmid[0] + ZQP[vv] * G.djz[0];
        const double m1 = G.dzmid[1] + ZQP[vv] * G.djz[1];
#pragma unroll
        for (int qq = 0; qq < 6; ++qq) {
          const double qm = qp[0][vv][qq] * (-m0 / jzq[qq]) + qp[1][vv][qq] * (-m1 / jzq[qq]);
#pragma unroll
          for (int a = 0; a < 3; ++a) met[a] += QW[qq] * qm * BARY[qq][a];
        }
      }
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        acc[a] += j2d * DV[0] * met[a];
        acc[3 + a] += j2d * DV[1] * met[a];
      }
    }
    // horizontal faces: {q/Jz} . grad(z_face) with one-sided values at surface and bed
    {
      double ut[6][2], ub[6][2];
      double t0[6], t1[6], b0[6], b1[6];
      hq(qv[0], t0);
      hq(qv[1], t1);
      hq(qv[0] + 3, b0);
      hq(qv[1] + 3, b1);
#pragma unroll
      for (int qq = 0; qq < 6; ++qq) {
        ut[qq][0] = t0[qq] / jzq[qq];
        ut[qq][1] = t1[qq] / jzq[qq];
        ub[qq][0] = b0[qq] / jzq[qq];
        ub[qq][1] = b1[qq] / jzq[qq];
      }
      double ubA[6][2];  // bottom-face q/Jz of the layer above (l-1)
      if (l > 0) {
        double jza[3], jzqa[6], qa0[6], qa1[6];
        layer_jz(C.b, eta, m.fracs[l - 1], ft, jza);
        hq(jza, jzqa);
        double v0[6], v1[6];
        ld6(q, l - 1, c, L, nt, v0);
        ld6(q + P6, l - 1, c, L, nt, v1);
        hq(v0 + 3, qa0);
        hq(v1 + 3, qa1);
#pragma unroll
        for (int qq = 0; qq < 6; ++qq) {
          ubA[qq][0] = qa0[qq] / jzqa[qq];
          ubA[qq][1] = qa1[qq] / jzqa[qq];
        }
      }
      double ftq[6], fbq[6];
#pragma unroll
      for (int qq = 0; qq < 6; ++qq) {
        double mt0 = ut[qq][0], mt1 = ut[qq][1], mb0 = ub[qq][0], mb1 = ub[qq][1];
        if (l > 0) {
          mt0 = 0.5 * (ut[qq][0] + ubA[qq][0]);
          mt1 = 0.5 * (ut[qq][1] + ubA[qq][1]);
        }
        if (l < L - 1) {
          mb0 = 0.5 * (ub[qq][0] + ut_below[qq][0]);
          mb1 = 0.5 * (ub[qq][1] + ut_below[qq][1]);
        }
        ftq[qq] = mt0 * G.dztop[0] + mt1 * G.dztop[1];
        fbq[qq] = mb0 * G.dzbot[0] + mb1 * G.dzbot[1];
      }
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        double tt = 0.0, tb = 0.0;
#pragma unroll
        for (int qq = 0; qq < 6; ++qq) {
          tt += QW[qq] * ftq[qq] * BARY[qq][a];
          tb += QW[qq] * fbq[qq] * BARY[qq][a];
        }
        acc[a] += j2d * tt;
        acc[3 + a] -= j2d * tb;
      }
#pragma unroll
      for (int qq = 0; qq < 6; ++qq) {
        ut_below[qq][0] = ut[qq][0];
        ut_below[qq][1] = ut[qq][1];
      }
    }
    // lateral stabilised flux
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (C.tag[k] != 0) continue;
      double f[2][2];
      ld_fac(fac, k, l, c, L, nt, f);
      lat_add(acc, k, f, -(0.5 * C.el[k]));
    }
    // bed kinematic fold w(bed) = u . grad_h(b)
    if (l == L - 1) {
      const double bx = (C.b[0] * C.dx[0] + C.b[1] * C.dx[1]) + C.b[2] * C.dx[2];
      const double by = (C.b[0] * C.dy[0] + C.b[1] * C.dy[1]) + C.b[2] * C.dy[2];
      double wb[3], mw[3];
#pragma unroll
      for (int a = 0; a < 3; ++a)
        wb[a] = ux[pix((3 + a), l, c, L, nt)] * bx + uy[pix((3 + a), l, c, L, nt)] * by;
      mh_apply3(wb, j2d, mw);
#pragma unroll
      for (int a = 0; a < 3; ++a) acc[3 + a] += mw[a];
    }
    double gt[3], gb[3], out[6];
    mh_inv3f(acc, f6, gt);
    mh_inv3f(acc + 3, f6, gb);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      out[3 + a] = s[a] + gb[a] - gt[a];
      out[a] = s[a] + gb[a] + gt[a];
      s[a] = out[a];
    }
    st6(w, l, c, L, nt, out);
  }
}

// ============================================================================ w~ (API + fused)
// internal3d.py:505-541.  FUSED: qbar = q + Jz mis and its factor rebuilt on the fly (Jz mis =
// jm * (H mis) on sigma layers).  Iso volume moment in closed form: S[m] = sum_l K[m][l] W1 . q_l.
template <bool FUSED, int MINB>
__global__ void __launch_bounds__(128, MINB) k_compute_wtilde(DMesh m, const double* __restrict__ eta_g,
                                                        const double* __restrict__ qb, const double* __restrict__ fac,
                                                        const double* __restrict__ mis, double g, Cols cs,
                                                        double* __restrict__ w) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cs.n) return;
  const int c = cs.col(i), nt = m.nt, L = m.L;
  const size_t P6 = (size_t)6 * L * nt;
  Col C;
  load_col(m, c, C);
  double eta[3];
  load_eta(eta_g, c, nt, eta);
  EdgeNb E[3];
  double mo[2][3], mn[3][2][2];  // H * mismatch: own corners, neighbour edge corners
  if (FUSED) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      edge_setup(m, C, eta, eta_g, k, g, E[k]);
      mo[0][k] = mis[k * nt + c] * (eta[k] - C.b[k]);
      mo[1][k] = mis[(3 + k) * nt + c] * (eta[k] - C.b[k]);
      if (C.tag[k] == 0) {
        const int e2 = E[k].e2, k2 = E[k].k2;
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          mn[k][cc][0] = mis[(cc * 3 + EV0(k2)) * nt + e2] * E[k].hn[0];
          mn[k][cc][1] = mis[(cc * 3 + EV1(k2)) * nt + e2] * E[k].hn[1];
        }
      }
    }
  }
  const double j2d = C.j2d;
  const double f6 = 6.0 / j2d;  // Mh^-1 factor (columns.py:59-69), once per column
  double s[3] = {0, 0, 0};
  for (int l = L - 1; l >= 0; --l) {
    const double jm = 0.5 * (m.fracs[l + 1] - m.fracs[l]);
    if (l > 0) {
      pf6(qb, l - 1, c, L, nt);
      pf6(qb + P6, l - 1, c, L, nt);
    }
    double qv[2][6];
    ld6(qb, l, c, L, nt, qv[0]);
    ld6(qb + P6, l, c, L, nt, qv[1]);
    if (FUSED) {
#pragma unroll
      for (int cc = 0; cc < 2; ++cc)
#pragma unroll
        for (int n = 0; n < 6; ++n) qv[cc][n] = qv[cc][n] + jm * mo[cc][n % 3];
    }
    double acc[6] = {0, 0, 0, 0, 0, 0};
    {
      double wq[2][2];
#pragma unroll
      for (int cc = 0; cc < 2; ++cc)
#pragma unroll
        for (int lev = 0; lev < 2; ++lev)
          wq[cc][lev] = W1[0] * qv[cc][3 * lev] + W1[1] * qv[cc][3 * lev + 1] + W1[2] * qv[cc][3 * lev + 2];
      double S[2][2];
#pragma unroll
      for (int mm = 0; mm < 2; ++mm) {
        S[mm][0] = KM[mm][0] * wq[0][0] + KM[mm][1] * wq[0][1];
        S[mm][1] = KM[mm][0] * wq[1][0] + KM[mm][1] * wq[1][1];
      }
      iso_add(C, S, acc);
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (C.tag[k] != 0) continue;
      double f[2][2];
      if (FUSED) {
        double qn[2][4];
        ld_nb4(qb, E[k].k2, E[k].e2, l, L, nt, qn[0]);
        ld_nb4(qb + P6, E[k].k2, E[k].e2, l, L, nt, qn[1]);
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          qn[cc][0] = qn[cc][0] + jm * mn[k][cc][0];
          qn[cc][1] = qn[cc][1] + jm * mn[k][cc][1];
          qn[cc][2] = qn[cc][2] + jm * mn[k][cc][0];
          qn[cc][3] = qn[cc][3] + jm * mn[k][cc][1];
        }
        lat_factor(C, E[k], k, jm, qv, qn, f);
      } else {
        ld_fac(fac, k, l, c, L, nt, f);
      }
      lat_add(acc, k, f, -(0.5 * C.el[k]));
    }
    double gt[3], gb[3], out[6];
    mh_inv3f(acc, f6, gt);
    mh_inv3f(acc + 3, f6, gb);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      out[3 + a] = s[a] + gb[a] - gt[a];
      out[a] = s[a] + gb[a] + gt[a];
      s[a] = out[a];
    }
    st6(w, l, c, L, nt, out);
  }
}

// the 4 lateral nodes (t0, t1, b0, b1) of the neighbour across local edge k2, staged word base w0
__device__ __forceinline__ void nb4_s(const double* S, int tj, int w0, int k2, int j, double n4[4]) {
  const int a = EV0(k2), b = EV1(k2);
  n4[0] = S[(w0 + a) * tj + j];
  n4[1] = S[(w0 + b) * tj + j];
  n4[2] = S[(w0 + 3 + a) * tj + j];
  n4[3] = S[(w0 + 3 + b) * tj + j];
}

// tiled baroclinic head (k_compute_r<FROM_T> with T / rho' staged: 6 words per column)
template <bool FROM_T, int TW>
__global__ void __launch_bounds__(TW, 384 / TW) k_compute_r_t(DMesh m, const double* __restrict__ eta_g, double alpha,
                                                   double tref, double g, const __grid_constant__ StagePlanes sp,
                                                   const int* __restrict__ tslot, const int* __restrict__ halo,
                                                   const int* __restrict__ hoff, int tj, double* __restrict__ r,
                                                   double* __restrict__ rsum) {
  extern __shared__ double sbuf[];  // [2][6][tj], then the sigma fractions [L + 1], then ints [6][TW]
  TileStage<6, TW> ts;
  ts.init(m, halo, hoff);
  const int c = ts.c, nt = m.nt, L = m.L, t = ts.t;
  double* frs = sbuf + (size_t)2 * 6 * tj;
  int* nsl = reinterpret_cast<int*>(frs + L + 1);   // [k][t] neighbour slot, [3 + k][t] its local edge
  for (int i2 = t; i2 <= L; i2 += TW) frs[i2] = m.fracs[i2];
  const size_t P6 = (size_t)6 * L * nt;
  ts.issue(sbuf, tj, sp, 0, halo);
  Col C;
  double eta[3], ex = 0.0, ey = 0.0;
  EdgeNb E[3];
  RSig R{};
  if (ts.act) {
    load_col(m, c, C);
    load_eta(eta_g, c, nt, eta);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      edge_setup(m, C, eta, eta_g, k, g, E[k]);
      nsl[k * TW + t] = tslot[k * nt + c];
      nsl[(3 + k) * TW + t] = E[k].k2;
    }
    rsig_init(C, eta, R);
    ex = R.ex;
    ey = R.ey;
  }
  const double j2d = ts.act ? C.j2d : 0.0;
  const double f6 = 6.0 / j2d;  // Mh^-1 factor (columns.py:59-69), once per column
  double s[2][3] = {{0, 0, 0}, {0, 0, 0}};
  // rsum (optional): sum over the layers of jm (r_top + r_bot) per corner, the only form of r the
  // F3D->2D column sum needs (its mass term is linear in r and Mjz = jm Mjz(H) on sigma layers)
  double rs[2][3] = {{0, 0, 0}, {0, 0, 0}};
  double prevb[3] = {0, 0, 0};
  cp_async_wait0();
  __syncthreads();
  for (int l = 0; l < L; ++l) {
    if (l + 1 < L) ts.issue(sbuf + (size_t)((l + 1) & 1) * 6 * tj, tj, sp, (unsigned)(l + 1) * (unsigned)nt, halo);
    const double* S = sbuf + (size_t)(l & 1) * 6 * tj;
    const double ft = frs[l], fb = frs[l + 1];
    if (ts.act) {
      const double jm = 0.5 * (fb - ft);
      RLay G;
      rsig_layer(R, ft, fb, G);
      double rho[6];
#pragma unroll
      for (int n = 0; n < 6; ++n) rho[n] = S[n * tj + t];
      if (FROM_T) {
#pragma unroll
        for (int n = 0; n < 6; ++n) rho[n] = -alpha * (rho[n] - tref);
      }
      double acc[2][6];
      {
        double gi[2][2], A[3], B[3], dzn[3];
#pragma unroll
        for (int lev = 0; lev < 2; ++lev) {
          gi[lev][0] = (rho[3 * lev] * C.dx[0] + rho[3 * lev + 1] * C.dx[1]) + rho[3 * lev + 2] * C.dx[2];
          gi[lev][1] = (rho[3 * lev] * C.dy[0] + rho[3 * lev + 1] * C.dy[1]) + rho[3 * lev + 2] * C.dy[2];
        }
#pragma unroll
        for (int a = 0; a < 3; ++a) dzn[a] = 0.5 * (rho[a] - rho[3 + a]);
  #pragma unroll
      for (int a = 0; a < 3; ++a) A[a] = G.A[a];
        mhq_vec(dzn, B);
#pragma unroll
        for (int d = 0; d < 2; ++d) {
          double tt[2][3];
#pragma unroll
          for (int vv = 0; vv < 2; ++vv) {
            const double gv = VS[vv][0] * gi[0][d] + VS[vv][1] * gi[1][d];
            const double md = d == 0 ? G.dzmid[0] + ZQP[vv] * G.djz[0] : G.dzmid[1] + ZQP[vv] * G.djz[1];
#pragma unroll
            for (int a = 0; a < 3; ++a) tt[vv][a] = gv * A[a] - md * B[a];
          }
#pragma unroll
          for (int lev = 0; lev < 2; ++lev)
#pragma unroll
            for (int a = 0; a < 3; ++a)
              acc[d][3 * lev + a] = -(g * j2d) * (VS[0][lev] * tt[0][a] + VS[1][lev] * tt[1][a]);
        }
      }
      if (l > 0) {
        double dr[3], fi[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) dr[a] = 0.5 * (rho[a] - prevb[a]);
        const double sdr = (dr[0] + dr[1]) + dr[2];
#pragma unroll
        for (int a = 0; a < 3; ++a) fi[a] = (dr[a] + sdr) * (1.0 / 24.0);
#pragma unroll
        for (int d = 0; d < 2; ++d)
#pragma unroll
          for (int a = 0; a < 3; ++a) acc[d][a] += 2.0 * g * j2d * (-G.dztop[d]) * fi[a];
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        if (C.tag[k] != 0) continue;
        double n4[4], dj[2][2];
        nb4_s(S, tj, 0, nsl[(3 + k) * TW + t], nsl[k * TW + t], n4);
        if (FROM_T) {
#pragma unroll
          for (int n = 0; n < 4; ++n) n4[n] = -alpha * (n4[n] - tref);
        }
        tr_jump(rho, k, n4, dj);
        // g n [[rho']] {Jz} Jedge: one scalar face field projected once, added with g Je n_d
        double xs[2][2], pr[2][2];
#pragma unroll
        for (int vv = 0; vv < 2; ++vv)
#pragma unroll
          for (int h = 0; h < 2; ++h) xs[vv][h] = dj[vv][h] * (jm * E[k].hm[h]);
        lat_proj(xs, pr);
        const double gje = g * (0.5 * C.el[k]);
        lat_put(acc[0], k, pr, gje * C.nx[k]);
        lat_put(acc[1], k, pr, gje * C.ny[k]);
      }
      if (l == 0) {
        double mr[3];
        mh_apply3(rho, j2d, mr);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          acc[0][a] -= g * mr[a] * ex;
          acc[1][a] -= g * mr[a] * ey;
        }
      }
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        double gt[3], gb[3], out[6];
        mh_inv3f(acc[d], f6, gt);
        mh_inv3f(acc[d] + 3, f6, gb);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          s[d][a] = s[d][a] + (gt[a] + gb[a]);
          out[a] = -s[d][a] + 2.0 * gb[a];
          out[3 + a] = -s[d][a];
          rs[d][a] += jm * (out[a] + out[3 + a]);
        }
        st6(r + d * P6, l, c, L, nt, out);
      }
#pragma unroll
      for (int a = 0; a < 3; ++a) prevb[a] = rho[3 + a];
    }
    cp_async_wait0();
    __syncthreads();
  }
  if (rsum && ts.act) {
#pragma unroll
    for (int d = 0; d < 2; ++d)
#pragma unroll
      for (int a = 0; a < 3; ++a) rsum[(d * 3 + a) * nt + c] = rs[d][a];
  }
}

// tiled fused w~ (k_compute_wtilde<true> with q staged: 12 words per column), bottom-up
template <int TW>
__global__ void __launch_bounds__(TW) k_compute_wtilde_t(DMesh m, const double* __restrict__ eta_g,
                                                        const double* __restrict__ mis, double g,
                                                        const __grid_constant__ StagePlanes sp,
                                                        const int* __restrict__ tslot, const int* __restrict__ halo,
                                                        const int* __restrict__ hoff, int tj, double* __restrict__ w) {
  extern __shared__ double sbuf[];  // [2][12][tj], then the sigma fractions [L + 1]
  TileStage<12, TW> ts;
  ts.init(m, halo, hoff);
  const int c = ts.c, nt = m.nt, L = m.L, t = ts.t;
  double* frs = sbuf + (size_t)2 * 12 * tj;
  for (int i2 = t; i2 <= L; i2 += TW) frs[i2] = m.fracs[i2];
  ts.issue(sbuf + (size_t)((L - 1) & 1) * 12 * tj, tj, sp, (unsigned)(L - 1) * (unsigned)nt, halo);
  Col C;
  double eta[3];
  EdgeNb E[3];
  int sl[3];
  double mo[2][3], mn[3][2][2];
  if (ts.act) {
    load_col(m, c, C);
    load_eta(eta_g, c, nt, eta);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      edge_setup(m, C, eta, eta_g, k, g, E[k]);
      sl[k] = tslot[k * nt + c];
      mo[0][k] = mis[k * nt + c] * (eta[k] - C.b[k]);
      mo[1][k] = mis[(3 + k) * nt + c] * (eta[k] - C.b[k]);
      if (C.tag[k] == 0) {
        const int e2 = E[k].e2, k2 = E[k].k2;
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          mn[k][cc][0] = mis[(cc * 3 + EV0(k2)) * nt + e2] * E[k].hn[0];
          mn[k][cc][1] = mis[(cc * 3 + EV1(k2)) * nt + e2] * E[k].hn[1];
        }
      }
    }
  }
  const double j2d = ts.act ? C.j2d : 0.0;
  const double f6 = 6.0 / j2d;  // Mh^-1 factor (columns.py:59-69), once per column
  double s[3] = {0, 0, 0};
  cp_async_wait0();
  __syncthreads();
  for (int l = L - 1; l >= 0; --l) {
    if (l > 0) ts.issue(sbuf + (size_t)((l - 1) & 1) * 12 * tj, tj, sp, (unsigned)(l - 1) * (unsigned)nt, halo);
    const double* S = sbuf + (size_t)(l & 1) * 12 * tj;
    if (ts.act) {
      const double jm = 0.5 * (frs[l + 1] - frs[l]);
      double qv[2][6];
#pragma unroll
      for (int cc = 0; cc < 2; ++cc)
#pragma unroll
        for (int n = 0; n < 6; ++n) qv[cc][n] = S[(cc * 6 + n) * tj + t] + jm * mo[cc][n % 3];
      double acc[6] = {0, 0, 0, 0, 0, 0};
      {
        double wq[2][2];
#pragma unroll
        for (int cc = 0; cc < 2; ++cc)
#pragma unroll
          for (int lev = 0; lev < 2; ++lev)
            wq[cc][lev] = W1[0] * qv[cc][3 * lev] + W1[1] * qv[cc][3 * lev + 1] + W1[2] * qv[cc][3 * lev + 2];
        double Sm[2][2];
#pragma unroll
        for (int mm = 0; mm < 2; ++mm) {
          Sm[mm][0] = KM[mm][0] * wq[0][0] + KM[mm][1] * wq[0][1];
          Sm[mm][1] = KM[mm][0] * wq[1][0] + KM[mm][1] * wq[1][1];
        }
        iso_add(C, Sm, acc);
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        if (C.tag[k] != 0) continue;
        double f[2][2], qn[2][4];
        nb4_s(S, tj, 0, E[k].k2, sl[k], qn[0]);
        nb4_s(S, tj, 6, E[k].k2, sl[k], qn[1]);
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          qn[cc][0] = qn[cc][0] + jm * mn[k][cc][0];
          qn[cc][1] = qn[cc][1] + jm * mn[k][cc][1];
          qn[cc][2] = qn[cc][2] + jm * mn[k][cc][0];
          qn[cc][3] = qn[cc][3] + jm * mn[k][cc][1];
        }
        lat_factor(C, E[k], k, jm, qv, qn, f);
        lat_add(acc, k, f, -(0.5 * C.el[k]));
      }
      double gt[3], gb[3], out[6];
      mh_inv3f(acc, f6, gt);
      mh_inv3f(acc + 3, f6, gb);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        out[3 + a] = s[a] + gb[a] - gt[a];
        out[a] = s[a] + gb[a] + gt[a];
        s[a] = out[a];
      }
      st6(w, l, c, L, nt, out);
    }
    cp_async_wait0();
    __syncthreads();
  }
}

// ============================================================================ horizontal RHS
// internal3d.py:695-751 (momentum, NC=2) and :754-792 (tracer, NC=1), kappa = nu = 0.
// MODE 0 (API):   explicit q_adv / factor / mass arrays; out = F (P6N); Coriolis and -M r/rho0
//                 only if mass_terms (the host adds them over ALL rows when els is given, as the
//                 reference does).
// MODE 1 (PRED):  q from array, factor from q on the fly, Mu from geometry, + stresses;
//                 out = vertical-DOF column sum of (F + stress) (the F3D->2D forcing).
// MODE 2 (STAGE): qbar = q + Jz mis on the fly, factor from qbar, Mu/M0/M1 from geometry;
//                 out = M0 u0 + dt (F + stress + M1 F2D/H1)  (momentum)  or  M0 T0 + dt F (tracer).
struct HArgs {
  const double* eta_u;   // grid of the stage values (C3)
  const double* u;       // advected field (NC planes of P6)
  const double* qa;      // q_adv (API, PRED) or q (STAGE), 2 x P6
  const double* fac;     // FAC (API)
  const double* r;       // 2 x P6 (momentum)
  const double* mass;    // MASS (API)
  const double* mis;     // [2][3][nt] (STAGE)
  const double* eta0;    // STAGE: step-start grid
  const double* eta1;    // STAGE: end-of-stage grid
  const double* u0;      // STAGE: step-start field (NC x P6)
  const double* f2d;     // STAGE momentum: [2][3][nt]
  double g, f, rho0, tsx, tsy, cd, dt;
  int mass_terms;
  // per-component planes (momentum x, y[, tracer]); filled from u / u0 / out by the entry points
  const double* uc[3];
  const double* u0c[3];
  double* outc[3];
  const double* rsum = nullptr;   // F3D->2D: per-column layer sum of jm (r_top + r_bot) (RS kernels)
  double* wt = nullptr;           // STAGE (WT kernels): w~ of the stage, [6][L][nt]
};

__device__ __forceinline__ void mjz(const double jz[3], double M[3][3]) {
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int q = p; q < 3; ++q) {
      const double s = T3[p][q][0] * jz[0] + T3[p][q][1] * jz[1] + T3[p][q][2] * jz[2];
      M[p][q] = s;
      M[q][p] = s;
    }
}
// y = (K (x) J2D Mjz) x  -- the prism mass of internal3d.py:114-123 applied in Kronecker form
__device__ __forceinline__ void kron_apply(const double M[3][3], double j2d, const double x[6], double y[6]) {
  double h0[3], h1[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    h0[a] = j2d * (M[a][0] * x[0] + M[a][1] * x[1] + M[a][2] * x[2]);
    h1[a] = j2d * (M[a][0] * x[3] + M[a][1] * x[4] + M[a][2] * x[5]);
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    y[a] = KM[0][0] * h0[a] + KM[0][1] * h1[a];
    y[3 + a] = KM[1][0] * h0[a] + KM[1][1] * h1[a];
  }
}

template <int NC, int MODE, int MINB>
__global__ void __launch_bounds__(128, MINB) k_hrhs(DMesh m, HArgs a, Cols cs, double* __restrict__ out) {
  asm volatile(".pragma \"enable_smem_spilling\";");
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cs.n) return;
  const int c = cs.col(i), nt = m.nt, L = m.L;
  const size_t P6 = (size_t)6 * L * nt;
  Col C;
  load_col(m, c, C);
  double eta[3];
  load_eta(a.eta_u, c, nt, eta);
  EdgeNb E[3];
  double mo[2][3], mn[3][2][2];   // H * mismatch (STAGE)
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (MODE != 0) {
      edge_setup(m, C, eta, a.eta_u, k, a.g, E[k]);
    } else {
      E[k].e2 = C.nb[k];
      E[k].k2 = C.nk[k];
    }
    if (MODE == 2) {
      const double H = eta[k] - C.b[k];
      mo[0][k] = a.mis[k * nt + c] * H;
      mo[1][k] = a.mis[(3 + k) * nt + c] * H;
      if (C.tag[k] == 0) {
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          mn[k][cc][0] = a.mis[(cc * 3 + EV0(E[k].k2)) * nt + E[k].e2] * E[k].hn[0];
          mn[k][cc][1] = a.mis[(cc * 3 + EV1(E[k].k2)) * nt + E[k].e2] * E[k].hn[1];
        }
      }
    }
  }
  double eta0[3], eta1[3], F1[2][3];
  if (MODE == 2) {
    load_eta(a.eta0, c, nt, eta0);
    load_eta(a.eta1, c, nt, eta1);
    if constexpr (NC >= 2) {
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double H1 = eta1[k] - C.b[k];
        F1[0][k] = a.f2d[k * nt + c] / H1;
        F1[1][k] = a.f2d[(3 + k) * nt + c] / H1;
      }
    }
  }
  const double j2d = C.j2d;
  double csum[NC][3];
#pragma unroll
  for (int cc = 0; cc < NC; ++cc)
#pragma unroll
    for (int k = 0; k < 3; ++k) csum[cc][k] = 0.0;
  for (int l = 0; l < L; ++l) {
    const double ft = m.fracs[l], fb = m.fracs[l + 1];
    const double jm = 0.5 * (fb - ft);
    double u[NC][6], qv[2][6];
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) ld6g(a.uc[cc], l, c, L, nt, u[cc]);
    ld6g(a.qa, l, c, L, nt, qv[0]);
    ld6g(a.qa + P6, l, c, L, nt, qv[1]);
    if (MODE == 2) {
#pragma unroll
      for (int cc = 0; cc < 2; ++cc)
#pragma unroll
        for (int n = 0; n < 6; ++n) qv[cc][n] = qv[cc][n] + jm * mo[cc][n % 3];
    }
    double acc[NC][6];
    // volume advection J2D grad_h(phi_h) . <phi_z u q>: bilinear closed form
    {
      double z[2][2][3];   // MHQ q_{d, level}
#pragma unroll
      for (int d = 0; d < 2; ++d)
#pragma unroll
        for (int lev = 0; lev < 2; ++lev) mhq_vec(qv[d] + 3 * lev, z[d][lev]);
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        double S[2][2];
#pragma unroll
        for (int d = 0; d < 2; ++d) {
          double dot[2][2];
#pragma unroll
          for (int l1 = 0; l1 < 2; ++l1)
#pragma unroll
            for (int l2 = 0; l2 < 2; ++l2)
              dot[l1][l2] = u[cc][3 * l1] * z[d][l2][0] + u[cc][3 * l1 + 1] * z[d][l2][1] + u[cc][3 * l1 + 2] * z[d][l2][2];
#pragma unroll
          for (int mm = 0; mm < 2; ++mm)
            S[mm][d] = K3[mm][0][0] * dot[0][0] + K3[mm][0][1] * dot[0][1] + K3[mm][1][0] * dot[1][0] +
                       K3[mm][1][1] * dot[1][1];
        }
#pragma unroll
        for (int lev = 0; lev < 2; ++lev)
#pragma unroll
          for (int p = 0; p < 3; ++p) acc[cc][3 * lev + p] = j2d * (C.dx[p] * S[lev][0] + C.dy[p] * S[lev][1]);
      }
    }
    // lateral upwind flux on interior faces
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (C.tag[k] != 0) continue;
      double f[2][2];
      if (MODE == 0) {
        ld_fac(a.fac, k, l, c, L, nt, f);
      } else {
        double qn[2][4];
        ld_nb4g(a.qa, E[k].k2, E[k].e2, l, L, nt, qn[0]);
        ld_nb4g(a.qa + P6, E[k].k2, E[k].e2, l, L, nt, qn[1]);
        if (MODE == 2) {
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            qn[cc][0] = qn[cc][0] + jm * mn[k][cc][0];
            qn[cc][1] = qn[cc][1] + jm * mn[k][cc][1];
            qn[cc][2] = qn[cc][2] + jm * mn[k][cc][0];
            qn[cc][3] = qn[cc][3] + jm * mn[k][cc][1];
          }
        }
        lat_factor(C, E[k], k, jm, qv, qn, f);
      }
      const double je = -(0.5 * C.el[k]);
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        double n4[4], ti[2][2], te[2][2], x[2][2];
        ld_nb4g(a.uc[cc], E[k].k2, E[k].e2, l, L, nt, n4);
        tr_own(u[cc], k, ti);
        tr_nb(n4, te);
#pragma unroll
        for (int vv = 0; vv < 2; ++vv)
#pragma unroll
          for (int h = 0; h < 2; ++h) x[vv][h] = (f[vv][h] >= 0.0 ? ti[vv][h] : te[vv][h]) * f[vv][h];
        lat_add(acc[cc], k, x, je);
      }
    }
    double Mu[3][3];
    bool have_mu = false;
    // Coriolis f M (u_y, -u_x) and -M r / rho0 (momentum), internal3d.py:746-750
    if constexpr (NC >= 2) {
      if (MODE != 0 || a.mass_terms) {
        double rr[2][6];
        ld6g(a.r, l, c, L, nt, rr[0]);
        ld6g(a.r + P6, l, c, L, nt, rr[1]);
        if (MODE == 0) {
          double M[6][6];
#pragma unroll
          for (int p = 0; p < 6; ++p)
#pragma unroll
            for (int q = 0; q < 6; ++q) M[p][q] = a.mass[pix36(p * 6 + q, l, c, L, nt)];
#pragma unroll
          for (int p = 0; p < 6; ++p) {
            double mu0 = 0, mu1 = 0, mr0 = 0, mr1 = 0;
#pragma unroll
            for (int q = 0; q < 6; ++q) {
              mu0 += M[p][q] * u[0][q];
              mu1 += M[p][q] * u[1][q];
              mr0 += M[p][q] * rr[0][q];
              mr1 += M[p][q] * rr[1][q];
            }
            if (a.f != 0.0) {
              acc[0][p] += a.f * mu1;
              acc[1][p] -= a.f * mu0;
            }
            acc[0][p] -= mr0 / a.rho0;
            acc[1][p] -= mr1 / a.rho0;
          }
        } else {
          double jz[3];
          layer_jz(C.b, eta, ft, fb, jz);
          mjz(jz, Mu);
          have_mu = true;
          const double ir = 1.0 / a.rho0;
          double y0[6], y1[6], m0[6], m1[6];
#pragma unroll
          for (int n = 0; n < 6; ++n) {
            y0[n] = a.f * u[1][n] - rr[0][n] * ir;
            y1[n] = -a.f * u[0][n] - rr[1][n] * ir;
          }
          kron_apply(Mu, j2d, y0, m0);
          kron_apply(Mu, j2d, y1, m1);
#pragma unroll
          for (int n = 0; n < 6; ++n) {
            acc[0][n] += m0[n];
            acc[1][n] += m1[n];
          }
        }
      }
    }
    (void)have_mu;
    // surface wind and bottom drag (internal3d.py:919-934)
    if constexpr (NC >= 2 && MODE != 0) {
      if (l == 0) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          acc[0][k] += j2d / 6.0 * a.tsx;
          acc[1][k] += j2d / 6.0 * a.tsy;
        }
      }
      if (l == L - 1 && a.cd != 0.0) {
        double dx3[3], dy3[3], mx[3], my[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double ubx = u[0][3 + k], uby = u[1][3 + k];
          const double sp = sqrt(ubx * ubx + uby * uby);
          dx3[k] = -a.cd * sp * ubx;
          dy3[k] = -a.cd * sp * uby;
        }
        mh_apply3(dx3, j2d, mx);
        mh_apply3(dy3, j2d, my);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          acc[0][3 + k] += mx[k];
          acc[1][3 + k] += my[k];
        }
      }
    }
    if (MODE == 1) {
#pragma unroll
      for (int cc = 0; cc < NC; ++cc)
#pragma unroll
        for (int k = 0; k < 3; ++k) csum[cc][k] += acc[cc][k] + acc[cc][3 + k];
    } else if (MODE == 2) {
      double j0[3], M0[3][3];
      layer_jz(C.b, eta0, ft, fb, j0);
      mjz(j0, M0);
      double mf[2][3] = {{0, 0, 0}, {0, 0, 0}};
      if constexpr (NC >= 2) {
        double j1[3], M1[3][3];
        layer_jz(C.b, eta1, ft, fb, j1);
        mjz(j1, M1);
        const double kk = (KM[0][0] + KM[0][1]) * j2d;   // F2D/H1 is the same on both levels
#pragma unroll
        for (int cc = 0; cc < 2; ++cc)
#pragma unroll
          for (int p = 0; p < 3; ++p) mf[cc][p] = kk * (M1[p][0] * F1[cc][0] + M1[p][1] * F1[cc][1] + M1[p][2] * F1[cc][2]);
      }
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        double x0[6], m0x[6], o[6];
        ld6g(a.u0c[cc], l, c, L, nt, x0);
        kron_apply(M0, j2d, x0, m0x);
#pragma unroll
        for (int n = 0; n < 6; ++n) {
          if (NC >= 2 && cc < 2)
            o[n] = m0x[n] + a.dt * (acc[cc][n] + mf[cc][n % 3]);
          else
            o[n] = m0x[n] + a.dt * acc[cc][n];
        }
        st6(a.outc[cc], l, c, L, nt, o);
      }
    } else {
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) st6(a.outc[cc], l, c, L, nt, acc[cc]);
    }
  }
  if (MODE == 1) {
#pragma unroll
    for (int cc = 0; cc < NC; ++cc)
#pragma unroll
      for (int k = 0; k < 3; ++k) out[(cc * 3 + k) * nt + c] = csum[cc][k];
  }
}

// ---------------------------------------------------------------------------------------------
// Shared-memory variant of the stepper flavours (MODE 1, 2): the ~58 per-column constants live in
// shared memory and are re-read (volatile) at the point of use instead of pinning ~120 registers
// for the whole layer loop; 64-thread blocks keep the static footprint under 48 KB.
namespace shf {
enum { J2D = 0, DX = 1, DY = 4, EL = 7, NX = 10, NY = 13, B = 16, ETA = 19, STAB = 22, MO = 28, MN = 34, E0 = 46,
       E1 = 49, F1 = 52, N = 58,
       // MODE 2: the per-column sigma-layer triangle masses Mjz(H) of the stage and start grids
       // (packed symmetric) over the B / ETA and E0 / E1 words, and in F1 the per-column factor
       // of the F2D/H1 term (the layer loop needs only these)
       MHU = 16, MH0 = 46, N2 = 58,
       F6 = 58 };   // WT: 6 / J2D (the Mh^-1 factor of the w~ sweep), one word past N2
}

__device__ __forceinline__ void lat_factor_v(double nx, double ny, double st0, double st1, int k, double jm,
                                             const double qo[2][6], const double qn[2][4], double fac[2][2]) {
  double o[6], n4[4];
#pragma unroll
  for (int i = 0; i < 6; ++i) o[i] = nx * qo[0][i] + ny * qo[1][i];
#pragma unroll
  for (int i = 0; i < 4; ++i) n4[i] = nx * qn[0][i] + ny * qn[1][i];
  double t[2][2];
  tr_mean(o, k, n4, t);
#pragma unroll
  for (int vv = 0; vv < 2; ++vv) {
    fac[vv][0] = t[vv][0] + jm * st0;
    fac[vv][1] = t[vv][1] + jm * st1;
  }
}

// SAME: the stage values are the step-start values (stage 1: u == u0, T == T0), so M0 u0 reuses
// the u words already loaded for the fluxes instead of loading them again.
// WT (MODE 2): also w~ (compute_wtilde, internal3d.py:505-541): its right-hand side is the iso-zeta
// volume moment of q~ and the lateral flux factor this kernel forms anyway, so the layer loop runs
// bottom-up (the stage RHS has no vertical recurrence) and carries the bed-anchored sweep
// (columns.py:125-151) -- q~ and its neighbour traces are read once per stage instead of twice.
template <int NC, int MODE, int MINB, bool SAME = false, bool WT = false>
__global__ void __launch_bounds__(64, MINB) k_hrhs_s(DMesh m, HArgs a, Cols cs, double* __restrict__ out) {
  __shared__ double sdm[(MODE == 2 ? shf::N2 + (WT ? 1 : 0) : shf::N) * 64];
  __shared__ int sim[9 * 64];
  const int tid = threadIdx.x;
  const int i = blockIdx.x * 64 + tid;
  if (i >= cs.n) return;  // no block-level synchronisation below: every thread owns its own slots
  const int c = cs.col(i), nt = m.nt, L = m.L;
  const size_t P6 = (size_t)6 * L * nt;
  volatile double* S = sdm;
#define SD(f) S[(f) * 64 + tid]
  {
    Col C;
    load_col(m, c, C);
    double eta[3];
    load_eta(a.eta_u, c, nt, eta);
    SD(shf::J2D) = C.j2d;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      SD(shf::DX + k) = C.dx[k];
      SD(shf::DY + k) = C.dy[k];
      SD(shf::EL + k) = C.el[k];
      SD(shf::NX + k) = C.nx[k];
      SD(shf::NY + k) = C.ny[k];
      SD(shf::B + k) = C.b[k];
      SD(shf::ETA + k) = eta[k];
      EdgeNb E;
      edge_setup(m, C, eta, a.eta_u, k, a.g, E);
      sim[(0 + k) * 64 + tid] = C.tag[k];
      sim[(3 + k) * 64 + tid] = E.e2;
      sim[(6 + k) * 64 + tid] = E.k2;
      if (C.tag[k] == 0) {
        SD(shf::STAB + 2 * k) = E.stab[0];
        SD(shf::STAB + 2 * k + 1) = E.stab[1];
      }
      if (MODE == 2) {
        const double H = eta[k] - C.b[k];
        SD(shf::MO + k) = a.mis[k * nt + c] * H;
        SD(shf::MO + 3 + k) = a.mis[(3 + k) * nt + c] * H;
        if (C.tag[k] == 0) {
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            SD(shf::MN + (k * 2 + cc) * 2) = a.mis[(cc * 3 + EV0(E.k2)) * nt + E.e2] * E.hn[0];
            SD(shf::MN + (k * 2 + cc) * 2 + 1) = a.mis[(cc * 3 + EV1(E.k2)) * nt + E.e2] * E.hn[1];
          }
        }
      }
    }
    if (MODE == 2) {
      // sigma layers: Jz = (f_b - f_t) H / 2 = jm H at every point, so each layer's triangle mass
      // is jm Mjz(H) with a per-column Mjz(H) (values equal the per-layer forms up to rounding)
      double Hu[3], H0[3], H1[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double e1 = a.eta1[k * nt + c];
        Hu[k] = eta[k] - C.b[k];
        H0[k] = a.eta0[k * nt + c] - C.b[k];
        H1[k] = e1 - C.b[k];
      }
      double MH1[3][3];
#pragma unroll
      for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int q = p; q < 3; ++q) {
          SD(shf::MHU + sym6(p, q)) = T3[p][q][0] * Hu[0] + T3[p][q][1] * Hu[1] + T3[p][q][2] * Hu[2];
          SD(shf::MH0 + sym6(p, q)) = T3[p][q][0] * H0[0] + T3[p][q][1] * H0[1] + T3[p][q][2] * H0[2];
          MH1[p][q] = MH1[q][p] = T3[p][q][0] * H1[0] + T3[p][q][1] * H1[1] + T3[p][q][2] * H1[2];
        }
      if (WT) SD(shf::F6) = 6.0 / C.j2d;
      if constexpr (NC >= 2) {
        // the F2D/H1 broadcast term (K (x) J2D Mjz(eta1)) F summed over the two levels is
        // jm (KM00 + KM01) J2D Mjz(H1) F: its per-column factor, scaled by jm per layer
        const double kk = (KM[0][0] + KM[0][1]) * C.j2d;
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          double F[3];
#pragma unroll
          for (int k = 0; k < 3; ++k) F[k] = a.f2d[(cc * 3 + k) * nt + c] / H1[k];
#pragma unroll
          for (int p = 0; p < 3; ++p)
            SD(shf::F1 + cc * 3 + p) = kk * (MH1[p][0] * F[0] + MH1[p][1] * F[1] + MH1[p][2] * F[2]);
        }
      }
    }
  }
  double csum[NC][3];
#pragma unroll
  for (int cc = 0; cc < NC; ++cc)
#pragma unroll
    for (int k = 0; k < 3; ++k) csum[cc][k] = 0.0;
  // sigma fractions, loaded one layer ahead (WT: bottom-up, from the bed)
  double fcur = WT ? m.fracs[L] : m.fracs[0], fnext = WT ? m.fracs[L - 1] : m.fracs[1];
  const double rdt = MODE == 2 ? 1.0 / a.dt : 0.0;
  double ws[3] = {0.0, 0.0, 0.0};   // WT: the w~ sweep value (columns.py:125-151)
  for (int li = 0; li < L; ++li) {
    const int l = WT ? L - 1 - li : li;
    const double ft = WT ? fnext : fcur, fb = WT ? fcur : fnext;
    fcur = fnext;
    if (WT)
      fnext = l >= 1 ? m.fracs[l - 1] : 0.0;
    else
      fnext = l + 2 <= L ? m.fracs[l + 2] : 0.0;
    const double jm = 0.5 * (fb - ft);
    unsigned ln = (unsigned)L * (unsigned)nt;   // plane stride, hidden from the optimiser (see k_vexpl2)
    asm volatile("" : "+r"(ln));
    const unsigned lnt = (unsigned)l * (unsigned)nt, lo = lnt + (unsigned)c;
    double u[NC][6], qv[2][6];
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) ld6g_o(a.uc[cc], lo, ln, u[cc]);
    ld6g_o(a.qa, lo, ln, qv[0]);
    ld6g_o(a.qa + P6, lo, ln, qv[1]);
    if (MODE == 2) {
#pragma unroll
      for (int cc = 0; cc < 2; ++cc)
#pragma unroll
        for (int n = 0; n < 6; ++n) qv[cc][n] = qv[cc][n] + jm * SD(shf::MO + cc * 3 + n % 3);
    }
    double acc[NC][6];
    // per-layer triangle masses: MODE 2 from the per-column sigma forms (scaled by jm)
    auto msym = [&](int w, double M[3][3]) {
#pragma unroll
      for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int q = 0; q < 3; ++q) M[p][q] = SD(w + sym6(p, q));
    };
    if constexpr (MODE == 2) {
      // the mass terms first, so their own loads (r, u0) issue together with u and q instead of
      // at the end of the layer:  out = dt (M0 u0 / dt + M (f u^perp - r / rho0) + M1 F2D/H1
      // + stresses + volume + lateral)
      const double j2d = SD(shf::J2D), jj = jm * j2d;
      double M0[3][3];
      msym(shf::MH0, M0);
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        double x0[6], m0x[6];
        if (SAME) {
#pragma unroll
          for (int n = 0; n < 6; ++n) x0[n] = u[cc][n];
        } else {
          ld6g_o(a.u0c[cc], lo, ln, x0);
        }
        kron_apply(M0, jj, x0, m0x);
#pragma unroll
        for (int n = 0; n < 6; ++n) acc[cc][n] = m0x[n] * rdt;
      }
      if constexpr (NC >= 2) {
        double rr[2][6];
        ld6g_o(a.r, lo, ln, rr[0]);
        ld6g_o(a.r + P6, lo, ln, rr[1]);
        double Mu[3][3];
        msym(shf::MHU, Mu);
        const double ir = 1.0 / a.rho0;
        double y0[6], y1[6], m0[6], m1[6];
#pragma unroll
        for (int n = 0; n < 6; ++n) {
          y0[n] = a.f * u[1][n] - rr[0][n] * ir;
          y1[n] = -a.f * u[0][n] - rr[1][n] * ir;
        }
        kron_apply(Mu, jj, y0, m0);
        kron_apply(Mu, jj, y1, m1);
        double mf[2][3];
#pragma unroll
        for (int cc = 0; cc < 2; ++cc)
#pragma unroll
          for (int p = 0; p < 3; ++p) mf[cc][p] = jm * SD(shf::F1 + cc * 3 + p);
#pragma unroll
        for (int n = 0; n < 6; ++n) {
          acc[0][n] += m0[n] + mf[0][n % 3];
          acc[1][n] += m1[n] + mf[1][n % 3];
        }
        if (l == 0) {
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            acc[0][k] += j2d / 6.0 * a.tsx;
            acc[1][k] += j2d / 6.0 * a.tsy;
          }
        }
        if (l == L - 1 && a.cd != 0.0) {
          double dx3[3], dy3[3], mx[3], my[3];
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            const double ubx = u[0][3 + k], uby = u[1][3 + k];
            const double sp = sqrt(ubx * ubx + uby * uby);
            dx3[k] = -a.cd * sp * ubx;
            dy3[k] = -a.cd * sp * uby;
          }
          mh_apply3(dx3, j2d, mx);
          mh_apply3(dy3, j2d, my);
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            acc[0][3 + k] += mx[k];
            acc[1][3 + k] += my[k];
          }
        }
      }
    }
    {
      double z[2][2][3];
#pragma unroll
      for (int d = 0; d < 2; ++d)
#pragma unroll
        for (int lev = 0; lev < 2; ++lev) mhq_vec(qv[d] + 3 * lev, z[d][lev]);
      const double j2d = SD(shf::J2D);
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        double Sm[2][2];
#pragma unroll
        for (int d = 0; d < 2; ++d) {
          double dot[2][2];
#pragma unroll
          for (int l1 = 0; l1 < 2; ++l1)
#pragma unroll
            for (int l2 = 0; l2 < 2; ++l2)
              dot[l1][l2] = u[cc][3 * l1] * z[d][l2][0] + u[cc][3 * l1 + 1] * z[d][l2][1] + u[cc][3 * l1 + 2] * z[d][l2][2];
#pragma unroll
          for (int mm = 0; mm < 2; ++mm)
            Sm[mm][d] = K3[mm][0][0] * dot[0][0] + K3[mm][0][1] * dot[0][1] + K3[mm][1][0] * dot[1][0] +
                        K3[mm][1][1] * dot[1][1];
        }
#pragma unroll
        for (int lev = 0; lev < 2; ++lev)
#pragma unroll
          for (int p = 0; p < 3; ++p)
          {
            const double v = j2d * (SD(shf::DX + p) * Sm[lev][0] + SD(shf::DY + p) * Sm[lev][1]);
            if (MODE == 2)
              acc[cc][3 * lev + p] += v;
            else
              acc[cc][3 * lev + p] = v;
          }
      }
    }
    // WT: w~ right-hand side, the iso-zeta volume moment of q~ first (k_compute_wtilde order)
    double aw[6];
    if constexpr (WT) {
      double wq[2][2], Sm[2][2];
#pragma unroll
      for (int cc = 0; cc < 2; ++cc)
#pragma unroll
        for (int lev = 0; lev < 2; ++lev)
          wq[cc][lev] = W1[0] * qv[cc][3 * lev] + W1[1] * qv[cc][3 * lev + 1] + W1[2] * qv[cc][3 * lev + 2];
#pragma unroll
      for (int mm = 0; mm < 2; ++mm) {
        Sm[mm][0] = KM[mm][0] * wq[0][0] + KM[mm][1] * wq[0][1];
        Sm[mm][1] = KM[mm][0] * wq[1][0] + KM[mm][1] * wq[1][1];
      }
      const double j2d = SD(shf::J2D);
#pragma unroll
      for (int lev = 0; lev < 2; ++lev)
#pragma unroll
        for (int p = 0; p < 3; ++p) aw[3 * lev + p] = j2d * (SD(shf::DX + p) * Sm[lev][0] + SD(shf::DY + p) * Sm[lev][1]);
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (sim[k * 64 + tid] != 0) continue;
      const int e2 = sim[(3 + k) * 64 + tid], k2 = sim[(6 + k) * 64 + tid];
      double f[2][2];
      {
        double qn[2][4];
        ld_nb4g_o(a.qa, k2, lnt + (unsigned)e2, ln, qn[0]);
        ld_nb4g_o(a.qa + P6, k2, lnt + (unsigned)e2, ln, qn[1]);
        if (MODE == 2) {
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const double m0 = SD(shf::MN + (k * 2 + cc) * 2), m1 = SD(shf::MN + (k * 2 + cc) * 2 + 1);
            qn[cc][0] = qn[cc][0] + jm * m0;
            qn[cc][1] = qn[cc][1] + jm * m1;
            qn[cc][2] = qn[cc][2] + jm * m0;
            qn[cc][3] = qn[cc][3] + jm * m1;
          }
        }
        lat_factor_v(SD(shf::NX + k), SD(shf::NY + k), SD(shf::STAB + 2 * k), SD(shf::STAB + 2 * k + 1), k, jm, qv,
                     qn, f);
      }
      const double je = -(0.5 * SD(shf::EL + k));
      if (WT) lat_add(aw, k, f, je);
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        double n4[4], ti[2][2], te[2][2], x[2][2];
        ld_nb4g_o(a.uc[cc], k2, lnt + (unsigned)e2, ln, n4);
        tr_own(u[cc], k, ti);
        tr_nb(n4, te);
#pragma unroll
        for (int vv = 0; vv < 2; ++vv)
#pragma unroll
          for (int h = 0; h < 2; ++h) x[vv][h] = (f[vv][h] >= 0.0 ? ti[vv][h] : te[vv][h]) * f[vv][h];
        lat_add(acc[cc], k, x, je);
      }
    }
    if constexpr (NC >= 2 && MODE != 2) {
      double rr[2][6];
      ld6g_o(a.r, lo, ln, rr[0]);
      ld6g_o(a.r + P6, lo, ln, rr[1]);
      double Mu[3][3];
      const double mscale = SD(shf::J2D);
      {
        double jz[3], bb[3], eta[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          bb[k] = SD(shf::B + k);
          eta[k] = SD(shf::ETA + k);
        }
        layer_jz(bb, eta, ft, fb, jz);
        mjz(jz, Mu);
      }
      const double ir = 1.0 / a.rho0;
      double y0[6], y1[6], m0[6], m1[6];
#pragma unroll
      for (int n = 0; n < 6; ++n) {
        y0[n] = a.f * u[1][n] - rr[0][n] * ir;
        y1[n] = -a.f * u[0][n] - rr[1][n] * ir;
      }
      const double j2d = SD(shf::J2D);
      kron_apply(Mu, mscale, y0, m0);
      kron_apply(Mu, mscale, y1, m1);
#pragma unroll
      for (int n = 0; n < 6; ++n) {
        acc[0][n] += m0[n];
        acc[1][n] += m1[n];
      }
      if (l == 0) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          acc[0][k] += j2d / 6.0 * a.tsx;
          acc[1][k] += j2d / 6.0 * a.tsy;
        }
      }
      if (l == L - 1 && a.cd != 0.0) {
        double dx3[3], dy3[3], mx[3], my[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double ubx = u[0][3 + k], uby = u[1][3 + k];
          const double sp = sqrt(ubx * ubx + uby * uby);
          dx3[k] = -a.cd * sp * ubx;
          dy3[k] = -a.cd * sp * uby;
        }
        mh_apply3(dx3, j2d, mx);
        mh_apply3(dy3, j2d, my);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          acc[0][3 + k] += mx[k];
          acc[1][3 + k] += my[k];
        }
      }
    }
    if (MODE == 1) {
#pragma unroll
      for (int cc = 0; cc < NC; ++cc)
#pragma unroll
        for (int k = 0; k < 3; ++k) csum[cc][k] += acc[cc][k] + acc[cc][3 + k];
    } else {
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        double o[6];
#pragma unroll
        for (int n = 0; n < 6; ++n) o[n] = a.dt * acc[cc][n];
        st6(a.outc[cc], l, c, L, nt, o);
      }
    }
    if constexpr (WT) {   // w_b = s + g_b - g_t, w_t = s + g_b + g_t, s = w_t (columns.py:125-151)
      const double f6 = SD(shf::F6);
      double gt[3], gb[3], wo[6];
      mh_inv3f(aw, f6, gt);
      mh_inv3f(aw + 3, f6, gb);
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        wo[3 + p] = ws[p] + gb[p] - gt[p];
        wo[p] = ws[p] + gb[p] + gt[p];
        ws[p] = wo[p];
      }
      st6(a.wt, l, c, L, nt, wo);
    }
  }
  if (MODE == 1) {
#pragma unroll
    for (int cc = 0; cc < NC; ++cc)
#pragma unroll
      for (int k = 0; k < 3; ++k) out[(cc * 3 + k) * nt + c] = csum[cc][k];
  }
#undef SD
}


// ---------------------------------------------------------------------------------------------
// Tile-staged variant of the stepper flavours (MODE 1 PRED, MODE 2 STAGE).  A block owns TW
// consecutive (Hilbert-ordered) columns.  Per layer it stages, with per-thread cp.async copies
// issued one layer ahead into a 2-slot ring, the u (NC x 6) and q (2 x 6) words of its TW columns
// and of its halo (the out-of-tile neighbours, ctx tile maps); every lateral trace -- own or
// neighbour -- is then read from shared memory through the precomputed slot map, so the layer
// loop never waits on a scattered HBM/L2 gather.  Arithmetic is identical to k_hrhs (bitwise).

// RS (MODE 1): the r terms come as their per-column layer sum (k_compute_r_t rsum), so the layer
// loop loads no r at all
template <int NC, int MODE, int TW, bool RS = false>
__global__ void __launch_bounds__(TW, 256 / TW) k_hrhs_t(DMesh m, HArgs a, const __grid_constant__ StagePlanes sp,
                                                       const int* __restrict__ tslot, const int* __restrict__ halo,
                                                       const int* __restrict__ hoff, int tj, double* __restrict__ out) {
  constexpr int NW = 6 * NC + 12;  // staged words per column: u comps, q comps
  extern __shared__ double sbuf[];  // [2][NW][tj]
  const int t = threadIdx.x, b = blockIdx.x;
  const int c = b * TW + t, nt = m.nt, L = m.L;
  const bool act = c < m.nown;
  const size_t P6 = (size_t)6 * L * nt;
  const int h0 = hoff[b], nh = hoff[b + 1] - h0;
  // halo work split: thread t copies words [w0, w1) of halo column hj (nparts threads per column)
  const int nparts = nh > 0 ? max(1, TW / nh) : 1;
  const int wpp = (NW + nparts - 1) / nparts;
  const int part = nh > 0 ? t / nh : nparts;
  const int hj = nh > 0 ? t - part * nh : 0;
  const int hw0 = part < nparts ? part * wpp : NW, hw1 = min(NW, hw0 + wpp);
  const int hcol = part < nparts ? halo[h0 + hj] : 0;
  // halo columns beyond TW threads (nh > TW) are covered by a strided fallback
  auto stage = [&](int l) {
    double* s = sbuf + (size_t)(l & 1) * NW * tj;
    const unsigned lo = (unsigned)l * (unsigned)nt;
    if (act) {
      const unsigned oc = lo + (unsigned)c;
#pragma unroll
      for (int w = 0; w < NW; ++w) cp_async8(s + w * tj + t, sp.p[w] + oc);
    }
    const unsigned oh = lo + (unsigned)hcol;
    for (int w = hw0; w < hw1; ++w) cp_async8(s + w * tj + TW + hj, sp.p[w] + oh);
    for (int j = TW + t; j < nh; j += TW) {
      const unsigned oj = lo + (unsigned)halo[h0 + j];
      for (int w = 0; w < NW; ++w) cp_async8(s + w * tj + TW + j, sp.p[w] + oj);
    }
    cp_async_commit();
  };
  stage(0);
  Col C;
  double eta[3];
  EdgeNb E[3];
  int sl[3];
  double mo[2][3], mn[3][2][2];
  double eta0[3], eta1[3], F1[2][3];
  if (act) {
    load_col(m, c, C);
    load_eta(a.eta_u, c, nt, eta);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      edge_setup(m, C, eta, a.eta_u, k, a.g, E[k]);
      sl[k] = tslot[k * nt + c];
      if (MODE == 2) {
        const double H = eta[k] - C.b[k];
        mo[0][k] = a.mis[k * nt + c] * H;
        mo[1][k] = a.mis[(3 + k) * nt + c] * H;
        if (C.tag[k] == 0) {
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            mn[k][cc][0] = a.mis[(cc * 3 + EV0(E[k].k2)) * nt + E[k].e2] * E[k].hn[0];
            mn[k][cc][1] = a.mis[(cc * 3 + EV1(E[k].k2)) * nt + E[k].e2] * E[k].hn[1];
          }
        }
      }
    }
    if (MODE == 2) {
      load_eta(a.eta0, c, nt, eta0);
      load_eta(a.eta1, c, nt, eta1);
      if constexpr (NC >= 2) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double H1 = eta1[k] - C.b[k];
          F1[0][k] = a.f2d[k * nt + c] / H1;
          F1[1][k] = a.f2d[(3 + k) * nt + c] / H1;
        }
      }
    }
  }
  const double j2d = act ? C.j2d : 0.0;
  double csum[NC][3], sv[NC][2], ysum[2][3];
#pragma unroll
  for (int cc = 0; cc < NC; ++cc) {
#pragma unroll
    for (int k = 0; k < 3; ++k) csum[cc][k] = 0.0;
    sv[cc][0] = sv[cc][1] = 0.0;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) ysum[0][k] = ysum[1][k] = 0.0;
  cp_async_wait0();
  __syncthreads();
  double fcur = m.fracs[0], fnext = m.fracs[1];  // sigma fractions, loaded one layer ahead
  for (int l = 0; l < L; ++l) {
    if (l + 1 < L) {
      stage(l + 1);
    }
    const double* S = sbuf + (size_t)(l & 1) * NW * tj;
    const double ft = fcur, fb = fnext;
    fcur = fnext;
    fnext = l + 2 <= L ? m.fracs[l + 2] : 0.0;
    if (act) {
      const double jm = 0.5 * (fb - ft);
      double u[NC][6], qv[2][6];
#pragma unroll
      for (int cc = 0; cc < NC; ++cc)
#pragma unroll
        for (int n = 0; n < 6; ++n) u[cc][n] = S[(cc * 6 + n) * tj + t];
#pragma unroll
      for (int cc = 0; cc < 2; ++cc)
#pragma unroll
        for (int n = 0; n < 6; ++n) qv[cc][n] = S[(6 * NC + cc * 6 + n) * tj + t];
      if (MODE == 2) {
#pragma unroll
        for (int cc = 0; cc < 2; ++cc)
#pragma unroll
          for (int n = 0; n < 6; ++n) qv[cc][n] = qv[cc][n] + jm * mo[cc][n % 3];
      }
      double acc[NC][6];
      // MODE 1 only needs the column sum acc[p] + acc[3+p] of every contribution: the sums over the
      // two levels of the phi_z test functions collapse (sum_m K3[m] = KM, sum_lev VS[v][lev] = 1,
      // KM column sums = 1), so the volume, lateral and mass terms are formed per horizontal node
      // only (cs[cc][p]); the values equal the per-node forms summed, up to rounding.
      if constexpr (MODE == 1) {
        double z[2][2][3];
#pragma unroll
        for (int d = 0; d < 2; ++d)
#pragma unroll
          for (int lev = 0; lev < 2; ++lev) mhq_vec(qv[d] + 3 * lev, z[d][lev]);
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) {
          double Sd[2];
#pragma unroll
          for (int d = 0; d < 2; ++d) {
            double dot[2][2];
#pragma unroll
            for (int l1 = 0; l1 < 2; ++l1)
#pragma unroll
              for (int l2 = 0; l2 < 2; ++l2)
                dot[l1][l2] =
                    u[cc][3 * l1] * z[d][l2][0] + u[cc][3 * l1 + 1] * z[d][l2][1] + u[cc][3 * l1 + 2] * z[d][l2][2];
            Sd[d] = KM[0][0] * dot[0][0] + KM[0][1] * dot[0][1] + KM[1][0] * dot[1][0] + KM[1][1] * dot[1][1];
          }
          // J2D grad phi_p . Sd is linear in Sd: summed over the layers, applied once per column
          sv[cc][0] += Sd[0];
          sv[cc][1] += Sd[1];
        }
      } else {
        double z[2][2][3];
#pragma unroll
        for (int d = 0; d < 2; ++d)
#pragma unroll
          for (int lev = 0; lev < 2; ++lev) mhq_vec(qv[d] + 3 * lev, z[d][lev]);
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) {
          double Sm[2][2];
#pragma unroll
          for (int d = 0; d < 2; ++d) {
            double dot[2][2];
#pragma unroll
            for (int l1 = 0; l1 < 2; ++l1)
#pragma unroll
              for (int l2 = 0; l2 < 2; ++l2)
                dot[l1][l2] =
                    u[cc][3 * l1] * z[d][l2][0] + u[cc][3 * l1 + 1] * z[d][l2][1] + u[cc][3 * l1 + 2] * z[d][l2][2];
#pragma unroll
            for (int mm = 0; mm < 2; ++mm)
              Sm[mm][d] = K3[mm][0][0] * dot[0][0] + K3[mm][0][1] * dot[0][1] + K3[mm][1][0] * dot[1][0] +
                          K3[mm][1][1] * dot[1][1];
          }
#pragma unroll
          for (int lev = 0; lev < 2; ++lev)
#pragma unroll
            for (int p = 0; p < 3; ++p) acc[cc][3 * lev + p] = j2d * (C.dx[p] * Sm[lev][0] + C.dy[p] * Sm[lev][1]);
        }
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        if (C.tag[k] != 0) continue;
        const int j = sl[k], k2 = E[k].k2;
        const int na = EV0(k2), nb = EV1(k2);
        auto nb4 = [&](int w0, double n4[4]) {
          n4[0] = S[(w0 + na) * tj + j];
          n4[1] = S[(w0 + nb) * tj + j];
          n4[2] = S[(w0 + 3 + na) * tj + j];
          n4[3] = S[(w0 + 3 + nb) * tj + j];
        };
        double f[2][2];
        {
          double qn[2][4];
          nb4(6 * NC, qn[0]);
          nb4(6 * NC + 6, qn[1]);
          if (MODE == 2) {
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
              qn[cc][0] = qn[cc][0] + jm * mn[k][cc][0];
              qn[cc][1] = qn[cc][1] + jm * mn[k][cc][1];
              qn[cc][2] = qn[cc][2] + jm * mn[k][cc][0];
              qn[cc][3] = qn[cc][3] + jm * mn[k][cc][1];
            }
          }
          lat_factor(C, E[k], k, jm, qv, qn, f);
        }
        const double je = -(0.5 * C.el[k]);
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) {
          double n4[4], ti[2][2], te[2][2], x[2][2];
          nb4(cc * 6, n4);
          tr_own(u[cc], k, ti);
          tr_nb(n4, te);
#pragma unroll
          for (int vv = 0; vv < 2; ++vv)
#pragma unroll
            for (int h = 0; h < 2; ++h) x[vv][h] = (f[vv][h] >= 0.0 ? ti[vv][h] : te[vv][h]) * f[vv][h];
          if constexpr (MODE == 1) {   // both levels of edge node hn: sum_vh ES[h][hn] x[v][h]
            const double x0 = x[0][0] + x[1][0], x1 = x[0][1] + x[1][1];
            csum[cc][EV0(k)] += je * (ES[0][0] * x0 + ES[1][0] * x1);
            csum[cc][EV1(k)] += je * (ES[0][1] * x0 + ES[1][1] * x1);
          } else {
            lat_add(acc[cc], k, x, je);
          }
        }
      }
      if constexpr (NC >= 2 && MODE == 1 && RS) {
#pragma unroll
        for (int n = 0; n < 3; ++n) {
          ysum[0][n] += jm * (a.f * (u[1][n] + u[1][3 + n]));
          ysum[1][n] += jm * (-a.f * (u[0][n] + u[0][3 + n]));
        }
        if (l == 0) {
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            csum[0][k] += j2d / 6.0 * a.tsx;
            csum[1][k] += j2d / 6.0 * a.tsy;
          }
        }
        if (l == L - 1 && a.cd != 0.0) {   // bottom drag
          double dx3[3], dy3[3], mx[3], my[3];
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            const double ubx = u[0][3 + k], uby = u[1][3 + k];
            const double sp = sqrt(ubx * ubx + uby * uby);
            dx3[k] = -a.cd * sp * ubx;
            dy3[k] = -a.cd * sp * uby;
          }
          mh_apply3(dx3, j2d, mx);
          mh_apply3(dy3, j2d, my);
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            csum[0][k] += mx[k];
            csum[1][k] += my[k];
          }
        }
      }
      if constexpr (NC >= 2 && !(MODE == 1 && RS)) {
        double rr[2][6];
        ld6g(a.r, l, c, L, nt, rr[0]);
        ld6g(a.r + P6, l, c, L, nt, rr[1]);
        const double ir = 1.0 / a.rho0;
        if constexpr (MODE == 1) {
          // column sum of (K (x) J2D Mjz) y = J2D Mjz (y_top + y_bot); on sigma layers
          // Mjz = (f_b - f_t)/2 Mjz(H) = jm Mjz(H), so jm (y_top + y_bot) is summed over the
          // layers and J2D Mjz(H) applied once per column
#pragma unroll
          for (int n = 0; n < 3; ++n) {
            ysum[0][n] += jm * (a.f * (u[1][n] + u[1][3 + n]) - (rr[0][n] + rr[0][3 + n]) * ir);
            ysum[1][n] += jm * (-a.f * (u[0][n] + u[0][3 + n]) - (rr[1][n] + rr[1][3 + n]) * ir);
          }
          if (l == 0) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
              csum[0][k] += j2d / 6.0 * a.tsx;
              csum[1][k] += j2d / 6.0 * a.tsy;
            }
          }
        } else {
        double jz[3], Mu[3][3];
        layer_jz(C.b, eta, ft, fb, jz);
        mjz(jz, Mu);
        double y0[6], y1[6], m0[6], m1[6];
#pragma unroll
        for (int n = 0; n < 6; ++n) {
          y0[n] = a.f * u[1][n] - rr[0][n] * ir;
          y1[n] = -a.f * u[0][n] - rr[1][n] * ir;
        }
        kron_apply(Mu, j2d, y0, m0);
        kron_apply(Mu, j2d, y1, m1);
#pragma unroll
        for (int n = 0; n < 6; ++n) {
          acc[0][n] += m0[n];
          acc[1][n] += m1[n];
        }
        if (l == 0) {
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            acc[0][k] += j2d / 6.0 * a.tsx;
            acc[1][k] += j2d / 6.0 * a.tsy;
          }
        }
        }
        if (l == L - 1 && a.cd != 0.0) {
          double dx3[3], dy3[3], mx[3], my[3];
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            const double ubx = u[0][3 + k], uby = u[1][3 + k];
            const double sp = sqrt(ubx * ubx + uby * uby);
            dx3[k] = -a.cd * sp * ubx;
            dy3[k] = -a.cd * sp * uby;
          }
          mh_apply3(dx3, j2d, mx);
          mh_apply3(dy3, j2d, my);
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            if constexpr (MODE == 1) {
              csum[0][k] += mx[k];
              csum[1][k] += my[k];
            } else {
              acc[0][3 + k] += mx[k];
              acc[1][3 + k] += my[k];
            }
          }
        }
      }
      if constexpr (MODE != 1) {
        double j0[3], M0[3][3];
        layer_jz(C.b, eta0, ft, fb, j0);
        mjz(j0, M0);
        double mf[2][3] = {{0, 0, 0}, {0, 0, 0}};
        if constexpr (NC >= 2) {
          double j1[3], M1[3][3];
          layer_jz(C.b, eta1, ft, fb, j1);
          mjz(j1, M1);
          const double kk = (KM[0][0] + KM[0][1]) * j2d;
#pragma unroll
          for (int cc = 0; cc < 2; ++cc)
#pragma unroll
            for (int p = 0; p < 3; ++p)
              mf[cc][p] = kk * (M1[p][0] * F1[cc][0] + M1[p][1] * F1[cc][1] + M1[p][2] * F1[cc][2]);
        }
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) {
          double x0[6], m0x[6], o[6];
          ld6g(a.u0c[cc], l, c, L, nt, x0);
          kron_apply(M0, j2d, x0, m0x);
#pragma unroll
          for (int n = 0; n < 6; ++n) {
            if (NC >= 2 && cc < 2)
              o[n] = m0x[n] + a.dt * (acc[cc][n] + mf[cc][n % 3]);
            else
              o[n] = m0x[n] + a.dt * acc[cc][n];
          }
          st6(a.outc[cc], l, c, L, nt, o);
        }
      }
    }
    cp_async_wait0();
    __syncthreads();
  }
  if (MODE == 1 && act) {
#pragma unroll
    for (int cc = 0; cc < NC; ++cc)
#pragma unroll
      for (int p = 0; p < 3; ++p) csum[cc][p] += j2d * (C.dx[p] * sv[cc][0] + C.dy[p] * sv[cc][1]);
    if constexpr (NC >= 2) {
      if constexpr (RS) {
        const double ir = 1.0 / a.rho0;
#pragma unroll
        for (int d = 0; d < 2; ++d)
#pragma unroll
          for (int n = 0; n < 3; ++n) ysum[d][n] -= a.rsum[(d * 3 + n) * nt + c] * ir;
      }
      double H[3], MH[3][3];
#pragma unroll
      for (int k = 0; k < 3; ++k) H[k] = eta[k] - C.b[k];
      mjz(H, MH);
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        csum[0][p] += j2d * (MH[p][0] * ysum[0][0] + MH[p][1] * ysum[0][1] + MH[p][2] * ysum[0][2]);
        csum[1][p] += j2d * (MH[p][0] * ysum[1][0] + MH[p][1] * ysum[1][1] + MH[p][2] * ysum[1][2]);
      }
    }
#pragma unroll
    for (int cc = 0; cc < NC; ++cc)
#pragma unroll
      for (int k = 0; k < 3; ++k) out[(cc * 3 + k) * nt + c] = csum[cc][k];
  }
}

// Coriolis and -M r / rho0 over all prisms (the reference applies them to every row even
// when `els` restricts the advective part, internal3d.py:745-750)
__global__ void k_mass_terms(int L, int nt, const double* __restrict__ mass, const double* __restrict__ u,
                             const double* __restrict__ r, double f, double rho0, double* __restrict__ out) {
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long P = (long long)L * nt;
  if (p >= P) return;
  double M[6][6], uu[2][6], rr[2][6];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
#pragma unroll
    for (int j = 0; j < 6; ++j) M[i][j] = mass[(i * 6 + j) * P + p];
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      uu[cc][i] = u[(cc * 6 + i) * P + p];
      rr[cc][i] = r[(cc * 6 + i) * P + p];
    }
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    double mu0 = 0, mu1 = 0, mr0 = 0, mr1 = 0;
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      mu0 += M[i][j] * uu[0][j];
      mu1 += M[i][j] * uu[1][j];
      mr0 += M[i][j] * rr[0][j];
      mr1 += M[i][j] * rr[1][j];
    }
    double o0 = out[i * P + p], o1 = out[(6 + i) * P + p];
    if (f != 0.0) {
      o0 += f * mu1;
      o1 -= f * mu0;
    }
    out[i * P + p] = o0 - mr0 / rho0;
    out[(6 + i) * P + p] = o1 - mr1 / rho0;
  }
}

// stress_rhs (internal3d.py:919-934), API flavour
__global__ void k_stress(DMesh m, const double* __restrict__ ux, const double* __restrict__ uy, double tsx,
                         double tsy, double cd, Cols cs, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cs.n) return;
  const int c = cs.col(i), nt = m.nt, L = m.L;
  const size_t P6 = (size_t)6 * L * nt;
  const double j2d = ldg(m.j2d + c);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    out[((size_t)k * L + 0) * nt + c] += j2d / 6.0 * tsx;
    out[P6 + ((size_t)k * L + 0) * nt + c] += j2d / 6.0 * tsy;
  }
  if (cd != 0.0) {
    double dx3[3], dy3[3], mx[3], my[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double bx = ux[pix((3 + k), L - 1, c, L, nt)], by = uy[pix((3 + k), L - 1, c, L, nt)];
      const double sp = sqrt(bx * bx + by * by);
      dx3[k] = -cd * sp * bx;
      dy3[k] = -cd * sp * by;
    }
    mh_apply3(dx3, j2d, mx);
    mh_apply3(dy3, j2d, my);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      out[pix((3 + k), L - 1, c, L, nt)] += mx[k];
      out[P6 + pix((3 + k), L - 1, c, L, nt)] += my[k];
    }
  }
}

}  // namespace pdg

// ============================================================================ C ABI
using namespace pdg;

#define DISPATCH_MINB(key, KERNEL, ...)                                     \
  switch (tune_get(key)) {                                                 \
    case 3: KERNEL<__VA_ARGS__, 3><<<grid, blk, 0, strm>>>(LAUNCH_ARGS); break; \
    case 4: KERNEL<__VA_ARGS__, 4><<<grid, blk, 0, strm>>>(LAUNCH_ARGS); break; \
    default: KERNEL<__VA_ARGS__, 1><<<grid, blk, 0, strm>>>(LAUNCH_ARGS); break; \
  }

#define COLS(els, n) Cols{els, (els) ? (n) : ctx->nown}
#define GRID1(nn) nblocks((nn), 128), 128, 0, (cudaStream_t)stream

template <typename K>
static void set_smem(K kernel, size_t sm, size_t (&attr)[64]) {   // per device (the attribute is)
  int dev = 0;
  cudaGetDevice(&dev);
  if (sm > attr[dev & 63]) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr[dev & 63] = sm;
  }
}
template <int NC, int MODE, int TW>
static int launch_tile(pdg_ctx* ctx, const HArgs& a, double* out, cudaStream_t s) {
  const pdg_ctx::TileMap* tm = ensure_tiles(ctx, TW);
  if (!tm) return PDG_ERR_CUDA;
  const int tj = TW + tm->nh_max;
  const size_t sm = (size_t)2 * (6 * NC + 12) * tj * sizeof(double);
  static size_t attr[64] = {}, attr_rs[64] = {};
  set_smem(k_hrhs_t<NC, MODE, TW>, sm, attr);
  if constexpr (MODE == 1 && NC >= 2) set_smem(k_hrhs_t<NC, MODE, TW, true>, sm, attr_rs);
  StagePlanes sp{};
  const size_t P6 = (size_t)6 * ctx->L * ctx->nt, LN = (size_t)ctx->L * ctx->nt;
  for (int w = 0; w < 6 * NC + 12; ++w)
    sp.p[w] = (w < 6 * NC ? a.uc[w / 6] : a.qa + (size_t)((w - 6 * NC) / 6) * P6) + (size_t)(w % 6) * LN;
  if constexpr (MODE == 1 && NC >= 2) {
    if (a.rsum) {
      k_hrhs_t<NC, MODE, TW, true><<<nblocks(ctx->nown, TW), TW, sm, s>>>(ctx->view(), a, sp, tm->tslot, tm->halo,
                                                                        tm->hoff, tj, out);
      return PDG_OK;
    }
  }
  k_hrhs_t<NC, MODE, TW><<<nblocks(ctx->nown, TW), TW, sm, s>>>(ctx->view(), a, sp, tm->tslot, tm->halo, tm->hoff,
                                                              tj, out);
  return PDG_OK;
}

// planes of an NC-component prism field: word cc*6+node -> base + cc P6 + node L nt
static StagePlanes planes_of(const double* base, int nc, const pdg_ctx* ctx) {
  StagePlanes sp{};
  const size_t P6 = (size_t)6 * ctx->L * ctx->nt, LN = (size_t)ctx->L * ctx->nt;
  for (int w = 0; w < 6 * nc; ++w) sp.p[w] = base + (size_t)(w / 6) * P6 + (size_t)(w % 6) * LN;
  return sp;
}
template <bool FROM_T, int TW>
static int launch_r_tile(pdg_ctx* ctx, const double* eta_g, const double* rho, double alpha, double tref, double g,
                         double* r, cudaStream_t s, double* rsum = nullptr) {
  const pdg_ctx::TileMap* tm = ensure_tiles(ctx, TW);
  if (!tm) return PDG_ERR_CUDA;
  const int tj = TW + tm->nh_max;
  const size_t sm = ((size_t)2 * 6 * tj + ctx->L + 1) * sizeof(double) + (size_t)6 * TW * sizeof(int);
  static size_t attr[64] = {};
  set_smem(k_compute_r_t<FROM_T, TW>, sm, attr);
  k_compute_r_t<FROM_T, TW><<<nblocks(ctx->nown, TW), TW, sm, s>>>(ctx->view(), eta_g, alpha, tref, g,
                                                                 planes_of(rho, 1, ctx), tm->tslot, tm->halo,
                                                                 tm->hoff, tj, r, rsum);
  return PDG_OK;
}
template <int TW>
static int launch_wt_tile(pdg_ctx* ctx, const double* eta_g, const double* qb, const double* mis, double g, double* w,
                          cudaStream_t s) {
  const pdg_ctx::TileMap* tm = ensure_tiles(ctx, TW);
  if (!tm) return PDG_ERR_CUDA;
  const int tj = TW + tm->nh_max;
  const size_t sm = ((size_t)2 * 12 * tj + ctx->L + 1) * sizeof(double);
  static size_t attr[64] = {};
  set_smem(k_compute_wtilde_t<TW>, sm, attr);
  k_compute_wtilde_t<TW><<<nblocks(ctx->nown, TW), TW, sm, s>>>(ctx->view(), eta_g, mis, g, planes_of(qb, 2, ctx),
                                                              tm->tslot, tm->halo, tm->hoff, tj, w);
  return PDG_OK;
}


extern "C" {


int pdg_prism_mass(pdg_ctx* ctx, const double* eta_g, const int* els, int n_els, double* out, void* stream) {
  Cols cs = COLS(els, n_els);
  if (cs.n == 0) return PDG_OK;
  k_prism_mass<<<GRID1(cs.n)>>>(ctx->view(), eta_g, cs, out);
  return check_launch(ctx);
}

int pdg_project_transport(pdg_ctx* ctx, const double* eta_g, const double* ux, const double* uy,
                          const double* mass, const int* els, int n_els, double* q, double* qsum, double* htot,
                          void* stream) {
  Cols cs = COLS(els, n_els);
  if (cs.n == 0) return PDG_OK;
  if (mass)
    k_project<true><<<GRID1(cs.n)>>>(ctx->view(), eta_g, ux, uy, mass, cs, q, qsum, htot);
  else
    k_project<false><<<GRID1(cs.n)>>>(ctx->view(), eta_g, ux, uy, nullptr, cs, q, qsum, htot);
  return check_launch(ctx);
}

int pdg_column_sum(int nt, int L, int ncomp, const double* f, double* out, void* stream) {
  k_colsum<<<GRID1(nt)>>>(nt, L, ncomp, f, out);
  return check_launch_noctx();
}

int pdg_total_thickness(pdg_ctx* ctx, const double* eta_g, double* htot, void* stream) {
  k_htot<<<GRID1(ctx->nown)>>>(ctx->view(), eta_g, htot);
  return check_launch(ctx);
}

int pdg_mismatch(pdg_ctx* ctx, const double* qbar, const double* qsum, const double* htot, double* mis,
                 void* stream) {
  k_mismatch<<<GRID1(ctx->nown)>>>(ctx->nt, ctx->nown, qbar, qsum, htot, mis);
  return check_launch(ctx);
}

int pdg_consistent_transport(pdg_ctx* ctx, const double* eta_g, const double* q, const double* mis,
                             const int* els, int n_els, double* out, void* stream) {
  Cols cs = COLS(els, n_els);
  if (cs.n == 0) return PDG_OK;
  k_consistent<<<GRID1(cs.n)>>>(ctx->view(), eta_g, q, mis, cs, out);
  return check_launch(ctx);
}

int pdg_lateral_flux_factor(pdg_ctx* ctx, const double* eta_g, const double* q, double g, const int* els,
                            int n_els, double* fac, void* stream) {
  Cols cs = COLS(els, n_els);
  if (cs.n == 0) return PDG_OK;
  k_factor<<<GRID1(cs.n)>>>(ctx->view(), eta_g, q, g, cs, fac);
  return check_launch(ctx);
}

int pdg_compute_r(pdg_ctx* ctx, const double* eta_g, const double* rho_or_T, int from_T, double alpha, double tref,
                  double g, const int* els, int n_els, double* r, void* stream) {
  Cols cs = COLS(els, n_els);
  if (cs.n == 0) return PDG_OK;
  const dim3 grid(nblocks(cs.n, 128)), blk(128);
  cudaStream_t strm = (cudaStream_t)stream;
  if (const int tw = tune_get(TUNE_TILE_COL); !els && (tw == 64 || tw == 128)) {
    int rc;
    if (tw == 64)
      rc = from_T ? launch_r_tile<true, 64>(ctx, eta_g, rho_or_T, alpha, tref, g, r, strm)
                  : launch_r_tile<false, 64>(ctx, eta_g, rho_or_T, alpha, tref, g, r, strm);
    else
      rc = from_T ? launch_r_tile<true, 128>(ctx, eta_g, rho_or_T, alpha, tref, g, r, strm)
                  : launch_r_tile<false, 128>(ctx, eta_g, rho_or_T, alpha, tref, g, r, strm);
    if (rc) return rc;
    return check_launch(ctx);
  }
#define LAUNCH_ARGS ctx->view(), eta_g, rho_or_T, alpha, tref, g, cs, r
  if (from_T) {
    DISPATCH_MINB(TUNE_R, k_compute_r, true)
  } else {
    DISPATCH_MINB(TUNE_R, k_compute_r, false)
  }
#undef LAUNCH_ARGS
  return check_launch(ctx);
}

int pdg_compute_w(pdg_ctx* ctx, const double* eta_g, const double* q, const double* ux, const double* uy,
                  const double* fac, const int* els, int n_els, double* w, void* stream) {
  Cols cs = COLS(els, n_els);
  if (cs.n == 0) return PDG_OK;
  k_compute_w<<<GRID1(cs.n)>>>(ctx->view(), eta_g, q, ux, uy, fac, cs, w);
  return check_launch(ctx);
}

int pdg_compute_wtilde(pdg_ctx* ctx, const double* eta_g, const double* qb, const double* fac, const double* mis,
                       double g, const int* els, int n_els, double* w, void* stream) {
  Cols cs = COLS(els, n_els);
  if (cs.n == 0) return PDG_OK;
  const dim3 grid(nblocks(cs.n, 128)), blk(128);
  cudaStream_t strm = (cudaStream_t)stream;
  if (const int tw = tune_get(TUNE_TILE_COL); !els && mis && (tw == 64 || tw == 128)) {
    const int rc = tw == 64 ? launch_wt_tile<64>(ctx, eta_g, qb, mis, g, w, strm)
                            : launch_wt_tile<128>(ctx, eta_g, qb, mis, g, w, strm);
    if (rc) return rc;
    return check_launch(ctx);
  }
#define LAUNCH_ARGS ctx->view(), eta_g, qb, fac, mis, g, cs, w
  if (mis) {
    DISPATCH_MINB(TUNE_WT, k_compute_wtilde, true)
  } else {
    DISPATCH_MINB(TUNE_WT, k_compute_wtilde, false)
  }
#undef LAUNCH_ARGS
  return check_launch(ctx);
}

// horizontal_rhs / tracer_horizontal_rhs, API flavour (internal3d.py:695-792)
int pdg_horizontal_rhs(pdg_ctx* ctx, const double* eta_g, const double* u, int ncomp, const double* q_adv,
                       const double* fac, const double* r, const double* mass, double f, double rho0, int mass_terms,
                       const int* els, int n_els, double* out, void* stream) {
  Cols cs = COLS(els, n_els);
  if (cs.n == 0) return PDG_OK;
  HArgs a{};
  a.eta_u = eta_g;
  a.u = u;
  {
    const size_t P6 = (size_t)6 * ctx->L * ctx->nt;
    for (int cc = 0; cc < ncomp; ++cc) {
      a.uc[cc] = u + cc * P6;
      a.outc[cc] = out + cc * P6;
    }
  }
  a.qa = q_adv;
  a.fac = fac;
  a.r = r;
  a.mass = mass;
  a.f = f;
  a.rho0 = rho0;
  a.mass_terms = mass_terms;
  if (ncomp == 2)
    k_hrhs<2, 0, 1><<<GRID1(cs.n)>>>(ctx->view(), a, cs, out);
  else
    k_hrhs<1, 0, 1><<<GRID1(cs.n)>>>(ctx->view(), a, cs, out);
  return check_launch(ctx);
}

int pdg_mass_terms(int L, int nt, const double* mass, const double* u, const double* r, double f, double rho0,
                   double* out, void* stream) {
  const long long P = (long long)L * nt;
  k_mass_terms<<<nblocks(P, 128), 128, 0, (cudaStream_t)stream>>>(L, nt, mass, u, r, f, rho0, out);
  return check_launch_noctx();
}

int pdg_stress_rhs(pdg_ctx* ctx, const double* ux, const double* uy, double tsx, double tsy, double cd,
                   const int* els, int n_els, double* out, void* stream) {
  Cols cs = COLS(els, n_els);
  if (cs.n == 0) return PDG_OK;
  k_stress<<<GRID1(cs.n)>>>(ctx->view(), ux, uy, tsx, tsy, cd, cs, out);
  return check_launch(ctx);
}

// fused stepper entries ----------------------------------------------------------------
// F3D->2D forcing: column sum of horizontal_rhs(u, q, fac(q)) + stresses  -> [2][3][nt]
// rsum (optional, pdg_step_r): the per-column layer sum of jm (r_top + r_bot); used by the
// tile-staged kernel, which then loads no r
int pdg_step_f3d2d_rsum(pdg_ctx* ctx, const double* eta_u, const double* u, const double* q, const double* r,
                        const double* rsum, double g, double f, double rho0, double tsx, double tsy, double cd,
                        double* f3d2d, void* stream) {
  HArgs a{};
  a.rsum = rsum;
  a.eta_u = eta_u;
  a.u = u;
  {
    const size_t P6 = (size_t)6 * ctx->L * ctx->nt;
    a.uc[0] = u;
    a.uc[1] = u + P6;
  }
  a.qa = q;
  a.r = r;
  a.g = g;
  a.f = f;
  a.rho0 = rho0;
  a.tsx = tsx;
  a.tsy = tsy;
  a.cd = cd;
  Cols cs{nullptr, ctx->nown};
  const dim3 grid(nblocks(cs.n, 128)), blk(128);
  cudaStream_t strm = (cudaStream_t)stream;
#define LAUNCH_ARGS ctx->view(), a, cs, f3d2d
  if (const int tw = tune_get(TUNE_TILE_PRED); tw == 64 || tw == 128) {
    if ((tw == 64 ? launch_tile<2, 1, 64>(ctx, a, f3d2d, strm) : launch_tile<2, 1, 128>(ctx, a, f3d2d, strm)))
      return PDG_ERR_CUDA;
  } else if (tune_get(TUNE_HRHS) >= 8) {
    const int t = tune_get(TUNE_HRHS);
    if (t == 9)
      k_hrhs_s<2, 1, 6><<<nblocks(cs.n, 64), 64, 0, strm>>>(LAUNCH_ARGS);
    else if (t == 10)
      k_hrhs_s<2, 1, 8><<<nblocks(cs.n, 64), 64, 0, strm>>>(LAUNCH_ARGS);
    else
      k_hrhs_s<2, 1, 1><<<nblocks(cs.n, 64), 64, 0, strm>>>(LAUNCH_ARGS);
  } else {
    DISPATCH_MINB(TUNE_HRHS, k_hrhs, 2, 1)
  }
#undef LAUNCH_ARGS
  return check_launch(ctx);
}

int pdg_step_f3d2d(pdg_ctx* ctx, const double* eta_u, const double* u, const double* q, const double* r, double g,
                   double f, double rho0, double tsx, double tsy, double cd, double* f3d2d, void* stream) {
  return pdg_step_f3d2d_rsum(ctx, eta_u, u, q, r, nullptr, g, f, rho0, tsx, tsy, cd, f3d2d, stream);
}

// the stepper's baroclinic head from T (EOS inline) and, with the tile-staged kernel, the layer
// sum rsum [2][3][nt] the F3D->2D kernel takes instead of r; returns 1 in *rsum_written when it did
int pdg_step_r(pdg_ctx* ctx, const double* eta_g, const double* T, double alpha, double tref, double g, double* r,
               double* rsum, int* rsum_written, void* stream) {
  cudaStream_t strm = (cudaStream_t)stream;
  const int tw = tune_get(TUNE_TILE_COL);
  if (rsum_written) *rsum_written = 0;
  if (ctx->nown == 0) return PDG_OK;
  if (tw == 64 || tw == 128) {
    const int rc = tw == 64 ? launch_r_tile<true, 64>(ctx, eta_g, T, alpha, tref, g, r, strm, rsum)
                            : launch_r_tile<true, 128>(ctx, eta_g, T, alpha, tref, g, r, strm, rsum);
    if (rc) return rc;
    if (rsum_written) *rsum_written = rsum != nullptr;
    return check_launch(ctx);
  }
  return pdg_compute_r(ctx, eta_g, T, 1, alpha, tref, g, nullptr, 0, r, stream);
}

// stage right-hand sides: momentum  M0 u0 + dt (F(u, qbar) + stress + M1 F2D/H1),
// tracer M0 T0 + dt F(T, qbar)
int pdg_step_rhs(pdg_ctx* ctx, int ncomp, const double* eta_u, const double* eta0, const double* eta1,
                 const double* u, const double* u0, const double* q, const double* mis, const double* r,
                 const double* f2d, double g, double f, double rho0, double tsx, double tsy, double cd, double dt,
                 double* out, void* stream) {
  HArgs a{};
  a.eta_u = eta_u;
  a.eta0 = eta0;
  a.eta1 = eta1;
  a.u = u;
  a.u0 = u0;
  {
    const size_t P6 = (size_t)6 * ctx->L * ctx->nt;
    for (int cc = 0; cc < (ncomp == 1 ? 1 : 2); ++cc) {
      a.uc[cc] = u + cc * P6;
      a.u0c[cc] = u0 + cc * P6;
      a.outc[cc] = out + cc * P6;
    }
  }
  a.qa = q;
  a.mis = mis;
  a.r = r;
  a.f2d = f2d;
  a.g = g;
  a.f = f;
  a.rho0 = rho0;
  a.tsx = tsx;
  a.tsy = tsy;
  a.cd = cd;
  a.dt = dt;
  Cols cs{nullptr, ctx->nown};
  const dim3 grid(nblocks(cs.n, 128)), blk(128);
  cudaStream_t strm = (cudaStream_t)stream;
#define LAUNCH_ARGS ctx->view(), a, cs, out
  if (ncomp == 2) {
    DISPATCH_MINB(TUNE_HRHS2, k_hrhs, 2, 2)
  } else {
    DISPATCH_MINB(TUNE_HRHS2, k_hrhs, 1, 2)
  }
#undef LAUNCH_ARGS
  return check_launch(ctx);
}

// momentum AND tracer stage right-hand sides in one pass (they share q~, the flux factor and the
// masses): rhs_u = M0 u0 + dt (F_h(u, q~) + stress + M1 F2D/H1), rhs_T = M0 T0 + dt F_T(T, q~)
static int step_rhs_ut(pdg_ctx* ctx, const double* eta_u, const double* eta0, const double* eta1, const double* u,
                       const double* T, const double* u0, const double* T0, const double* q, const double* mis,
                       const double* r, const double* f2d, double g, double f, double rho0, double tsx, double tsy,
                       double cd, double dt, double* out_u, double* out_T, double* w, void* stream) {
  HArgs a{};
  a.wt = w;
  a.eta_u = eta_u;
  a.eta0 = eta0;
  a.eta1 = eta1;
  const size_t P6 = (size_t)6 * ctx->L * ctx->nt;
  a.uc[0] = u;
  a.uc[1] = u + P6;
  a.uc[2] = T;
  a.u0c[0] = u0;
  a.u0c[1] = u0 + P6;
  a.u0c[2] = T0;
  a.outc[0] = out_u;
  a.outc[1] = out_u + P6;
  a.outc[2] = out_T;
  a.qa = q;
  a.mis = mis;
  a.r = r;
  a.f2d = f2d;
  a.g = g;
  a.f = f;
  a.rho0 = rho0;
  a.tsx = tsx;
  a.tsy = tsy;
  a.cd = cd;
  a.dt = dt;
  Cols cs{nullptr, ctx->nown};
  const dim3 grid(nblocks(cs.n, 128)), blk(128);
  cudaStream_t strm = (cudaStream_t)stream;
#define LAUNCH_ARGS ctx->view(), a, cs, out_u
  const int tw = tune_get(TUNE_TILE_STAGE), hv = tune_get(TUNE_HRHS2);
  const bool same = a.u0c[0] == a.uc[0] && a.u0c[1] == a.uc[1] && a.u0c[2] == a.uc[2];
  if (w && tw != 64 && tw != 128 && hv == 8) {   // w~ inside the stage RHS (k_hrhs_s<..., WT>)
    if (same)
      k_hrhs_s<3, 2, 1, true, true><<<nblocks(cs.n, 64), 64, 0, strm>>>(LAUNCH_ARGS);
    else
      k_hrhs_s<3, 2, 1, false, true><<<nblocks(cs.n, 64), 64, 0, strm>>>(LAUNCH_ARGS);
    return check_launch(ctx);
  }
  if (w) {   // other stage-RHS variants: the separate w~ kernel first
    const int rc = pdg_compute_wtilde(ctx, eta_u, q, nullptr, mis, g, nullptr, 0, w, stream);
    if (rc) return rc;
  }
  if (tw == 64 || tw == 128) {
    if ((tw == 64 ? launch_tile<3, 2, 64>(ctx, a, out_u, strm) : launch_tile<3, 2, 128>(ctx, a, out_u, strm)))
      return PDG_ERR_CUDA;
  } else if (tune_get(TUNE_HRHS2) >= 8) {
    const int t = tune_get(TUNE_HRHS2);
    if (t == 9)
      k_hrhs_s<3, 2, 6><<<nblocks(cs.n, 64), 64, 0, strm>>>(LAUNCH_ARGS);
    else if (t == 10)
      k_hrhs_s<3, 2, 8><<<nblocks(cs.n, 64), 64, 0, strm>>>(LAUNCH_ARGS);
    else if (same)
      k_hrhs_s<3, 2, 1, true><<<nblocks(cs.n, 64), 64, 0, strm>>>(LAUNCH_ARGS);
    else
      k_hrhs_s<3, 2, 1><<<nblocks(cs.n, 64), 64, 0, strm>>>(LAUNCH_ARGS);
  } else {
    DISPATCH_MINB(TUNE_HRHS2, k_hrhs, 3, 2)
  }
#undef LAUNCH_ARGS
  return check_launch(ctx);
}

int pdg_step_rhs_ut(pdg_ctx* ctx, const double* eta_u, const double* eta0, const double* eta1, const double* u,
                    const double* T, const double* u0, const double* T0, const double* q, const double* mis,
                    const double* r, const double* f2d, double g, double f, double rho0, double tsx, double tsy,
                    double cd, double dt, double* out_u, double* out_T, void* stream) {
  return step_rhs_ut(ctx, eta_u, eta0, eta1, u, T, u0, T0, q, mis, r, f2d, g, f, rho0, tsx, tsy, cd, dt, out_u, out_T,
                     nullptr, stream);
}

// the same, and w~ of the stage (compute_wtilde with q~ = q + Jz mis, as pdg_compute_wtilde) into w
// [6][L][nt]: formed inside the stage-RHS layer loop (bottom-up), which already forms q~ and its
// lateral flux factor
int pdg_step_rhs_ut_w(pdg_ctx* ctx, const double* eta_u, const double* eta0, const double* eta1, const double* u,
                      const double* T, const double* u0, const double* T0, const double* q, const double* mis,
                      const double* r, const double* f2d, double g, double f, double rho0, double tsx, double tsy,
                      double cd, double dt, double* out_u, double* out_T, double* w, void* stream) {
  if (!w) return PDG_ERR_SHAPE;
  return step_rhs_ut(ctx, eta_u, eta0, eta1, u, T, u0, T0, q, mis, r, f2d, g, f, rho0, tsx, tsy, cd, dt, out_u, out_T,
                     w, stream);
}

}  // extern "C"

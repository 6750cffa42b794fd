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
// assemble_vertical_operator (internal3d.py:800-899) in factorised form.  Every block is a
// combination of symmetric 3x3 "face / layer masses" of the triangle rule:
//   R_l[a][b]   = sum_q QW BARY_a BARY_b / jzq_l(q)          (diffusion: dphi/dzeta products / Jz)
//   Sadv_m[a][b]= J2D sum_c T3[a][b][c] (K[m][0] dw_top[c] + K[m][1] dw_bot[c])   (advective volume)
//   F(x)[a][b]  = sum_q QW BARY_a BARY_b x(q)                 (upwinded face fluxes)
// so a layer costs ~400 FMAs instead of the ~1500 of the literal 12-point contractions.
struct VG {
  double R[3][3];  // symmetric
  double m2a, m2b; // |m_h/m_z|^2 at the two vertical points (kappa_i = kv + kh m2, internal3d.py:838)
  double tt, bb;   // |grad z_top|^2, |grad z_bot|^2                               (:875-876)
  double hgt;      // 2 mean(Jz)                                                   (:888)
  double rhgt;     // 1 / hgt (the penalty's 1/min(L_a, L_b) = max(1/L_a, 1/L_b))
  double nz;       // 1/sqrt(1 + |grad z_top|^2)                                   (:891)
};

// KH0: kh == 0 (the stepper: explicit horizontal diffusion is out of scope), so the slope terms
// m2a, m2b, bb only ever multiply zero and are not formed
template <bool KH0 = false>
__device__ __forceinline__ void vgeo(const Col& C, const double eta[3], double ft, double fb, VG& V) {
  LGeo G;
  if constexpr (KH0) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double H = __dsub_rn(eta[i], C.b[i]);
      G.zt[i] = __dsub_rn(eta[i], __dmul_rn(ft, H));
      G.zb[i] = __dsub_rn(eta[i], __dmul_rn(fb, H));
      G.jz[i] = __dmul_rn(0.5, __dsub_rn(G.zt[i], G.zb[i]));
    }
    G.dztop[0] = dot3_rn(G.zt, C.dx);
    G.dztop[1] = dot3_rn(G.zt, C.dy);
  } else {
    layer_geo(C, eta, ft, fb, G);
  }
  double jzq[6], ij[6];
  hq(G.jz, jzq);
#pragma unroll
  for (int q = 0; q < 6; ++q) ij[q] = KH0 ? QW[q] * drcp(jzq[q]) : QW[q] / jzq[q];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = a; b < 3; ++b) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < 6; ++q) s += ij[q] * (BARY[q][a] * BARY[q][b]);
      V.R[a][b] = s;
      V.R[b][a] = s;
    }
  if constexpr (KH0) {
    V.m2a = V.m2b = V.bb = 0.0;
  } else {
    const double mx = G.dzmid[0] + ZQP[0] * G.djz[0], my = G.dzmid[1] + ZQP[0] * G.djz[1];
    V.m2a = mx * mx + my * my;
    const double nx = G.dzmid[0] + ZQP[1] * G.djz[0], ny = G.dzmid[1] + ZQP[1] * G.djz[1];
    V.m2b = nx * nx + ny * ny;
    V.bb = G.dzbot[0] * G.dzbot[0] + G.dzbot[1] * G.dzbot[1];
  }
  const double tt = G.dztop[0] * G.dztop[0] + G.dztop[1] * G.dztop[1];
  V.tt = tt;
  V.hgt = ((G.jz[0] + G.jz[1]) + G.jz[2]) * (2.0 / 3.0);
  V.rhgt = KH0 ? drcp(V.hgt) : 1.0 / V.hgt;
  V.nz = KH0 ? drsqrt(1.0 + tt) : rsqrt(1.0 + tt);
}

// sigma layers: z = eta - f (eta - b), so Jz = (f_b - f_t) H / 2 at every point and the layer's
// diffusion mass is R_l = 2 / (f_b - f_t) Rc with the per-column Rc = sum_q QW BARY BARY / H(q),
// and the mean height 2 mean(Jz) = (f_b - f_t) sum(H) / 3.  k_vcol forms Rc (packed symmetric),
// sum(H) and 1 / sum(H) once per column and stage; the kh == 0 kernels then build a layer's
// geometry from them with 6 multiplications and one reciprocal instead of 6 reciprocals and the
// 6-point contractions (the values agree with vgeo to rounding).
constexpr int NVC = 8;
// momentum implicit solve (split forward elimination / back substitution) in the sigma form as
// well (-82 FP64 per layer, measured -2 %); the assembled explicit stage measured +1.5 % with it
#ifndef PDG_SIGU
#define PDG_SIGU 1
#endif
constexpr bool SIGU = PDG_SIGU != 0;
__global__ void k_vcol(DMesh m, const double* __restrict__ eta_u, double* __restrict__ vc,
                       const int* __restrict__ cols, int ncols) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int nt = m.nt;
  if (i >= (cols ? ncols : m.nown)) return;
  const int c = cols ? cols[i] : i;
  double H[3], hqv[6], ih[6];
#pragma unroll
  for (int k = 0; k < 3; ++k) H[k] = __dsub_rn(__ldg(eta_u + k * nt + c), __ldg(m.b + k * nt + c));
  hq(H, hqv);
#pragma unroll
  for (int q = 0; q < 6; ++q) ih[q] = QW[q] * drcp(hqv[q]);
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = a; b < 3; ++b) {
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < 6; ++q) acc += ih[q] * (BARY[q][a] * BARY[q][b]);
      vc[(a == b ? a : 2 + a + b) * nt + c] = acc;   // (0,0)0 (1,1)1 (2,2)2 (0,1)3 (0,2)4 (1,2)5
    }
  const double sh = (H[0] + H[1]) + H[2];
  vc[6 * nt + c] = sh;
  vc[7 * nt + c] = drcp(sh);
}
// the column constants are re-read every layer: keep their lines resident in L1
__device__ __forceinline__ double ldg_keep(const double* p) {
  double v;
  asm("ld.global.nc.L1::evict_last.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void vgeo_sigma(const Col& C, const double eta[3], double ft, double fb,
                                           const double* __restrict__ vc, int c, int nt, VG& V) {
  const double df = __dsub_rn(fb, ft);
  const double rdf = drcp(df);
  const double s2 = 2.0 * rdf;
  const double r00 = ldg_keep(vc + c), r11 = ldg_keep(vc + nt + c), r22 = ldg_keep(vc + 2 * nt + c);
  const double r01 = ldg_keep(vc + 3 * nt + c), r02 = ldg_keep(vc + 4 * nt + c), r12 = ldg_keep(vc + 5 * nt + c);
  V.R[0][0] = s2 * r00;
  V.R[1][1] = s2 * r11;
  V.R[2][2] = s2 * r22;
  V.R[0][1] = V.R[1][0] = s2 * r01;
  V.R[0][2] = V.R[2][0] = s2 * r02;
  V.R[1][2] = V.R[2][1] = s2 * r12;
  V.m2a = V.m2b = V.bb = 0.0;
  double zt[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) zt[i] = __dsub_rn(eta[i], __dmul_rn(ft, __dsub_rn(eta[i], C.b[i])));
  const double gx = dot3_rn(zt, C.dx), gy = dot3_rn(zt, C.dy);
  const double tt = gx * gx + gy * gy;
  V.tt = tt;
  V.hgt = df * ldg_keep(vc + 6 * nt + c) * (1.0 / 3.0);
  V.rhgt = 3.0 * rdf * ldg_keep(vc + 7 * nt + c);
  V.nz = drsqrt(1.0 + tt);
}
// the kh == 0 split kernels of the tracer (NC = 1) take the sigma form (their dispatcher always
// provides the constants); the momentum kernels are at the register limit, where the extra live
// values cost more than the saved FP64 work (measured), and keep vgeo.  The forward elimination and
// the back substitution of one solve use the same form (the rebuilt coupling blocks match bitwise).
template <bool KH0, bool SIG>
__device__ __forceinline__ void vgeo_x(const Col& C, const double eta[3], double ft, double fb, const double* vc,
                                       int c, int nt, VG& V) {
  if constexpr (KH0 && SIG)
    vgeo_sigma(C, eta, ft, fb, vc, c, nt, V);
  else
    vgeo<KH0>(C, eta, ft, fb, V);
}

// interior penalty sigma (dg.py:161-173) with L = min(L_a, L_b): n0 (p+1)(p+3) / (2 3 L)
__device__ __forceinline__ double pen_sigma(const VG& A, const VG& B, double n0, int order, pdg_err* err) {
  const double lmin = fmin(A.hgt, B.hgt);
  if (lmin <= 0.0) report(err, PDG_ERR_NONPOS_LENGTH, 0, 0, lmin);
  return n0 * ((order + 1.0) * (order + 3.0) / 6.0) * fmax(A.rhgt, B.rhgt);
}


// F(x) for x at the 6 points, symmetric
__device__ __forceinline__ void face3(const double x[6], double F[3][3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = a; b < 3; ++b) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < 6; ++q) s += (QW[q] * BARY[q][a] * BARY[q][b]) * x[q];
      F[a][b] = s;
      F[b][a] = s;
    }
}

// per-layer factorised pieces of A: the advective part (shared by momentum and tracer) ...
struct VAdv {
  double Sa[2][3][3];   // advective volume per column level m (d[i][j] += DV[li] Sa[lj][ai][aj])
  double Ft[3][3];      // top face: pos part (whole speed at the surface)      -> d top-top (-)
  double Fn[3][3];      // top face: neg part (l >= 1)                           -> u[:,3:6] (-)
  double Fi[3][3];      // bottom face: inflow part (l <= L-2)                   -> d bot-bot (+)
  double Fo[3][3];      // bottom face: outflow part                             -> w[:,0:3] (+)
};
// ... and the diffusive part, one per (kh, kv)
struct VDif {
  double cvol;          // J2D * kis                (diffusion volume coefficient on R_l)
  double ct, ca;        // 0.5 J2D kt_l (on R_l), 0.5 J2D kb_{l-1} (on R_{l-1})  (top face, l >= 1)
  double cb, cn;        // 0.5 J2D kb_l (on R_l), 0.5 J2D kt_{l+1} (on R_{l+1})  (bottom face, l <= L-2)
  double pt, pb;        // 0.5 x penalty factor of the top / bottom face
};
struct VPieces : VAdv, VDif {};


// The same pieces pre-multiplied by a scale (the implicit elimination passes c = -dt, so every
// block entry of M1 - dt A is one FMA chain without the final -dt multiplication): Sa comes out
// as scale/2 * Sa (the 1/2 of DV folded in), the face masses as scale * F.
__device__ __forceinline__ void vop_adv_vol_s(double sj, const double wt[6], const double wm[6], double Sa[2][6]) {
  double dwt[3], dwb[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    dwt[c] = wt[c] - wm[c];
    dwb[c] = wt[3 + c] - wm[3 + c];
  }
  const double hs = 0.5 * sj;
#pragma unroll
  for (int mm = 0; mm < 2; ++mm) {
    double y[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) y[c] = hs * (KM[mm][0] * dwt[c] + KM[mm][1] * dwb[c]);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = a; b < 3; ++b) Sa[mm][sym6(a, b)] = T3[a][b][0] * y[0] + T3[a][b][1] * y[1] + T3[a][b][2] * y[2];
  }
}
// face mass of the positive part of a P1 speed s = a - b given at the corners (packed symmetric)
__device__ __forceinline__ void face_pos_s(double sj, const double e3[3], double F[6]) {
  double sp[6], sq[6];
  hq(e3, sp);
#pragma unroll
  for (int q = 0; q < 6; ++q) sq[q] = sj * (sp[q] > 0.0 ? sp[q] : 0.0);
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = a; b < 3; ++b) {
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < 6; ++q) acc += (QW[q] * BARY[q][a] * BARY[q][b]) * sq[q];
      F[sym6(a, b)] = acc;
    }
}
// scaled bottom face of layer l < L-1: Fo (outflow, point-wise positive part), Fi = whole - Fo
__device__ __forceinline__ void vop_adv_bot_s(double sj, const double wm[6], const double wtn[3], double Fo[6],
                                              double Fi[6]) {
  double e3[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) e3[c] = wtn[c] - wm[3 + c];
  face_pos_s(sj, e3, Fo);
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = a; b < 3; ++b)
      Fi[sym6(a, b)] = sj * (T3[a][b][0] * e3[0] + T3[a][b][1] * e3[1] + T3[a][b][2] * e3[2]) - Fo[sym6(a, b)];
}
// scaled surface face (l == 0): the whole speed
__device__ __forceinline__ void vop_adv_surf_s(double sj, const double wt[6], const double wm[6], double Ft[6]) {
  double sp[6], d3[3] = {wt[0] - wm[0], wt[1] - wm[1], wt[2] - wm[2]};
  hq(d3, sp);
#pragma unroll
  for (int q = 0; q < 6; ++q) sp[q] = sj * sp[q];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = a; b < 3; ++b) {
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < 6; ++q) acc += (QW[q] * BARY[q][a] * BARY[q][b]) * sp[q];
      Ft[sym6(a, b)] = acc;
    }
}

__device__ __forceinline__ void vop_adv(double j2d, int l, int L, const double wt[6], const double wm[6],
                                        const double wtn[3], VAdv& P) {
  double dwt[3], dwb[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    dwt[c] = wt[c] - wm[c];
    dwb[c] = wt[3 + c] - wm[3 + c];
  }
#pragma unroll
  for (int mm = 0; mm < 2; ++mm) {
    double y[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) y[c] = j2d * (KM[mm][0] * dwt[c] + KM[mm][1] * dwb[c]);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = a; b < 3; ++b) {
        const double s = T3[a][b][0] * y[0] + T3[a][b][1] * y[1] + T3[a][b][2] * y[2];
        P.Sa[mm][a][b] = s;
        P.Sa[mm][b][a] = s;
      }
  }
  // The sign-split parts sum to the whole (P1) speed whose face mass is exact in closed form, so
  // only the positive parts are integrated point-wise: F(neg) = F(whole) - F(pos).
  {
    double sp[6], spos[6];
    double d3[3] = {wt[0] - wm[0], wt[1] - wm[1], wt[2] - wm[2]};
    hq(d3, sp);
#pragma unroll
    for (int q = 0; q < 6; ++q) spos[q] = j2d * (l == 0 ? sp[q] : (sp[q] >= 0.0 ? sp[q] : 0.0));
    face3(spos, P.Ft);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = a; b < 3; ++b) {
        const double w = l == 0 ? P.Ft[a][b] : j2d * (T3[a][b][0] * d3[0] + T3[a][b][1] * d3[1] + T3[a][b][2] * d3[2]);
        P.Fn[a][b] = w - P.Ft[a][b];
        P.Fn[b][a] = P.Fn[a][b];
      }
    if (l < L - 1) {
      double a3[6], b3[6], sout[6], e3[3];
      hq(wtn, a3);
      hq(wm + 3, b3);
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const double sb = a3[q] - b3[q];
        sout[q] = j2d * (sb > 0.0 ? sb : 0.0);
      }
      face3(sout, P.Fo);
#pragma unroll
      for (int c = 0; c < 3; ++c) e3[c] = wtn[c] - wm[3 + c];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = a; b < 3; ++b) {
          const double w = j2d * (T3[a][b][0] * e3[0] + T3[a][b][1] * e3[1] + T3[a][b][2] * e3[2]);
          P.Fi[a][b] = w - P.Fo[a][b];
          P.Fi[b][a] = P.Fi[a][b];
        }
    } else {
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          P.Fi[a][b] = 0.0;
          P.Fo[a][b] = 0.0;
        }
    }
  }
}

__device__ __forceinline__ void vop_dif(double j2d, int l, int L, const VG& Vp, const VG& V, const VG& Vn, double kh,
                                        double kv, double n0, int order, pdg_err* err, VDif& P) {
  const double kis = (kv + kh * V.m2a) + (kv + kh * V.m2b);
  const double kt = kv + kh * V.tt, kb = kv + kh * V.bb;
  const double kbp = kv + kh * Vp.bb, ktn = kv + kh * Vn.tt;
  P.cvol = j2d * kis;
  P.ct = 0.5 * j2d * kt;
  P.ca = 0.5 * j2d * kbp;
  P.cb = 0.5 * j2d * kb;
  P.cn = 0.5 * j2d * ktn;
  P.pt = l > 0 ? 0.5 * (pen_sigma(V, Vp, n0, order, err) * fmax(kt, kbp) * V.nz * j2d) : 0.0;
  P.pb = l < L - 1 ? 0.5 * (pen_sigma(Vn, V, n0, order, err) * fmax(ktn, kb) * Vn.nz * j2d) : 0.0;
}

__device__ __forceinline__ void vop_pieces(double j2d, int l, int L, const VG& Vp, const VG& V, const VG& Vn,
                                           const double wt[6], const double wm[6], const double wtn[3], double kh,
                                           double kv, double n0, int order, pdg_err* err, VPieces& P) {
  vop_adv(j2d, l, L, wt, wm, wtn, P);
  vop_dif(j2d, l, L, Vp, V, Vn, kh, kv, n0, order, err, P);
}

// explicit blocks of layer l: d (6x6), u (3x6, to layer l-1), w (3x6, to layer l+1)
__device__ __forceinline__ void vop_blocks(int l, int L, const VG& Vp, const VG& V, const VG& Vn, const VAdv& A,
                                           const VDif& D, double d[6][6], double u[3][6], double w[3][6]) {
  struct {
    const double (&Sa)[2][3][3];
    const double (&Ft)[3][3];
    const double (&Fn)[3][3];
    const double (&Fi)[3][3];
    const double (&Fo)[3][3];
    double cvol, ct, ca, cb, cn, pt, pb;
  } P{A.Sa, A.Ft, A.Fn, A.Fi, A.Fo, D.cvol, D.ct, D.ca, D.cb, D.cn, D.pt, D.pb};
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      const int li = i / 3, lj = j / 3, a = i % 3, b = j % 3;
      double v = DV[li] * P.Sa[lj][a][b] - DV[li] * DV[lj] * P.cvol * V.R[a][b];
      if (li == 0 && lj == 0) v -= P.Ft[a][b] + P.pt * MHQ[a][b];
      if (li == 1 && lj == 1) v += P.Fi[a][b] - P.pb * MHQ[a][b];
      if (li == 0 && l > 0) v += DV[lj] * P.ct * V.R[a][b];
      if (li == 1 && l < L - 1) v -= DV[lj] * P.cb * V.R[a][b];
      d[i][j] = v;
    }
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      const int lj = j / 3, b = j % 3;
      double uu = 0.0, ww = 0.0;
      if (l > 0) {
        uu = DV[lj] * P.ca * Vp.R[a][b];
        if (lj == 1) uu += P.pt * MHQ[a][b] - P.Fn[a][b];
      }
      if (l < L - 1) {
        ww = -DV[lj] * P.cn * Vn.R[a][b];
        if (lj == 0) ww += P.Fo[a][b] + P.pb * MHQ[a][b];
      }
      u[a][j] = uu;
      w[a][j] = ww;
    }
}

__device__ __forceinline__ void mv3(const double M[3][3], const double x[3], double y[3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a) y[a] = M[a][0] * x[0] + M[a][1] * x[1] + M[a][2] * x[2];
}


struct VopArgs {
  const double* eta_u;  // grid the operator is assembled on (C3)
  const double* wt;     // w~ (P6)
  const double* wm;     // w_m (P6) when given explicitly (API); else from eta0/eta1
  const double* eta0;   // fused: mesh velocity (z(eta1) - z(eta0)) / dtm
  const double* eta1;   //        and M1 = mass(eta1)
  double dtm, rdtm;     // mesh-velocity step and its reciprocal
  double kh, kv, n0;
  int order;
  const double* vc = nullptr;  // kh == 0 kernels: per-column sigma constants [8][nt] (k_vcol)
  // stepper kernels: optional column list (partitioned runs: boundary columns first, so the
  // ring-1 exchange of the result overlaps the interior columns); null = all owned columns
  const int* cols = nullptr;
  int ncols = 0;
  __device__ __forceinline__ int ncol(const DMesh& m) const { return cols ? ncols : m.nown; }
  __device__ __forceinline__ int col(int i) const { return cols ? cols[i] : i; }
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
    wm[i] = (zt1 - zt0) * a.rdtm;
    wm[3 + i] = (zb1 - zb0) * a.rdtm;
  }
}

// node values of w_m at layer l on sigma layers: z = (1 - f) eta + f b, so z(eta1) - z(eta0) =
// (1 - f)(eta1 - eta0) exactly and w_m = (1 - f) (eta1 - eta0) / dtm (b cancels; the reference's
// difference of two depths agrees to rounding).  The stepper's vertical kernels.
__device__ __forceinline__ void wm_sigma(const VopArgs& a, const double e0[3], const double e1[3], double ft,
                                         double fb, double wm[6]) {
  const double gt = 1.0 - ft, gb = 1.0 - fb;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double d = (e1[i] - e0[i]) * a.rdtm;
    wm[i] = gt * d;
    wm[3 + i] = gb * d;
  }
}

// assemble_vertical_operator (API): writes d [36][L][n], u/w [18][L][n] (compact over els)
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
  VG Vp, V, Vn;
  vgeo(C, eta, m.fracs[0], m.fracs[1], V);
  Vp = V;
  Vn = V;
  for (int l = 0; l < L; ++l) {
    if (l < L - 1) vgeo(C, eta, m.fracs[l + 1], m.fracs[l + 2], Vn);
    double wt[6], wm[6], wtn[3] = {0, 0, 0};
    ld6(a.wt, l, c, L, nt, wt);
    wm_layer(a, C.b, nullptr, nullptr, 0, 0, l, c, L, nt, wm);
    if (l < L - 1) {
#pragma unroll
      for (int k = 0; k < 3; ++k) wtn[k] = a.wt[pix(k, l + 1, c, L, nt)];
    }
    VPieces P;
    vop_pieces(C.j2d, l, L, Vp, V, Vn, wt, wm, wtn, a.kh, a.kv, a.n0, a.order, m.err, P);
    double d[6][6], u[3][6], w[3][6];
    vop_blocks(l, L, Vp, V, Vn, P, P, d, u, w);
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

// the same elimination without early exit and with branch-free reciprocals; returns the first
// zero pivot or -1 (the caller reports it and abandons the column)
__device__ __forceinline__ int lu6r_bf(double a[6][6], double rp[6]) {
  int bad = -1;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    bad = (bad < 0 && a[k][k] == 0.0) ? k : bad;
    const double inv = drcp(a[k][k]);
    rp[k] = inv;
#pragma unroll
    for (int i = k + 1; i < 6; ++i) {
      a[i][k] = a[i][k] * inv;
#pragma unroll
      for (int j = k + 1; j < 6; ++j) a[i][j] = a[i][j] - a[i][k] * a[k][j];
    }
  }
  return bad;
}
template <int NR>
__device__ __forceinline__ void lu6r_solve(const double a[6][6], const double rp[6], double b[6][NR]) {
#pragma unroll
  for (int i = 1; i < 6; ++i)
#pragma unroll
    for (int j = 0; j < i; ++j)
#pragma unroll
      for (int r = 0; r < NR; ++r) b[i][r] = b[i][r] - a[i][j] * b[j][r];
#pragma unroll
  for (int i = 5; i >= 0; --i) {
#pragma unroll
    for (int j = i + 1; j < 6; ++j)
#pragma unroll
      for (int r = 0; r < NR; ++r) b[i][r] = b[i][r] - a[i][j] * b[j][r];
#pragma unroll
    for (int r = 0; r < NR; ++r) b[i][r] = b[i][r] * rp[i];
  }
}

// ============================================================================ split block Thomas
// IMPLICIT: (M1 - dt A) x = rhs by block Thomas (columns.py:292-348 order) with the layer blocks
// assembled in registers; the propagation tile is kept in factored, compact form (workspace) and
// the back substitution is its own streaming kernel; the reduced RHS g_l is parked in x.
//
// The coupling of layer l to layer l+1 is [0; W_l] with W_l = -dt w_l (3x6) and, from
// vop_blocks, w_l = [Fo + pb MHQ - DV0 cn R_{l+1}, -DV1 cn R_{l+1}] (all 3x3 blocks symmetric).
// With S0 = -dt (Fo + pb MHQ), S1 = -dt cn R_{l+1}:
//     W_l x = S0 x_top - S1 (DV0 x_top + DV1 x_bot)
// so G_l = Dt_l^-1 [0; W_l] = E_l W_l with E_l = Dt_l^-1 [0; I3] (6x3).  The tile is
// (E_l 18, S0 6, S1 6) = 30 doubles instead of 36, and forming E_l needs 3 (not 6) solves.
// Tile layout: [l][30][nt] (one coalesced 8-byte word per lane per element).
constexpr int VT = 30;
constexpr int VBLK = 128;



// Per-thread column constants parked in shared memory and re-read (volatile) inside the layer
// loop: J2D, grad phi, bed and the three free surfaces are used every layer but would otherwise
// pin ~40 registers for the whole loop and get spilled to local memory by the 255-register
// vertical kernels (the spill reloads were their main long-scoreboard stall).
constexpr int NCS = 19;
__device__ __forceinline__ void cs_put(double* cs, int t, const Col& C, const double eta[3], const double e0[3],
                                       const double e1[3]) {
  cs[t] = C.j2d;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    cs[(1 + k) * VBLK + t] = C.dx[k];
    cs[(4 + k) * VBLK + t] = C.dy[k];
    cs[(7 + k) * VBLK + t] = C.b[k];
    cs[(10 + k) * VBLK + t] = eta[k];
    cs[(13 + k) * VBLK + t] = e0[k];
    cs[(16 + k) * VBLK + t] = e1[k];
  }
}
__device__ __forceinline__ void cs_get(const double* csp, int t, Col& C, double eta[3], double e0[3], double e1[3]) {
  const volatile double* cs = csp;
  C.j2d = cs[t];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    C.dx[k] = cs[(1 + k) * VBLK + t];
    C.dy[k] = cs[(4 + k) * VBLK + t];
    C.b[k] = cs[(7 + k) * VBLK + t];
    eta[k] = cs[(10 + k) * VBLK + t];
    e0[k] = cs[(13 + k) * VBLK + t];
    e1[k] = cs[(16 + k) * VBLK + t];
  }
}


// FORWARD: assembles M1 - dt A per layer, eliminates, writes the compact tile and g_l (into x).
// Per-layer inputs (rhs NC x 6, w~ 6) stream through a 3-deep cp.async ring in shared memory
// (each thread stages and reads only its own words: no barriers), issued two layers ahead;
// the previous layer's tile lives in shared memory, not in registers or L2.
//
// BULK (nt even): the ring is filled by the copy engine instead -- per layer one thread issues NE
// cp.async.bulk copies of the block's contiguous plane segments (1 KB each) completing on the
// slot's mbarrier; the threads wait on it, and one __syncthreads per layer frees the slot read two
// layers earlier (threads past the owned range stay for the barriers).
template <int NC, int MINB, bool KH0, bool CT = false, bool BULK = false>
__global__ void __launch_bounds__(VBLK, MINB) k_vimpl_fwd(DMesh m, VopArgs a, double dt, const double* rhs,
                                                        double* __restrict__ Gs, double* x) {
  
  constexpr int NE = 6 * NC + 6;  // staged words per layer: rhs, w~
  extern __shared__ double smem[];
  double* ring = smem;                       // [3][NE][VBLK]
  double* tl = smem + 3 * NE * VBLK;         // [VT][VBLK]
  double* cst = tl + VT * VBLK;              // [NCS][VBLK] column constants
  double* fr = cst + NCS * VBLK;             // [L+1]
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(fr + m.L + 1);   // [3] (BULK)
  const int t = threadIdx.x;
  // BULK: every thread runs the layer loop (the block barriers must be met by all of them, also
  // inside a warp); threads past the owned range repeat the last owned column and store nothing
  const int nc = a.ncol(m);
  const bool act = blockIdx.x * VBLK + t < nc;
  const int c = a.col(act ? blockIdx.x * VBLK + t : nc - 1);
  const int nt = m.nt, L = m.L;
  const int c0 = blockIdx.x * VBLK;
  for (int i = t; i <= L; i += VBLK) fr[i] = m.fracs[i];
  if (BULK && t == 0) {
#pragma unroll
    for (int k = 0; k < 3; ++k) mbar_init(bars + k, 1);
    mbar_init_fence();
  }
  __syncthreads();
  if (!BULK && !act) return;
  const size_t P6 = (size_t)6 * L * nt;
  // 16-byte multiple of the block's owned columns (nt even: at most one column past nown, < nt)
  const unsigned seg = (unsigned)(min(VBLK, m.nown - c0) * 8 + 15) & ~15u;
  // plane stride hidden from the optimiser (see k_vexpl3)
  auto stage = [&](int l) {
    if (BULK) {
      if (t == 0 && l < L) {
        unsigned long long* bar = bars + l % 3;
        const unsigned ln = (unsigned)L * (unsigned)nt, lo = (unsigned)l * (unsigned)nt + (unsigned)c0;
        double* s = ring + (l % 3) * NE * VBLK;
        fence_proxy_async();
        mbar_expect_tx(bar, NE * seg);
#pragma unroll
        for (int cc = 0; cc < NC; ++cc)
#pragma unroll
          for (int i = 0; i < 6; ++i) bulk_g2s(s + (cc * 6 + i) * VBLK, rhs + cc * P6 + (i * ln + lo), seg, bar);
#pragma unroll
        for (int i = 0; i < 6; ++i) bulk_g2s(s + (6 * NC + i) * VBLK, a.wt + (i * ln + lo), seg, bar);
      }
      return;
    }
    if (l < L) {
      unsigned ln = (unsigned)L * (unsigned)nt;
      asm volatile("" : "+r"(ln));
      const unsigned lo = (unsigned)l * (unsigned)nt + (unsigned)c;
      double* s = ring + (l % 3) * NE * VBLK + t;
#pragma unroll
      for (int cc = 0; cc < NC; ++cc)
#pragma unroll
        for (int i = 0; i < 6; ++i) cp_async8(s + (cc * 6 + i) * VBLK, rhs + cc * P6 + (i * ln + lo));
#pragma unroll
      for (int i = 0; i < 6; ++i) cp_async8(s + (6 * NC + i) * VBLK, a.wt + (i * ln + lo));
    }
    cp_async_commit();
  };
  stage(0);
  stage(1);
  Col C;
  load_col(m, c, C);
  double eta[3], e0[3], e1[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    eta[k] = a.eta_u[k * nt + c];
    e0[k] = a.eta0[k * nt + c];
    e1[k] = a.eta1[k * nt + c];
  }
  cs_put(cst, t, C, eta, e0, e1);
  VG Vp, V, Vn;
  vgeo_x<KH0, (NC == 1 || SIGU)>(C, eta, fr[0], fr[1], a.vc, c, nt, V);
  Vp = V;
  Vn = V;
  double gp[6][NC];
  for (int l = 0; l < L; ++l) {
    if (BULK) __syncthreads();   // every thread is done with layer l-1: its slot may be refilled
    cs_get(cst, t, C, eta, e0, e1);
    const double j2d = C.j2d;
    stage(l + 2);
    if (BULK) {                  // layers l and l+1 have landed
      mbar_wait(bars + l % 3, (unsigned)(l / 3) & 1u);
      if (l + 1 < L) mbar_wait(bars + (l + 1) % 3, (unsigned)((l + 1) / 3) & 1u);
    } else {
      cp_async_wait1();
    }
    const double* cur = ring + (l % 3) * NE * VBLK + t;
    const double* nxt = ring + ((l + 1) % 3) * NE * VBLK + t;
    const double ft = fr[l], fb = fr[l + 1];
    if (l < L - 1) vgeo_x<KH0, (NC == 1 || SIGU)>(C, eta, fb, fr[l + 2], a.vc, c, nt, Vn);
    double wt[6], wm[6], wtn[3] = {0, 0, 0};
#pragma unroll
    for (int i = 0; i < 6; ++i) wt[i] = cur[(6 * NC + i) * VBLK];
    if constexpr (NC == 1)
      wm_sigma(a, e0, e1, ft, fb, wm);
    else   // (measured: the momentum forward elimination runs 1.7 % slower with wm_sigma)
      wm_layer(a, C.b, e0, e1, ft, fb, l, c, L, nt, wm);
    if (l < L - 1) {
#pragma unroll
      for (int k = 0; k < 3; ++k) wtn[k] = nxt[(6 * NC + k) * VBLK];
    }
    // Advective pieces scaled by c = -dt (every block entry of M1 - dt A is then one FMA chain),
    // with the interface face masses carried: the top face of layer l is the bottom face of layer
    // l-1 (same speed and mesh velocity), so Ft / Fn are that layer's Fo / Fi (tile words 18..29,
    // packed symmetric) and only the bottom face is integrated here.
    const double cdt = -dt, sj = cdt * j2d;
    double Sa[2][6], Ft[6], Fn[6], Fo[6], Fi[6];
    vop_adv_vol_s(sj, wt, wm, Sa);
    if (l == 0) {
      vop_adv_surf_s(sj, wt, wm, Ft);
#pragma unroll
      for (int k = 0; k < 6; ++k) Fn[k] = 0.0;
    } else {
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        Ft[k] = tl[(18 + k) * VBLK + t];
        Fn[k] = tl[(24 + k) * VBLK + t];
      }
    }
    if (l < L - 1) {
      vop_adv_bot_s(sj, wm, wtn, Fo, Fi);
    } else {
#pragma unroll
      for (int k = 0; k < 6; ++k) Fo[k] = Fi[k] = 0.0;
    }
    VDif D;
    vop_dif(j2d, l, L, Vp, V, Vn, a.kh, a.kv, a.n0, a.order, m.err, D);
    // M1 - dt A_d of layer l and the coupling U = -dt u to layer l-1 (vimpl_blocks, with the
    // -dt folded into the pieces): 24 entries of d, 12 of U (two symmetric blocks, packed)
    double d[6][6], Uc[2][6];
    {
      double jz1[3];
      layer_jz(C.b, e1, ft, fb, jz1);
      const double q4 = 0.25 * D.cvol;
      const double ht = l > 0 ? 0.5 * D.ct : 0.0, hb = l < L - 1 ? 0.5 * D.cb : 0.0;
      const double r00 = ht - q4, r01 = q4 - ht, r10 = q4 - hb, r11 = hb - q4;
      const double ptc = cdt * D.pt, pbc = cdt * D.pb, hca = 0.5 * cdt * D.ca;
#pragma unroll
      for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int q = p; q < 3; ++q) {
          const int k = sym6(p, q);
          const double m1 = j2d * (T3[p][q][0] * jz1[0] + T3[p][q][1] * jz1[1] + T3[p][q][2] * jz1[2]);
          const double Rc = cdt * V.R[p][q], mh = MHQ[p][q];
          const double v00 = KM[0][0] * m1 + (((Sa[0][k] + r00 * Rc) - Ft[k]) - ptc * mh);
          const double v01 = KM[0][1] * m1 + (Sa[1][k] + r01 * Rc);
          const double v10 = KM[1][0] * m1 + (r10 * Rc - Sa[0][k]);
          const double v11 = KM[1][1] * m1 + (((r11 * Rc - Sa[1][k]) + Fi[k]) - pbc * mh);
          d[p][q] = d[q][p] = v00;
          d[p][3 + q] = d[q][3 + p] = v01;
          d[3 + p][q] = d[3 + q][p] = v10;
          d[3 + p][3 + q] = d[3 + q][3 + p] = v11;
          const double u0 = hca * Vp.R[p][q];
          Uc[0][k] = u0;
          Uc[1][k] = (ptc * mh - Fn[k]) - u0;
        }
    }
    double g[6][NC];
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) g[i][cc] = cur[(cc * 6 + i) * VBLK];
    if (l > 0) {
      // Dt = D - U G_{l-1} = D - (U E_{l-1}) W_{l-1},  U = -dt u = [Uc0, Uc1]
      double Pm[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < 6; ++k) acc = acc + Uc[k / 3][sym6(i, k % 3)] * tl[(k * 3 + j) * VBLK + t];
          Pm[i][j] = acc;
        }
      // coupling of layer l-1 to l rebuilt from this layer's top-face pieces (the values layer l-1
      // would form: Fo_{l-1} = Ft_l, pb_{l-1} = pt_l, cn_{l-1} = ct_l, R_l):
      // S0 = -dt (Fo + pb MHQ), S1 = -dt cn R_l
      double S0[3][3], S1h[3][3];
      {
        const double ptc = cdt * D.pt, ctc = cdt * D.ct;
#pragma unroll
        for (int p = 0; p < 3; ++p)
#pragma unroll
          for (int q = p; q < 3; ++q) {
            const double s0 = Ft[sym6(p, q)] + ptc * MHQ[p][q];
            const double s1 = ctc * V.R[p][q];
            S1h[p][q] = S1h[q][p] = DV[1] * s1;    // W_bot = -DV1 S1  (sign folded below)
            S0[p][q] = S0[q][p] = s0 - DV[0] * s1; // W_top = S0 - DV0 S1
          }
      }
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          double at = 0.0, ab = 0.0;
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            at = at + Pm[i][k] * S0[k][j];
            ab = ab - Pm[i][k] * S1h[k][j];
          }
          d[i][j] = d[i][j] - at;
          d[i][3 + j] = d[i][3 + j] - ab;
        }
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) {
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < 6; ++k) acc = acc + Uc[k / 3][sym6(i, k % 3)] * gp[k][cc];
          g[i][cc] = g[i][cc] - acc;
        }
    }
    double rp[6];
    const int bad = lu6r_bf(d, rp);
    if (bad >= 0) {
      report(m.err, PDG_ERR_ZERO_PIVOT, l, bad, 0.0);
      if (!BULK) return;          // (BULK: keep meeting the block barriers; the step is void anyway)
    }
    lu6r_solve<NC>(d, rp, g);
    {
      unsigned ln = (unsigned)L * (unsigned)nt;
      asm volatile("" : "+r"(ln));
      const unsigned lo = (unsigned)l * (unsigned)nt + (unsigned)c;
#pragma unroll
      for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) {
          if (act) x[cc * P6 + (i * ln + lo)] = g[i][cc];
          gp[i][cc] = g[i][cc];
        }
    }
    if (l < L - 1) {
      // E = Dt^-1 [0; I3]: forward substitution starts at row 3
      constexpr int GT = CT ? 18 : VT;   // global tile words (CT: S0, S1 rebuilt by k_vimpl_bwd_r)
      double* gt = Gs + (size_t)l * GT * nt + c;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        double t3 = j == 0 ? 1.0 : 0.0, t4 = j == 1 ? 1.0 : 0.0, t5 = j == 2 ? 1.0 : 0.0;
        t4 = t4 - d[4][3] * t3;
        t5 = t5 - d[5][3] * t3 - d[5][4] * t4;
        double e[6];
        e[5] = t5 * rp[5];
        e[4] = (t4 - d[4][5] * e[5]) * rp[4];
        e[3] = (t3 - d[3][4] * e[4] - d[3][5] * e[5]) * rp[3];
        e[2] = (0.0 - d[2][3] * e[3] - d[2][4] * e[4] - d[2][5] * e[5]) * rp[2];
        e[1] = (0.0 - d[1][2] * e[2] - d[1][3] * e[3] - d[1][4] * e[4] - d[1][5] * e[5]) * rp[1];
        e[0] = (0.0 - d[0][1] * e[1] - d[0][2] * e[2] - d[0][3] * e[3] - d[0][4] * e[4] - d[0][5] * e[5]) * rp[0];
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          tl[(i * 3 + j) * VBLK + t] = e[i];
          if (act) gt[(size_t)(i * 3 + j) * nt] = e[i];
        }
      }
      // the bottom-face pieces become the next layer's top-face pieces (packed symmetric);
      // !CT: the global tile also holds S0 = -dt (Fo + pb MHQ), S1 = -dt cn R_{l+1}
#pragma unroll
      for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int q = p; q < 3; ++q) {
          const int k = sym6(p, q);
          tl[(18 + k) * VBLK + t] = Fo[k];
          tl[(24 + k) * VBLK + t] = Fi[k];
          if (!CT && act) {
            gt[(size_t)(18 + k) * nt] = Fo[k] + (cdt * D.pb) * MHQ[p][q];
            gt[(size_t)(24 + k) * nt] = D.cn * (cdt * Vn.R[p][q]);
          }
        }
    }
    Vp = V;
    V = Vn;
  }
}

// BACKWARD: x_l = g_l - E_l (W_l x_{l+1}), g_l parked in x by the forward kernel.  Pure
// streaming (30 + 6 NC words in, 6 NC out per prism), high occupancy.
template <int NC>
__global__ void __launch_bounds__(VBLK) k_vimpl_bwd(int nown, int nt, int L, const double* __restrict__ Gs,
                                                  double* x, const pdg_err* err, const int* __restrict__ cols) {
  const int i0 = blockIdx.x * VBLK + threadIdx.x;
  if (i0 >= nown || err->code == PDG_ERR_ZERO_PIVOT) return;
  const int c = cols ? cols[i0] : i0;
  const size_t P6 = (size_t)6 * L * nt;
  double xn[6][NC];
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) xn[i][cc] = x[cc * P6 + pix(i, L - 1, c, L, nt)];
  for (int l = L - 2; l >= 0; --l) {
    const double* gt = Gs + (size_t)l * VT * nt + c;
    double tv[VT];
#pragma unroll
    for (int e = 0; e < VT; ++e) tv[e] = gt[(size_t)e * nt];
    double gl[6][NC];
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) gl[i][cc] = x[cc * P6 + pix(i, l, c, L, nt)];
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) {
      double dz[3], y[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) dz[k] = DV[0] * xn[k][cc] + DV[1] * xn[3 + k][cc];
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < 3; ++q) acc = acc + tv[18 + sym6(p, q)] * xn[q][cc] - tv[24 + sym6(p, q)] * dz[q];
        y[p] = acc;
      }
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        const double v = gl[i][cc] - (tv[i * 3] * y[0] + tv[i * 3 + 1] * y[1] + tv[i * 3 + 2] * y[2]);
        x[cc * P6 + pix(i, l, c, L, nt)] = v;
        xn[i][cc] = v;
      }
    }
  }
}

// BACKWARD with the coupling rebuilt: the tile holds only E_l (18 words); S0 = -dt (Fo + pb MHQ)
// and S1 = -dt cn R_{l+1} are recomputed from the sigma geometry, w~ (top nodes of layer l+1) and
// the mesh velocity with the forward kernel's own functions -- 12 fewer words written and read
// per prism for ~200 FP64 operations in a kernel whose FP64 pipe is otherwise idle.
template <int NC>
__global__ void __launch_bounds__(VBLK, NC == 1 ? 3 : 1) k_vimpl_bwd_r(DMesh m, VopArgs a, double dt, const double* __restrict__ Gs,
                                                    double* x) {
  const int i0 = blockIdx.x * VBLK + threadIdx.x;
  const int nt = m.nt, L = m.L;
  if (i0 >= a.ncol(m) || m.err->code == PDG_ERR_ZERO_PIVOT) return;
  const int c = a.col(i0);
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
  VG Vu;  // geometry of layer l + 1
  vgeo_x<true, (NC == 1 || SIGU)>(C, eta, m.fracs[L - 1], m.fracs[L], a.vc, c, nt, Vu);
  double xn[6][NC];
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) xn[i][cc] = x[cc * P6 + pix(i, L - 1, c, L, nt)];
  for (int l = L - 2; l >= 0; --l) {
    const double* gt = Gs + (size_t)l * 18 * nt + c;
    double E[18];
#pragma unroll
    for (int e = 0; e < 18; ++e) E[e] = __ldg(gt + (size_t)e * nt);
    double gl[6][NC];
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) gl[i][cc] = x[cc * P6 + pix(i, l, c, L, nt)];
    double wtn[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) wtn[k] = __ldg(a.wt + pix(k, l + 1, c, L, nt));
    const double ft = m.fracs[l], fb = m.fracs[l + 1];
    VG Vl;
    vgeo_x<true, (NC == 1 || SIGU)>(C, eta, ft, fb, a.vc, c, nt, Vl);
    double wm[6];
    if constexpr (NC == 1)
      wm_sigma(a, e0, e1, ft, fb, wm);
    else   // (measured: the momentum forward elimination runs 1.7 % slower with wm_sigma)
      wm_layer(a, C.b, e0, e1, ft, fb, l, c, L, nt, wm);
    // Fo (bottom face of layer l, scaled by -dt as in the forward kernel) and the diffusion
    // pieces cn, pb (vop_dif): S0 = -dt (Fo + pb MHQ), S1 = -dt cn R_{l+1}
    const double cdt = -dt;
    double Fo[6];
    {
      double e3[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) e3[k] = wtn[k] - wm[3 + k];
      face_pos_s(cdt * j2d, e3, Fo);
    }
    const double kb = a.kv + a.kh * Vl.bb, ktn = a.kv + a.kh * Vu.tt;
    const double cn = 0.5 * j2d * ktn;
    const double pb = 0.5 * (pen_sigma(Vu, Vl, a.n0, a.order, m.err) * fmax(ktn, kb) * Vu.nz * j2d);
    const double pbc = cdt * pb, cnc = cdt * cn;
    double S0[3][3], S1[3][3];
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        S0[p][q] = Fo[sym6(p, q)] + pbc * MHQ[p][q];
        S1[p][q] = cnc * Vu.R[p][q];
      }
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) {
      double dz[3], y[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) dz[k] = DV[0] * xn[k][cc] + DV[1] * xn[3 + k][cc];
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < 3; ++q) acc = acc + S0[p][q] * xn[q][cc] - S1[p][q] * dz[q];
        y[p] = acc;
      }
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        const double v = gl[i][cc] - (E[i * 3] * y[0] + E[i * 3 + 1] * y[1] + E[i * 3 + 2] * y[2]);
        x[cc * P6 + pix(i, l, c, L, nt)] = v;
        xn[i][cc] = v;
      }
    }
    Vu = Vl;
  }
}

inline size_t vimpl_fwd_smem(int nc, int L) { return ((size_t)3 * (6 * nc + 6) * VBLK + (VT + NCS) * VBLK + L + 1 + 3) * 8; }

inline size_t vexpl3_smem(int nc, int L) { return ((size_t)3 * (12 * nc + 6) * VBLK + NCS * VBLK + L + 1 + (nc == 1 ? 12 * VBLK : 0)) * 8; }

// top face of layer l >= 1 (scaled): Ft (positive part, point-wise), Fn = whole - Ft
__device__ __forceinline__ void vop_adv_top_s(double sj, const double wt[6], const double wm[6], double Ft[6],
                                              double Fn[6]) {
  double d3[3] = {wt[0] - wm[0], wt[1] - wm[1], wt[2] - wm[2]};
  face_pos_s(sj, d3, Ft);
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = a; b < 3; ++b)
      Fn[sym6(a, b)] = sj * (T3[a][b][0] * d3[0] + T3[a][b][1] * d3[1] + T3[a][b][2] * d3[2]) - Ft[sym6(a, b)];
}
// y += M x for a packed symmetric 3x3 M
__device__ __forceinline__ void smv_add(const double M[6], const double x[3], double y[3]) {
  y[0] += M[0] * x[0] + M[3] * x[1] + M[4] * x[2];
  y[1] += M[3] * x[0] + M[1] * x[1] + M[5] * x[2];
  y[2] += M[4] * x[0] + M[5] * x[1] + M[2] * x[2];
}

// EXPLICIT, assembled: x = M1^-1 (rhs + dt A xin).  The blocks of dt A (the four 3x3 blocks of
// the diagonal block, the coupling U to layer l-1 and W to layer l+1 -- all symmetric, packed:
// vop_blocks' 72 entries as 48 words) are formed once per layer from the dt-scaled pieces and
// applied to every component (72 FMAs per component instead of ~180 for the matrix-free form).
// Per-layer inputs (rhs, xin, w~) stream through a 3-deep cp.async ring issued two layers ahead
// (each thread stages and reads only its own words); NC == 1 carries the interface face masses
// from the layer above in shared memory (FCS, see k_vimpl_fwd).  KH0: kh == 0 geometry.
template <int NC, int MINB, bool KH0>
__global__ void __launch_bounds__(VBLK, MINB) k_vexpl3(DMesh m, VopArgs a, double dt, const double* rhs,
                                                     const double* __restrict__ xin, double* x) {
  constexpr int NE = 12 * NC + 6;  // rhs, xin, w~
  extern __shared__ double smem[];
  double* ring = smem;             // [3][NE][VBLK]
  double* cst = smem + 3 * NE * VBLK;  // [NCS][VBLK] column constants
  double* fr = cst + NCS * VBLK;
  constexpr bool FCS = NC == 1;
  double* fc = fr + m.L + 1;       // [12][VBLK] carried face pieces (FCS)
  const int t = threadIdx.x;
  const int i0 = blockIdx.x * VBLK + t;
  const int nt = m.nt, L = m.L;
  for (int i = t; i <= L; i += VBLK) fr[i] = m.fracs[i];
  __syncthreads();
  if (i0 >= a.ncol(m)) return;
  const int c = a.col(i0);
  const size_t P6 = (size_t)6 * L * nt;
  auto stage = [&](int l) {
    if (l < L) {
      unsigned ln = (unsigned)L * (unsigned)nt;
      asm volatile("" : "+r"(ln));
      const unsigned lo = (unsigned)l * (unsigned)nt + (unsigned)c;
      double* s = ring + (l % 3) * NE * VBLK + t;
#pragma unroll
      for (int cc = 0; cc < NC; ++cc)
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const size_t o = cc * P6 + (i * ln + lo);
          cp_async8(s + (cc * 6 + i) * VBLK, rhs + o);
          cp_async8(s + (6 * NC + cc * 6 + i) * VBLK, xin + o);
        }
#pragma unroll
      for (int i = 0; i < 6; ++i) cp_async8(s + (12 * NC + i) * VBLK, a.wt + (i * ln + lo));
    }
    cp_async_commit();
  };
  stage(0);
  stage(1);
  Col C;
  load_col(m, c, C);
  double eta[3], e0[3], e1[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    eta[k] = a.eta_u[k * nt + c];
    e0[k] = a.eta0[k * nt + c];
    e1[k] = a.eta1[k * nt + c];
  }
  cs_put(cst, t, C, eta, e0, e1);
  constexpr double det = KM[0][0] * KM[1][1] - KM[0][1] * KM[1][0];
  constexpr double ki00 = KM[1][1] / det, ki01 = -KM[0][1] / det, ki10 = -KM[1][0] / det, ki11 = KM[0][0] / det;
  VG Vp, V, Vn;
  vgeo_x<KH0, NC == 1>(C, eta, fr[0], fr[1], a.vc, c, nt, V);
  Vp = V;
  Vn = V;
  double xa[NC][6];   // xin of layer l-1: its ring slot is refilled at the top of iteration l
  for (int l = 0; l < L; ++l) {
    cs_get(cst, t, C, eta, e0, e1);
    const double j2d = C.j2d;
    if (l > 0) {
      const double* prv = ring + ((l + 2) % 3) * NE * VBLK + t;
#pragma unroll
      for (int cc = 0; cc < NC; ++cc)
#pragma unroll
        for (int k = 0; k < 6; ++k) xa[cc][k] = prv[(6 * NC + cc * 6 + k) * VBLK];
    }
    stage(l + 2);
    cp_async_wait1();
    const double* cur = ring + (l % 3) * NE * VBLK + t;
    const double* nxt = ring + ((l + 1) % 3) * NE * VBLK + t;
    const double ft = fr[l], fb = fr[l + 1];
    if (l < L - 1) vgeo_x<KH0, NC == 1>(C, eta, fb, fr[l + 2], a.vc, c, nt, Vn);
    double wt[6], wm[6], wtn[3] = {0, 0, 0};
#pragma unroll
    for (int i = 0; i < 6; ++i) wt[i] = cur[(12 * NC + i) * VBLK];
    wm_sigma(a, e0, e1, ft, fb, wm);
    if (l < L - 1) {
#pragma unroll
      for (int k = 0; k < 3; ++k) wtn[k] = nxt[(12 * NC + k) * VBLK];
    }
    const double sj = dt * j2d;
    double Sa[2][6], Ft[6], Fn[6], Fo[6], Fi[6];
    vop_adv_vol_s(sj, wt, wm, Sa);
    if (l == 0) {
      vop_adv_surf_s(sj, wt, wm, Ft);
#pragma unroll
      for (int k = 0; k < 6; ++k) Fn[k] = 0.0;
    } else if (FCS) {
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        Ft[k] = fc[k * VBLK + t];
        Fn[k] = fc[(6 + k) * VBLK + t];
      }
    } else {
      vop_adv_top_s(sj, wt, wm, Ft, Fn);
    }
    if (l < L - 1) {
      vop_adv_bot_s(sj, wm, wtn, Fo, Fi);
      if (FCS) {
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          fc[k * VBLK + t] = Fo[k];
          fc[(6 + k) * VBLK + t] = Fi[k];
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < 6; ++k) Fo[k] = Fi[k] = 0.0;
    }
    VDif D;
    vop_dif(j2d, l, L, Vp, V, Vn, a.kh, a.kv, a.n0, a.order, m.err, D);
    // dt A: diagonal blocks B00, B01, B10, B11, coupling U0, U1 (layer l-1), W0, W1 (layer l+1)
    double B[4][6], U[2][6], W[2][6];
    {
      const double q4 = 0.25 * D.cvol;
      const double ht = l > 0 ? 0.5 * D.ct : 0.0, hb = l < L - 1 ? 0.5 * D.cb : 0.0;
      const double r00 = ht - q4, r01 = q4 - ht, r10 = q4 - hb, r11 = hb - q4;
      const double ptc = dt * D.pt, pbc = dt * D.pb, hca = 0.5 * dt * D.ca, hcn = 0.5 * dt * D.cn;
#pragma unroll
      for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int q = p; q < 3; ++q) {
          const int k = sym6(p, q);
          const double Rc = dt * V.R[p][q], mh = MHQ[p][q];
          B[0][k] = ((Sa[0][k] + r00 * Rc) - Ft[k]) - ptc * mh;
          B[1][k] = Sa[1][k] + r01 * Rc;
          B[2][k] = r10 * Rc - Sa[0][k];
          B[3][k] = ((r11 * Rc - Sa[1][k]) + Fi[k]) - pbc * mh;
          const double u0 = hca * Vp.R[p][q], w1 = hcn * Vn.R[p][q];
          U[0][k] = u0;
          U[1][k] = (ptc * mh - Fn[k]) - u0;
          W[0][k] = (Fo[k] + pbc * mh) - w1;
          W[1][k] = w1;
        }
    }
    double jz1[3], A1[3][3];
    layer_jz(C.b, e1, ft, fb, jz1);
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int q = p; q < 3; ++q) {
        const double s = j2d * (T3[p][q][0] * jz1[0] + T3[p][q][1] * jz1[1] + T3[p][q][2] * jz1[2]);
        A1[p][q] = s;
        A1[q][p] = s;
      }
    const double r0 = drcp(A1[0][0]);
    const double l10 = A1[1][0] * r0, l20 = A1[2][0] * r0;
    const double a11 = A1[1][1] - l10 * A1[0][1], a12 = A1[1][2] - l10 * A1[0][2];
    const double a22p = A1[2][2] - l20 * A1[0][2];
    const double r1 = drcp(a11);
    const double l21 = (A1[2][1] - l20 * A1[0][1]) * r1;
    const double r2 = drcp(a22p - l21 * a12);
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) {
      double yt[3], yb[3], xt[3], xb[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        yt[k] = cur[(cc * 6 + k) * VBLK];
        yb[k] = cur[(cc * 6 + 3 + k) * VBLK];
        xt[k] = cur[(6 * NC + cc * 6 + k) * VBLK];
        xb[k] = cur[(6 * NC + cc * 6 + 3 + k) * VBLK];
      }
      smv_add(B[0], xt, yt);
      smv_add(B[1], xb, yt);
      smv_add(B[2], xt, yb);
      smv_add(B[3], xb, yb);
      if (l > 0) {
        smv_add(U[0], xa[cc], yt);
        smv_add(U[1], xa[cc] + 3, yt);
      }
      if (l < L - 1) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          xt[k] = nxt[(6 * NC + cc * 6 + k) * VBLK];
          xb[k] = nxt[(6 * NC + cc * 6 + 3 + k) * VBLK];
        }
        smv_add(W[0], xt, yb);
        smv_add(W[1], xb, yb);
      }
      double o[6];
#pragma unroll
      for (int lev = 0; lev < 2; ++lev) {
        double z[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) z[k] = lev == 0 ? ki00 * yt[k] + ki01 * yb[k] : ki10 * yt[k] + ki11 * yb[k];
        z[1] -= l10 * z[0];
        z[2] -= l20 * z[0] + l21 * z[1];
        z[2] *= r2;
        z[1] = (z[1] - a12 * z[2]) * r1;
        z[0] = (z[0] - A1[0][1] * z[1] - A1[0][2] * z[2]) * r0;
#pragma unroll
        for (int k = 0; k < 3; ++k) o[3 * lev + k] = z[k];
      }
      {
        unsigned ln = (unsigned)L * (unsigned)nt;
        asm volatile("" : "+r"(ln));
        const unsigned lo = (unsigned)l * (unsigned)nt + (unsigned)c;
#pragma unroll
        for (int n = 0; n < 6; ++n) x[cc * P6 + (n * ln + lo)] = o[n];
      }
    }
    Vp = V;
    V = Vn;
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
  const int n = els ? n_els : ctx->nown;
  if (n == 0) return PDG_OK;
  VopArgs a{eta_g, wt, wm, nullptr, nullptr, 1.0, 1.0, kh, kv, n0, order};
  k_vop<<<nblocks(n, 128), 128, 0, (cudaStream_t)stream>>>(ctx->view(), a, els, n, d, u, w);
  return check_launch(ctx);
}

// fused vertical stage: implicit (M1 - dt A) x = rhs, or explicit x = M1^-1 (rhs + dt A xin)
//   implicit, kh == 0 and TUNE_VSPLIT 4 (default): k_vimpl_fwd (18-word E tiles) + k_vimpl_bwd_r
//       (coupling blocks rebuilt); otherwise k_vimpl_fwd (30-word tiles) + k_vimpl_bwd
//   explicit: k_vexpl3 (blocks of dt A assembled once per layer)
//   cols / ncols (optional): only the listed owned columns (partitioned runs: the boundary columns,
//   then the interior ones while the ring-1 exchange of the first part is in flight)
int pdg_step_vertical_cols(pdg_ctx* ctx, int ncomp, int implicit, const double* eta_u, const double* eta0,
                           const double* eta1, double dt_mesh, const double* wt, double kh, double kv, double n0,
                           int order, double dt, const double* rhs, const double* xin, double* x, const int* cols,
                           int ncols, void* stream) {
  if (ncomp != 1 && ncomp != 2) return PDG_ERR_SHAPE;
  if (cols && ncols <= 0) return PDG_OK;
  VopArgs a{eta_u, wt, nullptr, eta0, eta1, dt_mesh, 1.0 / dt_mesh, kh, kv, n0, order};
  a.cols = cols;
  a.ncols = ncols;
  const int nt = ctx->nt;
  const int ncol = cols ? ncols : ctx->nown;
  const dim3 grid(nblocks(ncol, VBLK)), blk(VBLK);
  cudaStream_t strm = (cudaStream_t)stream;
  DMesh m = ctx->view();
  const bool ct = implicit && kh == 0.0 && tune_get(TUNE_VSPLIT) == 4;
  // sigma-form column constants: the kh == 0 tracer kernels and the momentum implicit solve
  if (kh == 0.0 && (ncomp == 1 || (SIGU && implicit))) {
    double* vc = ctx->vcol();
    if (!vc) return PDG_ERR_CUDA;
    k_vcol<<<nblocks(ncol, 256), 256, 0, strm>>>(m, eta_u, vc, cols, ncols);
    if (check_launch(ctx) != PDG_OK) return PDG_ERR_CUDA;
    a.vc = vc;
  }
  if (implicit) {
    double* Gs = ctx->ws3((size_t)(ct ? 18 : VT) * ctx->L * nt, ncomp);
    if (!Gs) return PDG_ERR_CUDA;
    const size_t sm = vimpl_fwd_smem(ncomp, ctx->L);
    static unsigned long long attr = 0;
    if (first_on_device(attr)) {
      const int mx = (int)vimpl_fwd_smem(2, 4096), m1 = (int)vimpl_fwd_smem(1, 4096);
      cudaFuncSetAttribute(k_vimpl_fwd<2, 1, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
      cudaFuncSetAttribute(k_vimpl_fwd<1, 1, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, m1);
      cudaFuncSetAttribute(k_vimpl_fwd<2, 1, true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
      cudaFuncSetAttribute(k_vimpl_fwd<1, 1, true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, m1);
      cudaFuncSetAttribute(k_vimpl_fwd<2, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
      cudaFuncSetAttribute(k_vimpl_fwd<1, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, m1);
      cudaFuncSetAttribute(k_vimpl_fwd<2, 1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
      cudaFuncSetAttribute(k_vimpl_fwd<1, 1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, m1);
    }
    if (ct) {
      // bulk-copy ring: plane segments are 16-byte aligned when nt is even (TUNE_BULK bit 1 = on)
      const bool bulk = !cols && nt % 2 == 0 && (tune_get(TUNE_BULK) & 2);
      if (ncomp == 2) {
        if (bulk)
          k_vimpl_fwd<2, 1, true, true, true><<<grid, blk, sm, strm>>>(m, a, dt, rhs, Gs, x);
        else
          k_vimpl_fwd<2, 1, true, true><<<grid, blk, sm, strm>>>(m, a, dt, rhs, Gs, x);
        if (check_launch(ctx) != PDG_OK) return PDG_ERR_CUDA;
        k_vimpl_bwd_r<2><<<grid, blk, 0, strm>>>(m, a, dt, Gs, x);
      } else {
        if (bulk)
          k_vimpl_fwd<1, 1, true, true, true><<<grid, blk, sm, strm>>>(m, a, dt, rhs, Gs, x);
        else
          k_vimpl_fwd<1, 1, true, true><<<grid, blk, sm, strm>>>(m, a, dt, rhs, Gs, x);
        if (check_launch(ctx) != PDG_OK) return PDG_ERR_CUDA;
        k_vimpl_bwd_r<1><<<grid, blk, 0, strm>>>(m, a, dt, Gs, x);
      }
    } else {
      if (ncomp == 2) {
        if (kh == 0.0)
          k_vimpl_fwd<2, 1, true><<<grid, blk, sm, strm>>>(m, a, dt, rhs, Gs, x);
        else
          k_vimpl_fwd<2, 1, false><<<grid, blk, sm, strm>>>(m, a, dt, rhs, Gs, x);
        if (check_launch(ctx) != PDG_OK) return PDG_ERR_CUDA;
        k_vimpl_bwd<2><<<grid, blk, 0, strm>>>(ncol, nt, ctx->L, Gs, x, m.err, cols);
      } else {
        if (kh == 0.0)
          k_vimpl_fwd<1, 1, true><<<grid, blk, sm, strm>>>(m, a, dt, rhs, Gs, x);
        else
          k_vimpl_fwd<1, 1, false><<<grid, blk, sm, strm>>>(m, a, dt, rhs, Gs, x);
        if (check_launch(ctx) != PDG_OK) return PDG_ERR_CUDA;
        k_vimpl_bwd<1><<<grid, blk, 0, strm>>>(ncol, nt, ctx->L, Gs, x, m.err, cols);
      }
    }
  } else {
    const size_t sm = vexpl3_smem(ncomp, ctx->L);
    static unsigned long long attr = 0;
    if (first_on_device(attr)) {
      const int mx = (int)vexpl3_smem(2, 4096), m1 = (int)vexpl3_smem(1, 4096);
      cudaFuncSetAttribute(k_vexpl3<2, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
      cudaFuncSetAttribute(k_vexpl3<1, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, m1);
      cudaFuncSetAttribute(k_vexpl3<2, 1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
      cudaFuncSetAttribute(k_vexpl3<1, 1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, m1);
    }
    if (ncomp == 2) {
      if (kh == 0.0)
        k_vexpl3<2, 1, true><<<grid, blk, sm, strm>>>(m, a, dt, rhs, xin, x);
      else
        k_vexpl3<2, 1, false><<<grid, blk, sm, strm>>>(m, a, dt, rhs, xin, x);
    } else {
      if (kh == 0.0)
        k_vexpl3<1, 1, true><<<grid, blk, sm, strm>>>(m, a, dt, rhs, xin, x);
      else
        k_vexpl3<1, 1, false><<<grid, blk, sm, strm>>>(m, a, dt, rhs, xin, x);
    }
  }
  return check_launch(ctx);
}

int pdg_step_vertical(pdg_ctx* ctx, int ncomp, int implicit, const double* eta_u, const double* eta0,
                      const double* eta1, double dt_mesh, const double* wt, double kh, double kv, double n0, int order,
                      double dt, const double* rhs, const double* xin, double* x, void* stream) {
  return pdg_step_vertical_cols(ctx, ncomp, implicit, eta_u, eta0, eta1, dt_mesh, wt, kh, kv, n0, order, dt, rhs, xin,
                                x, nullptr, 0, stream);
}


}  // extern "C"

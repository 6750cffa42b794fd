// Shared device-side definitions for the prism-DG sm_100a kernels.
//
// Device layouts (all FP64; "c" = column = triangle, Hilbert order):
//   C3   2D nodal field           [3][nt]              idx  k*nt + c
//   P6   prism nodal field        [6][L][nt]           idx (k*L + l)*nt + c
//   P6N  prism field, N comps     [N][6][L][nt]
//   FAC  lateral flux factor      [3 edge][2 v][2 h][L][nt]
//   MASS per-prism 6x6            [36][L][nt]
//   BAND banded column blocks     d [36][L][nt], u [18][L][nt], w [18][L][nt]
// Layer-major planes make a thread-per-column layer loop read one coalesced
// 8-byte word per (node, comp) per warp lane, and keep every per-column 2D
// quantity (J2D, grad phi, normals, eta, b, ...) in registers for the whole
// column.  Prism geometry (z, Jz, grad z) is recomputed from eta, b and the
// sigma fractions instead of being stored (mesh.py:371-408 restated).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/prismdg_b200.h"

namespace pdg {

// ---------------------------------------------------------------- reference-element tables
// Dunavant 6-point rule (dg.py:27-45), 2-point Gauss (dg.py:54-67), edge shapes (dg.py:76-81)
__device__ constexpr double QW[6] = {0.111690794839005, 0.111690794839005, 0.111690794839005,
                                     0.054975871827661, 0.054975871827661, 0.054975871827661};
__device__ constexpr double BARY[6][3] = {{0.108103018168070, 0.445948490915965, 0.445948490915965},
                                          {0.445948490915965, 0.108103018168070, 0.445948490915965},
                                          {0.445948490915965, 0.445948490915965, 0.108103018168070},
                                          {0.816847572980459, 0.091576213509771, 0.091576213509771},
                                          {0.091576213509771, 0.816847572980459, 0.091576213509771},
                                          {0.091576213509771, 0.091576213509771, 0.816847572980459}};
constexpr double GZ = 0.5773502691896258;          // 1/sqrt(3)
constexpr double VLO = 0.21132486540518708;        // (1 - 1/sqrt3)/2
constexpr double VHI = 0.7886751345948129;         // (1 + 1/sqrt3)/2
// VS[v][lev]: vertical point v (zeta = -g, +g), level 0 top / 1 bottom
__device__ constexpr double VS[2][2] = {{VLO, VHI}, {VHI, VLO}};
__device__ constexpr double ZQP[2] = {-GZ, GZ};
__device__ constexpr double DV[2] = {0.5, -0.5};
// ES[h][s]: edge point h, shape s in the edge's own traversal order
__device__ constexpr double ES[2][2] = {{VHI, VLO}, {VLO, VHI}};

// Derived constants of the same quadrature (exact P1 integrals as the rule evaluates them):
//   W1[a]      = sum_q QW BARY_a            (= 1/6 up to the 13-digit rule literals)
//   MHQ[a][b]  = sum_q QW BARY_a BARY_b     (triangle mass pattern, = MH of columns.py:35)
//   T3[a][b][c]= sum_q QW BARY_a BARY_b BARY_c
//   K[a][b]    = sum_v VS[v][a] VS[v][b]   (1D P1 mass on [-1,1] / 2: [[2/3,1/3],[1/3,2/3]])
//   K3[m][a][b]= sum_v VS[v][m] VS[v][a] VS[v][b]
__device__ constexpr double W1[3] = {0.16666666666666607, 0.16666666666666607, 0.16666666666666605};
__device__ constexpr double MHQ[3][3] = {{0.08333333333333315, 0.041666666666666484, 0.041666666666666484},
                                         {0.041666666666666484, 0.08333333333333315, 0.041666666666666484},
                                         {0.041666666666666484, 0.041666666666666484, 0.08333333333333315}};
constexpr double T3D = 0.04999999999999996, T3A = 0.0166666666666666, T3C = 0.008333333333333285;
__device__ constexpr double T3[3][3][3] = {{{T3D, T3A, T3A}, {T3A, T3A, T3C}, {T3A, T3C, T3A}},
                                           {{T3A, T3A, T3C}, {T3A, T3D, T3A}, {T3C, T3A, T3A}},
                                           {{T3A, T3C, T3A}, {T3C, T3A, T3A}, {T3A, T3A, T3D}}};
__device__ constexpr double KM[2][2] = {{0.6666666666666666, 0.33333333333333326},
                                        {0.33333333333333326, 0.6666666666666666}};
constexpr double K3A = 0.5, K3B = 0.16666666666666663;
__device__ constexpr double K3[2][2][2] = {{{K3A, K3B}, {K3B, K3B}}, {{K3B, K3B}, {K3B, K3A}}};

__host__ __device__ constexpr int EV0(int k) { return k; }
__host__ __device__ constexpr int EV1(int k) { return k == 2 ? 0 : k + 1; }

// ---------------------------------------------------------------- error word
__device__ inline void report(pdg_err* e, int code, long long i0, long long i1, double v) {
  if (e && atomicCAS(&e->code, 0, code) == 0) {
    e->i0 = i0;
    e->i1 = i1;
    e->val = v;
  }
}

// ---------------------------------------------------------------- mesh view passed by value
struct DMesh {
  int nt, L;
  int nown;           // columns computed by the stepper (owned); nt = owned + ghosts
  const double* j2d;   // [nt]
  const double* dphx;  // [3][nt]
  const double* dphy;
  const double* elen;
  const double* enx;
  const double* eny;
  const double* b;     // [3][nt] bed at the corners
  const int* nbr;      // [3][nt]  neighbour column or -1
  const int* nbrk;     // [3][nt]  neighbour's local edge
  const int* btag;     // [3][nt]  0 interior, 1 wall, 2 open
  const double* fracs; // [L+1]    sigma fractions (0 surface, 1 bed)
  const int* ninfo;    // [3][nt]  packed (nbr << 4) | (nbrk << 2) | btag  (2D kernels)
  pdg_err* err;
};

// branch-free double reciprocal: MUFU seed + two Newton steps (within 1 ulp of 1/x for normal
// finite x; no IEEE slow-path call, so the scheduler can interleave it with independent work)
__device__ __forceinline__ double drcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
// branch-free double square root of x > 0: rsqrt seed, two Newton steps, one Heron correction
// (within 1 ulp of sqrt(x); the dry-cell checks reject x <= 0 before it matters)
__device__ __forceinline__ double dsqrt_bf(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double hx = 0.5 * x;
  r = r * fma(-hx * r, r, 1.5);
  r = r * fma(-hx * r, r, 1.5);
  const double s0 = x * r;
  return fma(0.5 * r, fma(-s0, s0, x), s0);
}

// branch-free 1/sqrt(x), x > 0: MUFU seed + two Newton steps (within ~1 ulp)
__device__ __forceinline__ double drsqrt(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double hx = 0.5 * x;
  r = r * fma(-hx * r, r, 1.5);
  return r * fma(-hx * r, r, 1.5);
}

// per-column 2D data held in registers for a whole column
struct Col {
  double j2d, dx[3], dy[3], el[3], nx[3], ny[3], b[3];
  int nb[3], nk[3], tag[3];
};

__device__ __forceinline__ double ldg(const double* p) { return __ldg(p); }

__device__ __forceinline__ void load_col(const DMesh& m, int c, Col& C) {
  const int nt = m.nt;
  C.j2d = ldg(m.j2d + c);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    C.dx[k] = ldg(m.dphx + k * nt + c);
    C.dy[k] = ldg(m.dphy + k * nt + c);
    C.el[k] = ldg(m.elen + k * nt + c);
    C.nx[k] = ldg(m.enx + k * nt + c);
    C.ny[k] = ldg(m.eny + k * nt + c);
    C.b[k] = ldg(m.b + k * nt + c);
    C.nb[k] = __ldg(m.nbr + k * nt + c);
    C.nk[k] = __ldg(m.nbrk + k * nt + c);
    C.tag[k] = __ldg(m.btag + k * nt + c);
  }
}

// lean per-triangle data of the 2D stage kernels: grad(phi) is rebuilt from the edge normals,
// grad phi_i = -n_k len_k / J2D with k = (i+1) % 3 the edge opposite vertex i, and the
// neighbour id / local edge / tag come packed in one int -- 116 instead of 188 bytes per triangle
struct Col2 {
  double j2d, dx[3], dy[3], el[3], nx[3], ny[3], b[3];
  int nb[3], nk[3], tag[3];
};
__device__ __forceinline__ void load_col2(const DMesh& m, int c, Col2& C) {
  const int nt = m.nt;
  C.j2d = ldg(m.j2d + c);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    C.el[k] = ldg(m.elen + k * nt + c);
    C.nx[k] = ldg(m.enx + k * nt + c);
    C.ny[k] = ldg(m.eny + k * nt + c);
    C.b[k] = ldg(m.b + k * nt + c);
    const int info = __ldg(m.ninfo + k * nt + c);
    C.tag[k] = info & 3;
    C.nk[k] = (info >> 2) & 3;
    C.nb[k] = info >> 4;
  }
  const double inv = drcp(C.j2d);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int k = i == 2 ? 0 : i + 1;
    C.dx[i] = -(C.nx[k] * C.el[k]) * inv;
    C.dy[i] = -(C.ny[k] * C.el[k]) * inv;
  }
}

__host__ __device__ __forceinline__ constexpr int sym6(int a, int b) {  // packed index of a symmetric 3x3
  return a == b ? a : 3 + a + b - 1;                  // (0,0)0 (1,1)1 (2,2)2 (0,1)3 (0,2)4 (1,2)5
}

// ---------------------------------------------------------------- small helpers
// values at the 6 horizontal points of a corner field (c3 @ BARY.T)
__device__ __forceinline__ void hq(const double c3[3], double out[6]) {
#pragma unroll
  for (int q = 0; q < 6; ++q) out[q] = c3[0] * BARY[q][0] + c3[1] * BARY[q][1] + c3[2] * BARY[q][2];
}

// (J2D/24)(v + sum v)   (columns.py:45-56)
__device__ __forceinline__ void mh_apply3(const double v[3], double j2d, double out[3]) {
  const double s = (v[0] + v[1]) + v[2];
  const double f = j2d / 24.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) out[i] = (v[i] + s) * f;
}
// (6/J2D)(4 v - sum v) with f6 = 6/J2D precomputed
__device__ __forceinline__ void mh_inv3f(const double v[3], double f6, double out[3]) {
  const double s = (v[0] + v[1]) + v[2];
#pragma unroll
  for (int i = 0; i < 3; ++i) out[i] = (4.0 * v[i] - s) * f6;
}
// (6/J2D)(4 v - sum v)  (columns.py:59-69)
__device__ __forceinline__ void mh_inv3(const double v[3], double j2d, double out[3]) {
  const double s = (v[0] + v[1]) + v[2];
  const double f = 6.0 / j2d;
#pragma unroll
  for (int i = 0; i < 3; ++i) out[i] = (4.0 * v[i] - s) * f;
}

// sum_i f_i * d_i with the products and the left-to-right sum rounded like numpy
__device__ __forceinline__ double dot3_rn(const double f[3], const double d[3]) {
  return __dadd_rn(__dadd_rn(__dmul_rn(f[0], d[0]), __dmul_rn(f[1], d[1])), __dmul_rn(f[2], d[2]));
}

// sigma-layer geometry of layer l for free surface eta (mesh.py:389-395, 349-355)
struct LGeo {
  double jz[3];      // half thickness per corner
  double zt[3], zb[3];
  double dzmid[2], djz[2], dztop[2], dzbot[2];
};

__device__ __forceinline__ void layer_geo(const Col& C, const double eta[3], double ft, double fb, LGeo& G) {
  double zm[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double H = __dsub_rn(eta[i], C.b[i]);
    G.zt[i] = __dsub_rn(eta[i], __dmul_rn(ft, H));
    G.zb[i] = __dsub_rn(eta[i], __dmul_rn(fb, H));
    G.jz[i] = __dmul_rn(0.5, __dsub_rn(G.zt[i], G.zb[i]));
    zm[i] = __dmul_rn(0.5, __dadd_rn(G.zt[i], G.zb[i]));
  }
  G.dzmid[0] = dot3_rn(zm, C.dx);
  G.dzmid[1] = dot3_rn(zm, C.dy);
  G.djz[0] = dot3_rn(G.jz, C.dx);
  G.djz[1] = dot3_rn(G.jz, C.dy);
  G.dztop[0] = dot3_rn(G.zt, C.dx);
  G.dztop[1] = dot3_rn(G.zt, C.dy);
  G.dzbot[0] = dot3_rn(G.zb, C.dx);
  G.dzbot[1] = dot3_rn(G.zb, C.dy);
}

// only the half thicknesses (cheap path)
__device__ __forceinline__ void layer_jz(const double b[3], const double eta[3], double ft, double fb, double jz[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double H = __dsub_rn(eta[i], b[i]);
    jz[i] = __dmul_rn(0.5, __dsub_rn(__dsub_rn(eta[i], __dmul_rn(ft, H)), __dsub_rn(eta[i], __dmul_rn(fb, H))));
  }
}

// Mjz[a][b] = sum_q QW BARY_a BARY_b jzq  (the 3x3 horizontal factor of the prism
// mass: M = K (x) (J2D Mjz) with K = [[2/3,1/3],[1/3,2/3]], internal3d.py:114-123)
__device__ __forceinline__ void mass_h(const double jzq[6], double M[3][3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = a; b < 3; ++b) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < 6; ++q) s += QW[q] * BARY[q][a] * BARY[q][b] * jzq[q];
      M[a][b] = s;
      M[b][a] = s;
    }
}

// y = M x for the prism mass in Kronecker form, x/y 6 nodal values
__device__ __forceinline__ void mass_apply_k(const double Mh[3][3], double j2d, const double x[6], double y[6]) {
  double hx[2][3];
#pragma unroll
  for (int lev = 0; lev < 2; ++lev)
#pragma unroll
    for (int a = 0; a < 3; ++a)
      hx[lev][a] = j2d * (Mh[a][0] * x[3 * lev] + Mh[a][1] * x[3 * lev + 1] + Mh[a][2] * x[3 * lev + 2]);
  // K = sum_v VS[v][a] VS[v][b]
  const double k00 = VS[0][0] * VS[0][0] + VS[1][0] * VS[1][0];
  const double k01 = VS[0][0] * VS[0][1] + VS[1][0] * VS[1][1];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    y[a] = k00 * hx[0][a] + k01 * hx[1][a];
    y[3 + a] = k01 * hx[0][a] + k00 * hx[1][a];
  }
}

// 3x3 unpivoted LU solve in place (SPD Mjz); returns false on a zero pivot
__device__ __forceinline__ bool solve3(double A[3][3], double x[3]) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (A[k][k] == 0.0) return false;
    const double inv = 1.0 / A[k][k];
#pragma unroll
    for (int i = k + 1; i < 3; ++i) {
      A[i][k] *= inv;
#pragma unroll
      for (int j = k + 1; j < 3; ++j) A[i][j] -= A[i][k] * A[k][j];
    }
  }
  x[1] -= A[1][0] * x[0];
  x[2] -= A[2][0] * x[0] + A[2][1] * x[1];
  x[2] /= A[2][2];
  x[1] = (x[1] - A[1][2] * x[2]) / A[1][1];
  x[0] = (x[0] - A[0][1] * x[1] - A[0][2] * x[2]) / A[0][0];
  return true;
}

// unpivoted 6x6 LU in place, columns.py:266-277 order; returns failing pivot or -1
__device__ __forceinline__ int lu6(double a[6][6]) {
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    if (a[k][k] == 0.0) return k;
    const double inv = 1.0 / a[k][k];
#pragma unroll
    for (int i = k + 1; i < 6; ++i) {
      a[i][k] = a[i][k] * inv;
#pragma unroll
      for (int j = k + 1; j < 6; ++j) a[i][j] = a[i][j] - a[i][k] * a[k][j];
    }
  }
  return -1;
}

// forward/backward substitution, columns.py:280-289
template <int NR>
__device__ __forceinline__ void lu6_solve(const double a[6][6], double b[6][NR]) {
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
    for (int r = 0; r < NR; ++r) b[i][r] = b[i][r] / a[i][i];
  }
}

__host__ __device__ inline size_t pidx(int k, int l, int c, int L, int nt) {
  return ((size_t)k * L + l) * nt + c;
}

inline int nblocks(long long n, int bs) { return (int)((n + bs - 1) / bs); }
// kernel attributes (dynamic shared-memory limits) are per device: true the first time this
// call site runs on the current device
inline bool first_on_device(unsigned long long& seen) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (seen & bit) return false;
  seen |= bit;
  return true;
}

// occupancy variants of the heavy thread-per-column kernels: __launch_bounds__(128, MINB)
// (MINB 1 -> up to 255 regs / 8 warps per SM, 3 -> 168 regs, 4 -> 128 regs); chosen per
// kernel family at run time through pdg_tune() so one binary can be measured in every variant.
// keys 1, 2 and 13 are retired (superseded vertical-kernel variants, removed)
enum TuneKey { TUNE_HRHS = 0, TUNE_R = 3, TUNE_WT = 4, TUNE_HRHS2 = 5, TUNE_RK = 6, TUNE_VSPLIT = 7, TUNE_PF = 8, TUNE_TILE_PRED = 9, TUNE_TILE_STAGE = 10, TUNE_TILE_COL = 11, TUNE_BULKPF = 12, TUNE_NKEYS = 16 };
constexpr int TUNE_BULK = TUNE_BULKPF;   // bit 1: bulk-copy (cp.async.bulk) rings; bit 0 retired (the F3D->2D
                                         // L2 bulk prefetch of r measured no gain once the stage RHS changed)
int tune_get(int key);

}  // namespace pdg
